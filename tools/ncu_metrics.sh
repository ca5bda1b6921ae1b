#!/bin/bash
# ncu_metrics.sh KERNEL_REGEX METRICS -- bench args...   (one launch after 3 warm-up launches)
k=$1; m=$2; shift 3
ncu --metrics "$m" --clock-control none -k "regex:$k" -s 3 -c 1 --csv python bench.py "$@" 2>/dev/null \
  | python3 -c '
import csv, sys
rows = list(csv.reader(sys.stdin))
i = next(j for j, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i]
for r in rows[i + 1:]:
    if len(r) != len(h):
        continue
    d = dict(zip(h, r))
    print(d.get("Metric Name"), d.get("Metric Unit"), d.get("Metric Value"))
'
