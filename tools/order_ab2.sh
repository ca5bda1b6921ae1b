#!/bin/bash
# Sustained-load A/B of query orders 2 (longest first) and 1 (L2 locality): 20 timed steps
# each, alternating, to see whether fewer DRAM bytes buy clock headroom under the power cap.
mkdir -p gpurun_out
for rep in 1 2 3; do
  for qo in 2 1; do
    timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --query-order $qo 2>/dev/null \
      | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('order $qo', round(d['value']), 'scan', round(d['stages_ms']['scan'], 3), d['clocks'])" \
      >> gpurun_out/order_ab2.log 2>&1
  done
done
