#!/bin/bash
# Same-box A/B of the query order (bench.py --query-order 0 vs 2 = longest first).
mkdir -p gpurun_out
for cfg in ${CFGS:-2 3}; do
  for rep in 1 2 3; do
    for qo in 0 2; do
      timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --query-order $qo 2>/dev/null \
        | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $cfg order $qo', round(d['value']), 'scan', round(d['stages_ms']['scan'], 3), d['clocks']['sm_mhz'], d['config']['recall_at_k'])" \
        >> gpurun_out/order_ab.log 2>&1
    done
  done
done
