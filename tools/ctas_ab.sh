#!/bin/bash
# Resident search CTAs per SM (0 = occupancy maximum, 9 at config 2) under sustained load.
mkdir -p gpurun_out
for rep in 1 2; do
  for c in 0 8 7 6; do
    timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --ctas-per-sm $c 2>/dev/null \
      | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ctas $c', round(d['value']), 'scan', round(d['stages_ms']['scan'], 3), d['clocks']['sm_mhz'])" \
      >> gpurun_out/ctas_ab.log 2>&1
  done
done
