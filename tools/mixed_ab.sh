#!/bin/bash
# MIXED scan (certified fp32 walkers + one exact warp, lag-1 merge; ADS_SCAN_MIXED=1) vs the exact kernel:
# parity against the lag-1 oracle first, then alternating sustained runs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mixed.py -m gpu -x -q \
    > gpurun_out/mixed_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/mixed_parity.log
for cfg in ${CFGS:-2}; do
  for rep in 1 2; do
    for m in 0 1; do
      ADS_SCAN_MIXED=$m timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null \
        | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $cfg mixed=$m', round(d['value']), 'scan', round(d['stages_ms']['scan'], 3), 'dims', round(d['dims_per_query']), d['clocks']['sm_mhz'], d['config']['recall_at_k'])" \
        >> gpurun_out/mixed_ab.log 2>&1
    done
  done
done
