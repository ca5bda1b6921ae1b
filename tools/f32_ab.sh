#!/bin/bash
# A/B of the certified fp32 walk (ADS_SCAN_F32=1) against the exact fp64 walk:
# parity first (the whole GPU parity suite and the full-size test under F32),
# then alternating bench runs on the same box.
set -u
mkdir -p gpurun_out
ADS_SCAN_F32=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q \
    > gpurun_out/f32_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/f32_parity.log
for cfg in ${CFGS:-2 3}; do
  for rep in 1 2; do
    for f in 0 1; do
      ADS_SCAN_F32=$f timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 2>/dev/null \
        | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $cfg f32=$f', round(d['value']), d['clocks']['sm_mhz'], d.get('roofline',{}).get('frac'), d.get('recall'))" \
        >> gpurun_out/f32_ab.log 2>&1
    done
  done
done
