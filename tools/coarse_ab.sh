#!/bin/bash
# Same-box A/B of the coarse GEMM: ADS_TC_COARSE=0 (tiled tc_gemm_kernel) vs the default
# persistent kernel; coarse-stage ms and end-to-end q/s at nprobe 64 and 8.
mkdir -p gpurun_out
for np in 64 8; do
  for rep in 1 2; do
    for v in 1 0; do
      ADS_TC_COARSE=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --nprobe $np 2>gpurun_out/coarse_ab_$v.err \
        | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nprobe $np tc_coarse=$v', round(d['value']), 'coarse', round(d['stages_ms']['coarse'], 4), 'scan', round(d['stages_ms']['scan'], 3), d['clocks']['sm_mhz'])" \
        >> gpurun_out/coarse_ab.log 2>&1
      grep "coarse prefilter" gpurun_out/coarse_ab_$v.err | tail -1 >> gpurun_out/coarse_ab.log
    done
  done
done
