#!/bin/bash
# 10 CTAs/SM attempt: 48-register build + step 128 (smem fits 10) vs the default (9 CTAs, step 256).
mkdir -p gpurun_out
for rep in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', round(d['value']), d['clocks']['sm_mhz'])" >> gpurun_out/occ10.log
  ADS_LIB_PATH=paper_2303_09855_b200/libadsann_r48.so timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --step 128 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r48 step128', round(d['value']), d['clocks']['sm_mhz'])" >> gpurun_out/occ10.log
  ADS_LIB_PATH=paper_2303_09855_b200/libadsann_r48.so timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r48 step256', round(d['value']), d['clocks']['sm_mhz'])" >> gpurun_out/occ10.log
done
