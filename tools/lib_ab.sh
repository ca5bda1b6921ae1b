#!/bin/bash
# Same-box A/B of library builds: VARIANT (a .so built with other flags, e.g.
#   make -C paper_2303_09855_b200/csrc OUT=../libadsann_qf.so OBJDIR=../../build/objqf EXTRA=-DADS_QF32)
# against the default library.  Parity of the variant first (GPU parity suite),
# then alternating config runs.  Output: gpurun_out/lib_ab.log
set -u
V=${VARIANT:?path of the variant .so}
mkdir -p gpurun_out
ADS_LIB_PATH=$V timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/lib_ab_parity.log 2>&1
echo "variant parity rc=$?" >> gpurun_out/lib_ab.log
for cfg in ${CFGS:-2}; do
  for rep in 1 2 3; do
    for lib in paper_2303_09855_b200/libadsann_b200.so $V; do
      ADS_LIB_PATH=$lib timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null \
        | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $cfg', '$lib'.split('/')[-1], round(d['value']), 'scan', round(d['stages_ms']['scan'], 3), d['clocks']['sm_mhz'])" \
        >> gpurun_out/lib_ab.log 2>&1
    done
  done
done
