#!/bin/bash
# Every bench line of the round on one box, outputs under gpurun_out/final/.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/final
cd "${GRAFT_REPO_ROOT:-.}"
run() { local tag=$1; shift; timeout 1500 python bench.py "$@" > gpurun_out/final/$tag.json 2> gpurun_out/final/$tag.log; echo "$tag rc=$?" >> gpurun_out/final/rc.txt; }
run default
run reference --impl reference --steps 3 --warmup 3
run cfg1 --config 1
run cfg3 --config 3
run transform --mode transform --steps 5 --warmup 3
run dco --mode dco --steps 3 --warmup 3
run theory --mode theory --steps 3 --warmup 3
run cfg2 --config 2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/final/rc.txt
# launch list of the default command's timed region (the scan's share of the step)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
  --log-file gpurun_out/final/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra \
  > gpurun_out/final/launches.log 2>&1; echo "launches rc=$?" >> gpurun_out/final/rc.txt
