#!/bin/bash
# Same-box A/B of builds of the engine, interleaved, one process per run (tools/ab_scan.py):
#   bash tools/ab_lib.sh CONFIG REPS OUTDIR "base new ca"
# "new" = paper_2303_09855_b200/libadsann_b200.so, X = paper_2303_09855_b200/libadsann_b200_X.so
CFG=${1:-5}; REPS=${2:-2}; OUT=${3:-gpurun_out}; LIBS=${4:-"base new"}
for r in $(seq 1 $REPS); do
  for lib in $LIBS; do
    if [ $lib = new ]; then unset ADS_LIB_PATH; else export ADS_LIB_PATH=$PWD/paper_2303_09855_b200/libadsann_b200_$lib.so; fi
    python tools/ab_scan.py --config $CFG --steps 10 --reps 1 --variants dense > $OUT/ablib_${CFG}_${lib}_$r.json 2> $OUT/ablib_${CFG}_${lib}_$r.err
    echo "cfg$CFG $lib rep $r: $(grep variant $OUT/ablib_${CFG}_${lib}_$r.err)"
  done
done
