#!/bin/bash
# Launch times (ns, ncu serialised) of the coarse-stage kernels for one config.
cfg=${1:-2}
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k 'regex:tc_gemm|tc_rotate|prefilter|center_norms|apply_kernel|approx_gemm|split_tf32' -c 12 --csv \
    python bench.py --config "$cfg" --steps 1 --warmup 3 --no-cpu-baseline --kmeans-init 1 --kmeans-iters 3 2>/dev/null \
  | grep -E 'tc_gemm|tc_rotate|prefilter|center_norms|apply_kernel|approx_gemm|split_tf32' \
  | awk -F'","' '{n=$5; sub(/\(.*/, "", n); sub(/.*::/, "", n); v=$NF; gsub(/"/, "", v); print "cfg'"$cfg"' " n " " v " ns"}'
