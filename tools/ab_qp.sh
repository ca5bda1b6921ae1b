mkdir -p gpurun_out/qp
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/qp/tests.txt 2>&1; tail -2 gpurun_out/qp/tests.txt
for r in 1 2; do for lib in qp0 new; do
  if [ $lib = new ]; then unset ADS_LIB_PATH; else export ADS_LIB_PATH=$PWD/paper_2303_09855_b200/libadsann_b200_$lib.so; fi
  for v in dense dense+lag; do
    python tools/ab_scan.py --config 3 --steps 10 --reps 1 --variants $v > gpurun_out/qp/ab3_${lib}_${v}_$r.json 2> gpurun_out/qp/ab3_${lib}_${v}_$r.err
    echo "cfg3 $lib $v rep $r: $(grep variant gpurun_out/qp/ab3_${lib}_${v}_$r.err)"
  done
  python tools/ab_scan.py --config 2 --steps 10 --reps 1 --variants dense > gpurun_out/qp/ab2_${lib}_$r.json 2> gpurun_out/qp/ab2_${lib}_$r.err
  echo "cfg2 $lib rep $r: $(grep variant gpurun_out/qp/ab2_${lib}_$r.err)"
done; done
