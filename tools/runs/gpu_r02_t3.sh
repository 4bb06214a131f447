# warp-tile trace kernel: tests, then cfg 4 timing of variants
timeout 900 python -m pytest tests -m gpu -x -q -k "trace" > gpurun_out/t3_test.log 2>&1; echo "test rc=$?"; tail -3 gpurun_out/t3_test.log
for v in default twI1; do
  if [ $v = default ]; then unset AS_LIB_PATH; else export AS_LIB_PATH=$PWD/paper_1805_03380_b200/build/variants/$v.so; fi
  echo "[$v]"; timeout 300 python tools/time_ops.py trace 20
done
