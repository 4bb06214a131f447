set -x
timeout 900 python -m pytest tests/test_largen_gpu.py -x -q > gpurun_out/r02_largen_test4.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02_largen_test4.log
timeout 600 python tools/ln_time.py transpose1e7 transpose5e7 --reps 5
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ln_transpose_finish|ln_scatter|ln_count" -c 6 -o gpurun_out/r02_ln_full2 -f python tools/ln_time.py transpose1e7 --reps 1 > gpurun_out/r02_ln_full2.log 2>&1
echo ncu rc=$?
