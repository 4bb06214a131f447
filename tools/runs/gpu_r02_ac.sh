set -x
timeout 1200 python -m pytest tests/test_largen_gpu.py tests/test_kernels_gpu.py tests/test_configs_gpu.py -x -q > gpurun_out/r02_t16.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r02_t16.log
timeout 600 python tools/ln_time.py build1e7 build1e8 --reps 5
timeout 300 python tools/sr_time.py build transpose flush 40
