set -x
timeout 900 python -m pytest tests/test_largen_gpu.py -x -q > gpurun_out/r02_largen_test.log 2>&1; echo "largen rc=$?"
tail -30 gpurun_out/r02_largen_test.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu2.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02_pytest_gpu2.log
timeout 600 python tools/ln_time.py --reps 5 > gpurun_out/r02_ln1.log 2>&1
cat gpurun_out/r02_ln1.log
timeout 300 python tools/sr_time.py build transpose flush 20
