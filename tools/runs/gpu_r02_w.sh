set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_t12.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02_t12.log
timeout 300 python tools/sr_time.py build transpose flush 60
timeout 600 python tools/ln_time.py --reps 5
