set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_t9.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02_t9.log
timeout 300 python tools/sr_time.py build transpose flush 40
timeout 300 python tools/sr_time.py build transpose flush 40
timeout 600 python tools/ln_time.py build1e7 --reps 5
