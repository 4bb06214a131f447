set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_t17.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r02_t17.log
timeout 300 python tools/sr_time.py build transpose flush 40
AS_SR_NODENSE=1 timeout 300 python tools/sr_time.py build transpose flush 40
timeout 300 python tools/sr_time.py build transpose flush 40
