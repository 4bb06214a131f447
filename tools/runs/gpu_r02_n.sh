set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_configs_gpu.py tests/test_edges_gpu.py tests/test_largen_gpu.py -x -q > gpurun_out/r02_t7.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02_t7.log
timeout 300 python tools/sr_time.py build transpose flush 30
AS_SR_NODEFER=1 timeout 300 python tools/sr_time.py build transpose flush 30
AS_LIB_PATH=paper_1805_03380_b200/build/variants/nb2048.so timeout 300 python tools/sr_time.py build transpose flush 30
