timeout 900 python -m pytest tests -m gpu -x -q -k "dropin or ref_kernels or api" > gpurun_out/w5_test.log 2>&1; echo "test rc=$?"; tail -3 gpurun_out/w5_test.log
timeout 600 python bench.py --steps 5 --warmup 3 --headline-only > gpurun_out/w5_bench.log 2>&1; echo rc=$?
python -c "
import json
l=json.loads(open('gpurun_out/w5_bench.log').read().strip().splitlines()[-1])
print(l['cpu_baseline']['reference_api_gpu_backend'])"
