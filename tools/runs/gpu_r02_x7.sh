timeout 1500 python -m pytest tests -m gpu -x -q -k "kernels or edges or api or funnel or largen" > gpurun_out/x7_test.log 2>&1; echo "test rc=$?"; tail -2 gpurun_out/x7_test.log
timeout 600 python bench.py --steps 20 --warmup 5 --ops flush,transpose --no-cpu > gpurun_out/x7_bench.log 2>&1; echo rc=$?
python -c "
import json
l=json.loads(open('gpurun_out/x7_bench.log').read().strip().splitlines()[-1])
print('build', l['ms_per_step']); [print(k, v['ms']) for k,v in l['ops'].items() if 'ms' in v]"
