timeout 1500 python -m pytest tests -m gpu -x -q -k "largen or configs or funnel or kernels" > gpurun_out/x9_test.log 2>&1; echo "test rc=$?"; tail -2 gpurun_out/x9_test.log
timeout 600 python bench.py --steps 5 --warmup 3 --ops large --no-cpu > gpurun_out/x9_bench.log 2>&1
python -c "
import json
l=json.loads(open('gpurun_out/x9_bench.log').read().strip().splitlines()[-1])
print({k: (round(v['ms'],4), round(v['roofline']['frac'],4)) for k,v in l['ops']['large_n'].items()})"
