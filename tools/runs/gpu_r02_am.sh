set -x
timeout 600 python -m pytest tests/test_api_gpu.py -x -q 2>&1 | tail -3
timeout 300 python tools/e2e_timeline.py 2>&1 | tail -10
timeout 300 python bench.py --headline-only > gpurun_out/am_bench.log 2>&1; echo rc=$?
python -c "
import json;l=json.loads(open('gpurun_out/am_bench.log').read().strip().splitlines()[-1]);print(l['value'],l['ms_per_step'],l['e2e'])"
