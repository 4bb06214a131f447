timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/e2e_timeline.py 2>&1 | grep -E "upload|build|d2h|api_step"
timeout 600 python bench.py --headline-only --no-cpu > gpurun_out/hl.log 2>&1; python -c "
import json; l=json.loads(open('gpurun_out/hl.log').read().strip().splitlines()[-1]); print(l['value'], l['ms_per_step'], l['e2e'])"
