timeout 900 python -m pytest tests -m gpu -x -q -k "api or dropin or ref_kernels or configs" > gpurun_out/w1_test.log 2>&1; echo "test rc=$?"; tail -3 gpurun_out/w1_test.log
timeout 600 python bench.py --steps 5 --warmup 3 --ops flush_api --no-cpu > gpurun_out/w1_bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=json.loads(open("gpurun_out/w1_bench.log").read().strip().splitlines()[-1])
print(json.dumps(l["ops"]["flush_cfg2_api"], indent=0)[:900])
PY
