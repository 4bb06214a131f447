set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu3.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_pytest_gpu3.log
timeout 900 python bench.py > gpurun_out/r02_bench3.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02_bench3.log
python - <<'PY'
import json
l=json.loads(open("gpurun_out/r02_bench3.log").read().strip().splitlines()[-1])
print(l["value"], l["ms_per_step"], l["roofline"]["frac"])
for k,v in l["ops"].items():
    if isinstance(v, dict) and "ms" in v: print(k, v["ms"], v.get("roofline",{}).get("frac"))
for k,v in l["ops"].get("large_n",{}).items(): print(k, v["ms"], v["roofline"]["frac"], v["parity"])
PY
bash tools/ncu_ops.sh r02b
python tools/make_traffic.py r02b gpurun_out/r02b_traffic.json
