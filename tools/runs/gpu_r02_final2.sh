set -x
start=$(date +%s)
timeout 900 python bench.py > gpurun_out/r02f_bench.log 2> gpurun_out/r02f_bench.err; echo "bench rc=$? seconds=$(( $(date +%s) - start ))"
tail -3 gpurun_out/r02f_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r02f_bench_ref.log 2>&1; echo "ref rc=$?"
python - <<'PY'
import json
l=json.loads(open("gpurun_out/r02f_bench.log").read().strip().splitlines()[-1])
print("headline", l["value"], l["ms_per_step"], l["roofline"]["frac"], l["clocks"])
print("e2e", l["e2e"]["value"], l["e2e"]["ms_median"])
print("cpu", l["cpu_baseline"]["value"], l["cpu_baseline"]["reference_numba"]["value"] if l["cpu_baseline"].get("reference_numba") else None)
for k,v in l["ops"].items():
    if isinstance(v, dict) and "ms" in v: print(k, round(v["ms"],4), v.get("roofline",{}).get("frac"), v.get("api_ms"), v.get("reference_ms"))
for k,v in l["ops"].get("large_n",{}).items(): print(k, round(v["ms"],4), v["roofline"]["frac"])
r=json.loads(open("gpurun_out/r02f_bench_ref.log").read().strip().splitlines()[-1])
print("ref", r["value"], r["ms_per_step"], r.get("reference_numba",{}).get("value"))
PY
