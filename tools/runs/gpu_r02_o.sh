set -x
timeout 300 python tools/sr_time.py build transpose flush 30
AS_LIB_PATH=paper_1805_03380_b200/build/variants/nb2048.so timeout 300 python tools/sr_time.py build transpose flush 30
timeout 900 python bench.py > gpurun_out/r02_bench4.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=json.loads(open("gpurun_out/r02_bench4.log").read().strip().splitlines()[-1])
print(l["value"], l["ms_per_step"], l["roofline"]["frac"])
for k,v in l["ops"].items():
    if isinstance(v, dict) and "ms" in v: print(k, v["ms"], v.get("roofline",{}).get("frac"), v.get("api_ms"))
for k,v in l["ops"].get("large_n",{}).items(): print(k, v["ms"], v["roofline"]["frac"])
PY
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench4_ref.log 2>&1; echo "ref rc=$?"
KEEP_REP="build transpose_1e7_f32" bash tools/ncu_ops.sh r02b
python tools/make_traffic.py r02b gpurun_out/r02b_traffic.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02b_launches_bench.csv python bench.py --steps 2 --warmup 3 --ops transpose --no-cpu > gpurun_out/r02b_ncu_bench.log 2>&1; echo "launches rc=$?"
du -sh gpurun_out
