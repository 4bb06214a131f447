set -x
timeout 900 python -m pytest tests/test_dropin_gpu.py -x -q > gpurun_out/r02_dropin.log 2>&1; echo "dropin rc=$?"
tail -15 gpurun_out/r02_dropin.log
timeout 900 python bench.py > gpurun_out/r02_bench2.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=json.loads(open("gpurun_out/r02_bench2.log").read().strip().splitlines()[-1])
print(json.dumps(l["cpu_baseline"])); print(json.dumps(l["ops"].get("flush_cfg2_api")))
PY
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_ref2.log 2>&1; echo "ref rc=$?"
tail -c 1500 gpurun_out/r02_bench_ref2.log
bash tools/ncu_ops.sh r02a
python tools/make_traffic.py r02a gpurun_out/r02a_traffic.json
