set -x
timeout 900 python -m pytest tests/test_largen_gpu.py tests/test_api_gpu.py -x -q > gpurun_out/r02_t8.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02_t8.log
timeout 600 python tools/ln_time.py transpose1e7 transpose5e7 --reps 5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_ln_launches6.csv python tools/ln_time.py transpose1e7 --reps 1 > /dev/null 2>&1
python - <<'PY'
import csv, io
txt = open("gpurun_out/r02_ln_launches6.csv").read()
i = txt.index('"ID"')
rows = list(csv.reader(io.StringIO(txt[i:])))
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
for r in rows[1:][-11:]:
    if len(r) > iv and "as::" in r[ik]:
        print("%-80s %s" % (r[ik][:80], r[iv]))
PY
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --mg --steps 3 --warmup 3 --no-cpu --ops trace,spmm,spgemm > gpurun_out/r02_mg1.log 2>&1; echo "mg rc=$?"
python - <<'PY'
import json
l=json.loads(open("gpurun_out/r02_mg1.log").read().strip().splitlines()[-1])
print(json.dumps(l.get("ops_multi_gpu"))[:2500])
PY
