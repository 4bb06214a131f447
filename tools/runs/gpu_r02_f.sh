set -x
timeout 900 python -m pytest tests/test_largen_gpu.py tests/test_kernels_gpu.py -x -q > gpurun_out/r02_largen_test2.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02_largen_test2.log
timeout 600 python tools/ln_time.py --reps 5
AS_LN_GENERIC_TRANSPOSE=1 timeout 600 python tools/ln_time.py transpose1e7 --reps 5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_ln_launches2.csv python tools/ln_time.py build1e7 transpose1e7 --reps 1 > /dev/null 2>&1
python - <<'PY'
import csv, io
txt = open("gpurun_out/r02_ln_launches2.csv").read()
i = txt.index('"ID"')
rows = list(csv.reader(io.StringIO(txt[i:])))
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
for r in rows[1:]:
    if len(r) > iv and "as::" in r[ik]:
        print("%-80s %s" % (r[ik][:80], r[iv]))
PY
