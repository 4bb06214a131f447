set -x
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_ln_launches.csv python tools/ln_time.py build1e7 transpose1e7 --reps 1 > gpurun_out/r02_ln_ncu.log 2>&1
python - <<'PY'
import csv, io, collections
txt = open("gpurun_out/r02_ln_launches.csv").read()
i = txt.index('"ID"')
rows = list(csv.reader(io.StringIO(txt[i:])))
h = rows[0]
ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
for r in rows[1:]:
    if len(r) > iv and ("ln_" in r[ik] or "sortreduce" in r[ik] or "tiles" in r[ik]):
        print(r[ik][:70], r[im], r[iv])
PY
