for c in build1e7 transpose1e7; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lnk_$c.csv python tools/ln_time.py $c --reps 1 > /dev/null 2>&1
python - $c <<'PY'
import csv, io, sys, collections
txt = open("gpurun_out/lnk_%s.csv" % sys.argv[1]).read()
i = txt.index('"ID"')
rows = list(csv.reader(io.StringIO(txt[i:])))
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = collections.OrderedDict()
for r in rows[1:]:
    if len(r) > iv and "as::" in r[ik]:
        d.setdefault(r[iid], [r[ik][:60], {}])[1][r[im]] = float(r[iv].replace(",",""))
items = list(d.values())[-11:]
tot = 0
for k, m in items:
    t = m.get("gpu__time_duration.sum", 0) / 1e3; tot += t
    print("%-60s %8.1f us %8.1f MB" % (k, t, (m.get("dram__bytes_read.sum",0)+m.get("dram__bytes_write.sum",0))/1e6))
print(sys.argv[1], "total", round(tot,1))
PY
done
