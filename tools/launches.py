"""Per-kernel average durations from an `ncu --metrics gpu__time_duration.sum --csv` log."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ix = {k: j for j, k in enumerate(hdr)}
agg = collections.OrderedDict()
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    v = float(r[ix["Metric Value"]])
    u = r[ix["Metric Unit"]]
    v = v / 1000.0 if u in ("ns", "nsecond") else (v * 1000.0 if u in ("ms", "msecond") else v)
    name = r[ix["Kernel Name"]].split("(")[0][:70]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
for k, (c, t) in agg.items():
    print("%-72s n=%4d avg=%10.2f us" % (k, c, t / c))
