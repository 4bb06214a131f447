"""Summarise an `ncu --page source --print-source sass --csv` dump: stall
reasons and the hottest SASS instructions (with their source mapping)."""
import csv
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
data = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
i_a = hdr.index("Address")
stall_cols = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(f(r[i_s]) for r in data)
print("total samples", tot)
agg = {k: sum(f(r[hdr.index(k)]) for r in data) for k in stall_cols}
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]:
    print("  %-26s %5.1f%%" % (k, 100 * v / max(tot, 1)))
for r in sorted(data, key=lambda r: -f(r[i_s]))[:ntop]:
    print("%6s %6.0f  %s" % (r[i_a], f(r[i_s]), r[i_src][:100]))
