"""DRAM traffic per launch from `ncu --set full --csv --page raw` output files:
    python tools/ncu_traffic.py gpurun_out/full_build.csv [...]
Prints kernel, dram read/write MB and duration; used for bench.py's
roofline.traffic (profiles/r01_traffic.json)."""
import csv
import io
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TSCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def parse(path):
    txt = open(path).read()
    i = txt.index('"ID","Process ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    h, units = rows[0], rows[1]
    ir, iw, it, ik = (h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"),
                      h.index("gpu__time_duration.sum"), h.index("Kernel Name"))
    out = []
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        f = lambda j: float(r[j].replace(",", ""))
        out.append({"kernel": r[ik].split("(")[0], "dram_read": f(ir) * SCALE.get(units[ir], 1),
                    "dram_write": f(iw) * SCALE.get(units[iw], 1), "us": f(it) * TSCALE.get(units[it], 1)})
    return out


if __name__ == "__main__":
    res = {}
    for p in [a for a in sys.argv[1:] if not a.startswith("--")]:
        for k in parse(p):
            print("%-40s %-50s read %9.2f MB write %9.2f MB %9.2f us" % (p.split("/")[-1], k["kernel"][:50],
                                                                          k["dram_read"] / 1e6, k["dram_write"] / 1e6,
                                                                          k["us"]))
            res[p.split("/")[-1]] = k
    if "--json" in sys.argv:
        print(json.dumps(res))
