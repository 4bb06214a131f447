"""profiles/rNN_traffic.json from the per-op `ncu --set full` captures of
tools/ncu_ops.sh (one NVTX-ranged call of each op per capture): per op, the
DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) and the duration
summed over EVERY launch of that call, plus the per-kernel breakdown.

    python tools/make_traffic.py TAG out.json   (reads gpurun_out/TAG_ncu_<op>.csv)
"""
import glob
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_traffic import parse  # noqa: E402


def main():
    tag, dst = sys.argv[1], sys.argv[2]
    out = {}
    for path in sorted(glob.glob("gpurun_out/%s_ncu_*.csv" % tag)):
        op = os.path.basename(path)[len(tag) + 5:-4]
        try:
            rows = parse(path)
        except ValueError:
            continue
        if not rows:
            continue
        ks = [{"kernel": r["kernel"].replace("as::", "")[:90], "dram_read": r["dram_read"],
               "dram_write": r["dram_write"], "us": r["us"]} for r in rows]
        out[op] = {"launches": len(ks), "dram_read": sum(k["dram_read"] for k in ks),
                   "dram_write": sum(k["dram_write"] for k in ks), "us": sum(k["us"] for k in ks), "kernels": ks}
    json.dump(out, open(dst, "w"), indent=1, sort_keys=True)
    for op, r in sorted(out.items()):
        print("%-12s %2d launches %10.2f MB %9.2f us" % (op, r["launches"], (r["dram_read"] + r["dram_write"]) / 1e6,
                                                        r["us"]))


if __name__ == "__main__":
    main()
