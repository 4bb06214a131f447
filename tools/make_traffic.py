"""profiles/r01_traffic.json from one `ncu --set full --csv --page raw`
capture of `tools/op_runner.py all 1`: per op, the DRAM bytes and duration
of its dominant kernel (the last matching launch)."""
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_traffic import parse  # noqa: E402

MATCH = {
    "build": "persist_bucket_kernel<double, CooSrc<int",
    "transpose": "persist_bucket_kernel<double, CscSrc<double>, NoSrc",
    "flush": "persist_bucket_kernel<double, CscSrc<double>, CooSrc",
    "spmm": "spmm_rows_lanes_kernel",
    "trace": "trace_partial_kernel",
    "add": "add_tile_kernel",
    "spgemm": "persist_bucket_kernel<double, NoSrc<double>, NoSrc",
}


def main():
    rows = parse(sys.argv[1])
    for r in rows:
        r["kernel"] = r["kernel"].replace("as::", "")
    out = {}
    for op, pat in MATCH.items():
        hits = [r for r in rows if pat in r["kernel"]]
        if hits:
            out[op] = hits[-1]
    json.dump(out, open(sys.argv[2], "w"), indent=1, sort_keys=True)
    for op, r in sorted(out.items()):
        print("%-10s %-60s %8.2f MB %9.2f us" % (op, r["kernel"][:60], (r["dram_read"] + r["dram_write"]) / 1e6,
                                                 r["us"]))


if __name__ == "__main__":
    main()
