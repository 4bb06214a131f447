"""Hottest CUDA source lines of one kernel from an ncu report:
    python tools/ncu_lines.py report.ncu-rep <kernel-regex> [launch-skip] [top]
Aggregates 'Warp Stall Sampling (All Samples)' per (file, line) using
`ncu --page source --print-source cuda,sass --csv`."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
import os
METRIC = os.environ.get("NCU_METRIC", "Warp Stall Sampling (All Samples)")
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
cur_file = "?"
hdr = None
agg = []
total = 0.0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        i_s = r.index(METRIC)
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    try:
        v = float(r[i_s])
    except (ValueError, IndexError):
        continue
    total += v
    agg.append((v, cur_file, r[0], r[1].strip()[:90]))
print("total samples %.0f" % total)
for v, f, ln, src in sorted(agg, reverse=True)[:top]:
    print("%6.1f%%  %-14s %5s  %s" % (100 * v / max(total, 1), f, ln, src))
