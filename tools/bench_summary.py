"""Print a compact table of a bench.py JSON line (headline + ops)."""
import json
import sys

for line in open(sys.argv[1]):
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "ms_per_step" not in d:
        continue
    print("headline %-10s %10.2f us  %.3e %s  frac=%.3f  e2e=%.3e" % (
        "build", d["ms_per_step"] * 1e3, d["value"], d["unit"], d["roofline"]["frac"],
        (d.get("e2e") or {}).get("value", 0)))
    for k, v in (d.get("ops") or {}).items():
        if "ms" not in v:  # nested sections
            for k2, v2 in v.items():
                if isinstance(v2, dict):
                    print("next %-26s %9.3f ms  %8.1f GB/s  %s" % (k2, v2.get("ms", 0), v2.get("GB/s", 0),
                                                                  v2.get("parity", "")[:30]))
                else:
                    print("next %-26s %s" % (k2, v2))
            continue
        print("op %-16s %10.2f us  %.3e %-10s frac=%.3f  %s" % (k, v["ms"] * 1e3, v["value"], v["unit"],
                                                             v["roofline"]["frac"], v.get("parity", "")[:40]))
    if d.get("cpu_baseline"):
        print("cpu_baseline", d["cpu_baseline"]["value"], d["cpu_baseline"]["unit"])
