timeout 300 python tools/e2e_timeline.py 2>&1 | tail -12
