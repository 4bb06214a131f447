# SpMM: 128-bit chunk transposition
timeout 900 python -m pytest tests -m gpu -x -q -k "spmm or cfg3 or mat_times or spmv or matvec or mg_capi" > gpurun_out/x11_test.log 2>&1; echo "test rc=$?"; tail -2 gpurun_out/x11_test.log
timeout 600 python bench.py --steps 5 --warmup 3 --ops spmm --no-cpu > gpurun_out/x11_bench.log 2>&1
python -c "
import json
l=json.loads(open('gpurun_out/x11_bench.log').read().strip().splitlines()[-1])
print({k: (round(v['ms'],4), round(v['roofline']['frac'],4)) for k,v in l['ops'].items() if 'ms' in v})"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x11.csv python tools/op_runner.py spmm 2 > /dev/null 2>&1
grep -i "transpose" gpurun_out/x11.csv | awk -F'","' '{print $NF}' | tr -d '"' | head -8 | tr '\n' ' '; echo
