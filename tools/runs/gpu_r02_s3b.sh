set -x
timeout 600 python -m pytest tests/test_spmm_csc_gpu.py tests/test_configs_gpu.py -x -q -k "spmm or csc or first" > gpurun_out/s3b_test.log 2>&1; echo "test rc=$?"
tail -15 gpurun_out/s3b_test.log
timeout 600 python bench.py --ops spmm > gpurun_out/s3b_bench.log 2> gpurun_out/s3b_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/s3b_bench.err
python - <<'PY'
import json
l=json.loads(open("gpurun_out/s3b_bench.log").read().strip().splitlines()[-1])
for k,v in l["ops"].items():
    if "spmm" in k: print(k, json.dumps({a:b for a,b in v.items() if a!="roofline"}), v["roofline"]["frac"])
PY
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "op_spmm_first/" --csv python tools/op_runner.py spmm_first 2 > gpurun_out/s3b_ncu.csv 2> gpurun_out/s3b_ncu.err; echo "ncu rc=$?"
grep -E "merge|ct_to_c|tile_col" gpurun_out/s3b_ncu.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | head -20
