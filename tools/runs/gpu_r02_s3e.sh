timeout 600 python -m pytest tests/test_spmm_csc_gpu.py -x -q > gpurun_out/s3e_test.log 2>&1; echo "test rc=$?"; tail -3 gpurun_out/s3e_test.log
timeout 600 python bench.py --ops spmm > gpurun_out/s3e_bench.log 2> gpurun_out/s3e_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
l=json.loads(open("gpurun_out/s3e_bench.log").read().strip().splitlines()[-1])
for k,v in l["ops"].items():
    if "spmm" in k: print(k, round(v["ms"]*1e3,1), v.get("via_csr_ms"), v["parity"][:40])
PY
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "op_spmm_first/" --csv python tools/op_runner.py spmm_first 1 > gpurun_out/s3e_ncu.csv 2> gpurun_out/s3e_ncu.err; echo "ncu rc=$?"
grep -E "merge|ct_to_c|tile_col" gpurun_out/s3e_ncu.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | grep duration | head -20
