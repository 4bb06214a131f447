for v in "" "AS_CM_NO_HINTS=1"; do
  env $v timeout 600 python bench.py --ops spmm --skip-slow-checks > gpurun_out/s3c_bench.log 2> gpurun_out/s3c_bench.err; echo "[$v] bench rc=$?"
  python - <<'PY'
import json
l=json.loads(open("gpurun_out/s3c_bench.log").read().strip().splitlines()[-1])
for k,v in l["ops"].items():
    if "spmm" in k: print(k, round(v["ms"]*1e3,1), v.get("via_csr_ms"))
PY
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_red.sum --clock-control none --nvtx --nvtx-include "op_spmm_first/" --csv python tools/op_runner.py spmm_first 1 > gpurun_out/s3c_ncu.csv 2> gpurun_out/s3c_ncu.err; echo "ncu rc=$?"
grep -E "merge|ct_to_c|tile_col" gpurun_out/s3c_ncu.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | head -20
