timeout 600 python -m pytest tests -m gpu -x -q -k "spmm or mat_times or cfg3 or csc or first or spmv or matvec" > gpurun_out/s3g_test.log 2>&1; echo "test rc=$?"; tail -3 gpurun_out/s3g_test.log
for v in "" "AS_SPMM_UNSTAGED=1"; do echo "[$v]"; env $v python tools/time_ops.py spmm 10; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/s3g.csv python tools/op_runner.py spmm 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/s3g.csv | grep -i "spmm\|transpose" | head -8
