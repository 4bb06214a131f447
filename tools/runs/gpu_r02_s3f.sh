for v in "" kc32 kc8; do
  if [ -n "$v" ]; then export AS_LIB_PATH=paper_1805_03380_b200/build/variants/$v.so; else unset AS_LIB_PATH; fi
  echo "== variant [$v]"
  python tools/time_ops.py spmm 10
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/s3f_$v.csv python tools/op_runner.py spmm 1 > /dev/null 2>&1
  python tools/launches.py gpurun_out/s3f_$v.csv | grep -i "spmm\|transpose" | head -8
done
