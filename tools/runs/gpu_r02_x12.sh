# trace: more warps with smaller buffers
for v in default tw9 tw10; do
  if [ $v = default ]; then unset AS_LIB_PATH; else export AS_LIB_PATH=$PWD/paper_1805_03380_b200/build/variants/$v.so; fi
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x12.csv python tools/op_runner.py trace 5 > /dev/null 2>&1
  echo "[$v] $(grep trace_warp gpurun_out/x12.csv | awk -F'","' '{print $NF}' | tr -d '"' | head -5 | tr '\n' ' ')"
done
