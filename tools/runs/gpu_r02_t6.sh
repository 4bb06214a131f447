for rep in 1 2 3; do
for v in default prev; do
  if [ $v = default ]; then unset AS_LIB_PATH; else export AS_LIB_PATH=$PWD/paper_1805_03380_b200/build/variants/$v.so; fi
  echo "[$v] $(timeout 300 python tools/time_ops.py trace 30)"
done; done
unset AS_LIB_PATH
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t6_new.csv python tools/op_runner.py trace 5 > /dev/null 2>&1
AS_LIB_PATH=$PWD/paper_1805_03380_b200/build/variants/prev.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t6_prev.csv python tools/op_runner.py trace 5 > /dev/null 2>&1
grep trace_warp gpurun_out/t6_new.csv | awk -F'","' '{print "new", $NF}' | tr -d '"' | head -6
grep trace_warp gpurun_out/t6_prev.csv | awk -F'","' '{print "prev", $NF}' | tr -d '"' | head -6
