for v in default tr4 tr6; do
  if [ $v = default ]; then unset AS_LIB_PATH; else export AS_LIB_PATH=$PWD/paper_1805_03380_b200/build/variants/$v.so; fi
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tr_$v.csv python tools/op_runner.py trace 3 > /dev/null 2>&1
  echo "$v $(python tools/launches.py gpurun_out/tr_$v.csv | grep trace_partial)"
done
