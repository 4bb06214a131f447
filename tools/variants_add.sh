for v in default; do
  if [ $v = default ]; then unset AS_LIB_PATH; else export AS_LIB_PATH=$PWD/paper_1805_03380_b200/build/variants/$v.so; fi
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/var_$v.csv python tools/op_runner.py add 3 > /dev/null 2>&1
  echo "$v $(grep add_tile gpurun_out/var_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ') part $(grep add_part gpurun_out/var_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
