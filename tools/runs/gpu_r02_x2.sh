# add: count published before the output staging (default) vs after (prev)
timeout 600 python -m pytest tests -m gpu -x -q -k "add or linear_combine or cfg5" > gpurun_out/x2_test.log 2>&1; echo "test rc=$?"; tail -2 gpurun_out/x2_test.log
for rep in 1 2; do for v in default prev; do
  if [ $v = default ]; then unset AS_LIB_PATH; else export AS_LIB_PATH=$PWD/paper_1805_03380_b200/build/variants/$v.so; fi
  echo "[$v] $(timeout 300 python tools/time_ops.py add 30)"
done; done
unset AS_LIB_PATH
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x2_new.csv python tools/op_runner.py add 5 > /dev/null 2>&1
AS_LIB_PATH=$PWD/paper_1805_03380_b200/build/variants/prev.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x2_prev.csv python tools/op_runner.py add 5 > /dev/null 2>&1
grep add_tile gpurun_out/x2_new.csv | awk -F'","' '{print "new", $NF}' | tr -d '"' | head -6
grep add_tile gpurun_out/x2_prev.csv | awk -F'","' '{print "prev", $NF}' | tr -d '"' | head -6
