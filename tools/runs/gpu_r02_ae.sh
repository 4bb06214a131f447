for v in dense nodense dense nodense; do
  if [ $v = dense ]; then E=""; else E="AS_SR_NODENSE=1"; fi
  env $E timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dn_$v.csv python tools/op_runner.py build 5 > /dev/null 2>&1
  env $E timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dnt_$v.csv python tools/op_runner.py transpose 5 > /dev/null 2>&1
  echo "== $v"; python tools/launches.py gpurun_out/dn_$v.csv | grep sortreduce; python tools/launches.py gpurun_out/dnt_$v.csv | grep sortreduce
done
