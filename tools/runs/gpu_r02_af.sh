AS_LIB_PATH=paper_1805_03380_b200/build/variants/t256.so timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_configs_gpu.py tests/test_edges_gpu.py -x -q 2>&1 | tail -2
for v in base t256 base t256; do
  if [ $v = base ]; then L=""; else L="AS_LIB_PATH=paper_1805_03380_b200/build/variants/$v.so"; fi
  env $L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sh_$v.csv python tools/op_runner.py build 5 > /dev/null 2>&1
  env $L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sht_$v.csv python tools/op_runner.py transpose 5 > /dev/null 2>&1
  env $L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/shf_$v.csv python tools/op_runner.py flush 5 > /dev/null 2>&1
  echo "== $v"; for f in sh sht shf; do python tools/launches.py gpurun_out/${f}_$v.csv | grep sortreduce | tail -1; done
  env $L timeout 300 python tools/sr_time.py build transpose flush 40
done
