# SpMM row/transpose kernel times with and without the L2 persisting window
for w in 0 1; do
  AS_SPMM_L2WIN=$w ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/spmm_w$w.csv python tools/op_runner.py spmm 2 > /dev/null 2>&1
  echo "win=$w"; python tools/launches.py gpurun_out/spmm_w$w.csv | grep -i "spmm\|transpose"
  AS_SPMM_L2WIN=$w python tools/time_ops.py spmm 10
done
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p.L2_cache_size, getattr(p,'persisting_l2_cache_max_size',None))"
