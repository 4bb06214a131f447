# bench restructure check + trace on skewed (Zipf) columns with both kernels
timeout 300 python bench.py --steps 5 --warmup 3 --headline-only > gpurun_out/t4_bench.log 2>&1; echo "bench rc=$?"; tail -c 300 gpurun_out/t4_bench.log; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --mg --ops trace > gpurun_out/t4_mg.log 2>&1; echo "mg rc=$?"; tail -c 600 gpurun_out/t4_mg.log; echo
for v in "AS_TRACE_ENGINE=0" "AS_TRACE_ENGINE=1"; do echo "[$v]"; env $v timeout 300 python tools/time_ops.py trace5 20; done
