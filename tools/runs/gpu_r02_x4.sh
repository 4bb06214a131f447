# source-level profile of the bucket kernel in SpGEMM's pre-bucketed mode (cfg 5)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:persist_bucket --launch-skip 1 --launch-count 1 -o gpurun_out/x4_spgemm -f python tools/op_runner.py spgemm 2 > gpurun_out/x4_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/x4_ncu.log
