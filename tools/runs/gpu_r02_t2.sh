# ncu of the tile trace kernel on cfg 4
timeout 600 ncu --set full --import-source on --clock-control none -k regex:trace_warp_tile --launch-skip 1 --launch-count 1 -o gpurun_out/t2_trace -f python tools/op_runner.py trace 3 > gpurun_out/t2_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/t2_ncu.log
