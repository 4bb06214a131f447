timeout 600 ncu --set full --import-source on --clock-control none -k regex:trace_partial -c 1 -o gpurun_out/r02c_trace -f python tools/op_runner.py trace 1 > /dev/null 2>&1; echo rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:add_tile -c 1 -o gpurun_out/r02c_add -f python tools/op_runner.py add 1 > /dev/null 2>&1; echo rc=$?
