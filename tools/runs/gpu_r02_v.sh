timeout 600 ncu --set full --import-source on --clock-control none -k regex:sortreduce -c 1 -o gpurun_out/r02c_build -f python tools/op_runner.py build 1 > /dev/null 2>&1; echo rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"ln_scatter" -c 2 -o gpurun_out/r02c_ln_build -f python tools/op_runner.py build_1e7 1 > /dev/null 2>&1; echo rc=$?
