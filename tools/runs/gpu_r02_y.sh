set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_t13.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02_t13.log
timeout 300 python tools/time_ops.py add spgemm 10
timeout 600 python tools/ln_time.py build1e7 transpose1e7 --reps 5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_sg_launches.csv python tools/op_runner.py spgemm 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/r02_sg_launches.csv 2>/dev/null | tail -14
