timeout 900 python -m pytest tests/test_largen_gpu.py -x -q 2>&1 | tail -3
timeout 300 python tools/ln_time.py transpose1e7 transpose5e7 2>&1 | tail -4
AS_NO_SLOT=1 timeout 300 python tools/ln_time.py transpose1e7 transpose5e7 2>&1 | tail -4
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/slot_1e7.csv python tools/ln_time.py transpose1e7 --reps 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/slot_1e7.csv 2>&1 | tail -12
