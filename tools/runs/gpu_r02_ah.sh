timeout 900 python -m pytest tests/test_largen_gpu.py tests/test_kernels_gpu.py -x -q 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin.csv python tools/ln_time.py transpose1e7 transpose5e7 --reps 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/fin.csv | grep finish
timeout 600 python tools/ln_time.py transpose1e7 transpose5e7 --reps 5
