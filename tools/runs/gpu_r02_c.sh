set -x
AS_LIB_PATH=paper_1805_03380_b200/build/variants/srdbg.so AS_PHASE_TIMES=1 timeout 300 python tools/sr_time.py build transpose flush 3 > gpurun_out/r02_srphases.log 2>&1
tail -40 gpurun_out/r02_srphases.log
timeout 600 python tools/ln_time.py --reps 5 > gpurun_out/r02_ln_base.log 2>&1
cat gpurun_out/r02_ln_base.log
