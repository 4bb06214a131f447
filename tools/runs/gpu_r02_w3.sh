timeout 300 python tools/cfg2_csc_phases.py
timeout 900 python -m pytest tests -m gpu -x -q -k "api or dropin or ref_kernels or configs or funnel or mmio" > gpurun_out/w3_test.log 2>&1; echo "test rc=$?"; tail -3 gpurun_out/w3_test.log
