# tile trace kernel: tests, then cfg 4 timing of both kernels
timeout 900 python -m pytest tests -m gpu -x -q -k "trace" > gpurun_out/t1_test.log 2>&1; echo "test rc=$?"; tail -5 gpurun_out/t1_test.log
for v in "AS_TRACE_ENGINE=0" "AS_TRACE_ENGINE=1"; do echo "[$v]"; env $v timeout 300 python tools/time_ops.py trace 20; done
