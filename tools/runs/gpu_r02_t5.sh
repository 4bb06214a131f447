timeout 900 python -m pytest tests -m gpu -x -q -k "trace" > gpurun_out/t5_test.log 2>&1; echo "test rc=$?"; tail -3 gpurun_out/t5_test.log
for op in trace trace5; do timeout 300 python tools/time_ops.py $op 20; done
