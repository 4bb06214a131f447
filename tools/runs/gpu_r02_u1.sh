# whole GPU suite on the restored tree + both bench arms
start=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/u1_test.log 2>&1; echo "test rc=$? seconds=$(( $(date +%s) - start ))"; tail -3 gpurun_out/u1_test.log
bash tools/runs/gpu_r02_final2.sh 2>&1 | grep -v "^+"
