# SpMM row split: chunk c + 1 transposed on a helper stream while chunk c is gathered (AS_SPMM_OVERLAP=1)
AS_SPMM_OVERLAP=1 timeout 900 python -m pytest tests -m gpu -x -q -k "spmm or cfg3 or mat_times or spmv or matvec" > gpurun_out/x5_test.log 2>&1; echo "test rc=$?"; tail -2 gpurun_out/x5_test.log
for rep in 1 2; do for v in "AS_SPMM_OVERLAP=0" "AS_SPMM_OVERLAP=1"; do echo "[$v] $(env $v timeout 300 python tools/time_ops.py spmm 20)"; done; done
