#!/bin/bash
# One `ncu --set full` capture per hot-path op, restricted by NVTX to exactly
# one call of the op (tools/op_runner.py wraps each call in "op_<name>"), so
# the raw page lists every launch of that call and tools/make_traffic.py can
# sum DRAM bytes over the whole op.  Usage: tools/ncu_ops.sh TAG [ops...]
set -u
TAG=$1; shift
OPS=${@:-build transpose flush spmm spmm_first trace add spgemm build_1e7 transpose_1e7_f32}
mkdir -p gpurun_out
for op in $OPS; do
  timeout 900 ncu --nvtx --nvtx-include "op_${op}/" --set full --clock-control none --import-source on \
    -o gpurun_out/${TAG}_ncu_${op} -f python tools/op_runner.py $op 1 > gpurun_out/${TAG}_ncu_${op}.log 2>&1
  echo "$op rc=$?"
  ncu -i gpurun_out/${TAG}_ncu_${op}.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_${op}.csv 2>/dev/null
  # the report itself only for the ops named in KEEP_REP (gpurun copies back <= 64 MiB)
  case " ${KEEP_REP:-} " in *" $op "*) ;; *) rm -f gpurun_out/${TAG}_ncu_${op}.ncu-rep ;; esac
done
