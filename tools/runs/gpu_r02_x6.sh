# single-launch kernel on small inputs: one CTA per SM below AS_SR_SMALL_N elements
for v in "AS_SR_SMALL_N=0" "AS_SR_SMALL_N=300000" "AS_SR_SMALL_N=0" "AS_SR_SMALL_N=300000"; do echo "[$v] $(env $v timeout 300 python tools/time_ops.py flush 40)"; done
for v in "AS_SR_SMALL_N=0" "AS_SR_SMALL_N=300000"; do
  env $v ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x6.csv python tools/op_runner.py flush 6 > /dev/null 2>&1
  echo "[$v]"; grep sortreduce gpurun_out/x6.csv | awk -F'","' '{print $NF}' | tr -d '"' | head -6 | tr '\n' ' '; echo
done
