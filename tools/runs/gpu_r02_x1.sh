for v in "" "AS_SR_CTAS=1" "AS_SR_FILL=0.6" "AS_SR_FILL=0.95" "AS_SR_WAVE=0"; do echo "[$v]"; env $v timeout 300 python tools/time_ops.py flush build transpose 30; done
