# large-input pipeline: the bucket id's bits split evenly between the two passes (default) vs the fixed 8-bit low digit
for v in "AS_LN_LOB=8" "AS_LN_LOB=0" "AS_LN_LOB=6"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --ops large --no-cpu > gpurun_out/x8_bench.log 2>&1
  echo "[$v] $(python -c "
import json
l=json.loads(open('gpurun_out/x8_bench.log').read().strip().splitlines()[-1])
print({k: round(v['ms'],4) for k,v in l['ops']['large_n'].items()})")"
done
