# large-input pipeline: mean bucket size as a fraction of the tile
for v in "AS_LN_FILL=0.85" "AS_LN_FILL=0.90" "AS_LN_FILL=0.93" "AS_LN_FILL=0.75"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --ops large --no-cpu > gpurun_out/x10_bench.log 2>&1
  echo "[$v] $(python -c "
import json
l=json.loads(open('gpurun_out/x10_bench.log').read().strip().splitlines()[-1])
print({k: round(v['ms'],4) for k,v in l['ops']['large_n'].items()})")"
done
