set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_t15.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r02_t15.log
for v in new old new old; do
  if [ $v = new ]; then L=""; else L="AS_LIB_PATH=paper_1805_03380_b200/build/variants/old_lb.so"; fi
  env $L timeout 600 python bench.py --ops spgemm --no-cpu --steps 5 --warmup 3 --skip-slow-checks > gpurun_out/sg_$v.log 2>&1
  python - $v <<'PY'
import json, sys
l=json.loads(open("gpurun_out/sg_%s.log" % sys.argv[1]).read().strip().splitlines()[-1])
o=l["ops"]
print(sys.argv[1], "spgemm %.1f api %.1f" % (o["spgemm_cfg5"]["ms"]*1e3, o["spgemm_cfg5"]["api_ms"]*1e3))
PY
done
