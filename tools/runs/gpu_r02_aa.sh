set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_t14.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r02_t14.log
for v in new old new old; do
  if [ $v = new ]; then L=""; else L="AS_LIB_PATH=paper_1805_03380_b200/build/variants/old_lb.so"; fi
  env $L timeout 600 python bench.py --ops add,spgemm,large --no-cpu --steps 5 --warmup 3 --skip-slow-checks > gpurun_out/sc_$v.log 2>&1
  python - $v <<'PY'
import json, sys
l=json.loads(open("gpurun_out/sc_%s.log" % sys.argv[1]).read().strip().splitlines()[-1])
o=l["ops"]
print(sys.argv[1], "build %.1f" % (l["ms_per_step"]*1e3), "add %.1f" % (o["add_cfg5"]["ms"]*1e3), "spgemm %.1f" % (o["spgemm_cfg5"]["ms"]*1e3),
      " ".join("%s %.1f" % (k, v["ms"]*1e3) for k, v in o["large_n"].items()))
PY
done
