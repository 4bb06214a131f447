set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_t11.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02_t11.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
for v in base kc8 kb16 kb4; do
  if [ $v = base ]; then L=""; else L="AS_LIB_PATH=paper_1805_03380_b200/build/variants/$v.so"; fi
  echo "== $v"; env $L timeout 300 python tools/time_ops.py spmm 10
done
