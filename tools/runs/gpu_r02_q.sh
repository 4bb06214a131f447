for v in base unroll2 unroll4; do
  if [ $v = base ]; then L=""; else L="AS_LIB_PATH=paper_1805_03380_b200/build/variants/$v.so"; fi
  echo "== $v"; env $L timeout 300 python tools/sr_time.py build transpose flush 40
done
echo "== base again"; timeout 300 python tools/sr_time.py build transpose flush 40
