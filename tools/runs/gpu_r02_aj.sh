nproc
for cfg in "8 4" "16 4" "12 8" "8 8" "16 16" "4 4"; do
  set -- $cfg
  echo "== threads=$1 chunks=$2"
  AS_UPLOAD_THREADS=$1 AS_UPLOAD_CHUNKS=$2 timeout 300 python tools/e2e_timeline.py 2>&1 | grep -E "upload|api_step"
done
