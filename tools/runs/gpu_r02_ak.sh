for cfg in "8 1" "8 2" "16 1" "16 2" "8 4"; do
  set -- $cfg
  echo "== threads=$1 chunks=$2"
  AS_UPLOAD_THREADS=$1 AS_UPLOAD_CHUNKS=$2 timeout 300 python tools/e2e_timeline.py 2>&1 | grep -E "upload|api_step"
done
