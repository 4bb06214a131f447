set -x
start=$(date +%s)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s3a_gputest.log 2>&1; echo "gputest rc=$? seconds=$(( $(date +%s) - start ))"
tail -3 gpurun_out/s3a_gputest.log
timeout 600 python bench.py > gpurun_out/s3a_bench.log 2> gpurun_out/s3a_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/s3a_bench.err
python tools/bench_summary.py gpurun_out/s3a_bench.log 2>&1 | head -40
