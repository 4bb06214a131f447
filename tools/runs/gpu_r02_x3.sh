# compute-sanitizer memcheck over the kernels added this session
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_trace_tile_gpu.py tests/test_mg_capi_gpu.py -x -q -k "not every_lane_count or (every_lane_count and (100 or 300 or 3-))" > gpurun_out/x3_memcheck.log 2>&1; echo "memcheck rc=$?"
grep -E "ERROR SUMMARY|passed|failed|Invalid|out of bounds" gpurun_out/x3_memcheck.log | head -10
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_trace_tile_gpu.py -x -q -k "tile_boundaries or long_and_oversized" > gpurun_out/x3_racecheck.log 2>&1; echo "racecheck rc=$?"
grep -E "RACECHECK SUMMARY|passed|failed|hazard" gpurun_out/x3_racecheck.log | head -10
