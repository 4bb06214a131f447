timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ln_scatter|ln_transpose_finish|ln_count" -c 4 -o gpurun_out/r02_ln_full -f python tools/ln_time.py transpose1e7 --reps 1 > gpurun_out/r02_ln_full.log 2>&1
echo rc=$?
