timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ln_transpose_finish|ln_scatter" --launch-skip 2 -c 3 -o gpurun_out/r02_ln_full3 -f python tools/ln_time.py transpose1e7 --reps 1 > gpurun_out/r02_ln_full3.log 2>&1
echo ncu rc=$?
