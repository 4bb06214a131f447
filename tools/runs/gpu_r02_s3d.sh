timeout 600 ncu --set full --import-source on --clock-control none -k regex:spmm_csc_merge -c 1 -o gpurun_out/s3d_merge -f python tools/op_runner.py spmm_first 1 > gpurun_out/s3d_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/s3d_merge.ncu-rep --page details > gpurun_out/s3d_merge_details.txt 2>&1
ncu -i gpurun_out/s3d_merge.ncu-rep --page source --csv > gpurun_out/s3d_merge_source.csv 2>&1
grep -E "Duration|Issue Slots|Eligible|Occupancy|Throughput|Stall|Registers|L2 Hit" gpurun_out/s3d_merge_details.txt | head -40
