set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gram_kernel" -s 0 -c 1 -o gpurun_out/r2_rowscan_c5 python tools/diag_fp64_pair.py c5 > gpurun_out/r2_rowscan_c5.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_rowscan_c5.ncu-rep > gpurun_out/r2_rowscan_c5.summary.txt 2>&1
ncu -i gpurun_out/r2_rowscan_c5.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_rowscan_c5.src.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/r2_rowscan_c5.src.csv 40 >> gpurun_out/r2_rowscan_c5.summary.txt 2>&1
python tools/ncu_byop.py gpurun_out/r2_rowscan_c5.src.csv 16 >> gpurun_out/r2_rowscan_c5.summary.txt 2>&1
cat gpurun_out/r2_rowscan_c5.summary.txt | head -100
bash tools/gpu_bench_world2.sh
