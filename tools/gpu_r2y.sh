set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gram_kernel" -s 0 -c 1 -o gpurun_out/r2_rowscan_c4 python tools/diag_fp64_pair.py c4 > gpurun_out/r2_rowscan_c4.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_rowscan_c4.ncu-rep > gpurun_out/r2_rowscan_c4.summary.txt 2>&1
ncu -i gpurun_out/r2_rowscan_c4.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_rowscan_c4.src.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/r2_rowscan_c4.src.csv 40 >> gpurun_out/r2_rowscan_c4.summary.txt 2>&1
head -80 gpurun_out/r2_rowscan_c4.summary.txt
timeout 300 python tools/diag_fp64_pair.py c4 2>&1 | tail -3
