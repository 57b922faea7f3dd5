set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gram_kernel" -s 0 -c 1 -o gpurun_out/r2_rowscan python tools/diag_fp64_pair.py c3 > gpurun_out/r2_rowscan.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_rowscan.ncu-rep > gpurun_out/r2_rowscan.summary.txt 2>&1
ncu -i gpurun_out/r2_rowscan.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_rowscan.src.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/r2_rowscan.src.csv 30 >> gpurun_out/r2_rowscan.summary.txt 2>&1
head -60 gpurun_out/r2_rowscan.summary.txt
cuobjdump -res-usage paper_2501_07145_b200/_lib/libsigkern_b200.so 2>/dev/null | grep -A1 "gram_kernelINS0_10LaneState1INS0_10PointStageILi4ELi8ELi0EEELi8EEELb1EE" | head -4
