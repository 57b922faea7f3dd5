set -x
timeout 300 python tools/devtime.py c4 4096 fp32 2 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cert_redo" -s 0 -c 1 -o gpurun_out/r2_redo_c4 python tools/devtime.py c4 512 fp32 1 > gpurun_out/r2_redo_c4.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_redo_c4.ncu-rep > gpurun_out/r2_redo_c4.summary.txt 2>&1
ncu -i gpurun_out/r2_redo_c4.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_redo_c4.src.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/r2_redo_c4.src.csv 40 >> gpurun_out/r2_redo_c4.summary.txt 2>&1
head -60 gpurun_out/r2_redo_c4.summary.txt
