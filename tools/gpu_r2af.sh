set -x
mkdir -p gpurun_out
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"cert_redo_kernel" -c 1 \
  -o /tmp/r2_c4_redo python tools/devtime.py c4 512 fp32 1 > gpurun_out/r2_c4_redo.log 2>&1
ncu -i /tmp/r2_c4_redo.ncu-rep --page source --csv --print-source cuda,sass > /tmp/r2_c4_redo.src.csv 2>/dev/null
python tools/ncu_summary.py /tmp/r2_c4_redo.ncu-rep > gpurun_out/r2_c4_redo.summary.txt 2>&1
python tools/ncu_lines.py /tmp/r2_c4_redo.src.csv 40 >> gpurun_out/r2_c4_redo.summary.txt 2>&1
tail -3 gpurun_out/r2_c4_redo.log
