timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"gram_kernel" -c 1 \
  -o /tmp/r2_c5_pair python tools/diag_fp64_pair.py c5 > /dev/null 2>&1
ncu -i /tmp/r2_c5_pair.ncu-rep --page source --csv --print-source sass > /tmp/r2_c5_pair.src.csv 2>/dev/null
python tools/ncu_summary.py /tmp/r2_c5_pair.ncu-rep > gpurun_out/r2_c5_pair.summary.txt 2>&1
python tools/ncu_stalls.py /tmp/r2_c5_pair.src.csv 40 >> gpurun_out/r2_c5_pair.summary.txt 2>&1
