timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"gram_kernel" -c 1 \
  -o /tmp/r2_c5_pair python tools/diag_fp64_pair.py c5 > /dev/null 2>&1
ncu -i /tmp/r2_c5_pair.ncu-rep --page source --csv --print-source cuda,sass > /tmp/r2_c5_pair.cs.csv 2>gpurun_out/cs.err
ls -la /tmp/r2_c5_pair.cs.csv
gzip -c /tmp/r2_c5_pair.cs.csv > gpurun_out/r2_c5_pair.cs.csv.gz
ls -la gpurun_out/
