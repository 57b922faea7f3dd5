timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"pde_warp" -c 1 \
  -o /tmp/r2_pde python tools/pde_once.py > /dev/null 2>&1
ncu -i /tmp/r2_pde.ncu-rep --page source --csv --print-source cuda,sass > /tmp/r2_pde.cs.csv 2>/dev/null
python tools/ncu_summary.py /tmp/r2_pde.ncu-rep > gpurun_out/r2_pde.summary.txt 2>&1
python tools/ncu_lines.py /tmp/r2_pde.cs.csv 30 >> gpurun_out/r2_pde.summary.txt 2>&1
