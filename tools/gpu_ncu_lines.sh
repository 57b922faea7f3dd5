# ncu --set full of one launch + warp-stall samples per CUDA source line.
# usage: bash tools/gpu_ncu_lines.sh <tag> <kernel regex> <python args...>
# e.g.   bash tools/gpu_ncu_lines.sh c4_redo cert_redo_kernel tools/devtime.py c4 512 fp32 1
#        bash tools/gpu_ncu_lines.sh c5_pair gram_kernel tools/diag_fp64_pair.py c5
#        bash tools/gpu_ncu_lines.sh pde pde_warp tools/pde_once.py
# The report stays in /tmp (too large for gpurun_out); the summary and the
# per-line table land in gpurun_out/<tag>.summary.txt.
tag=$1; kre=$2; shift 2
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$kre" -c 1 \
  -o /tmp/$tag python "$@" > gpurun_out/$tag.log 2>&1
ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source cuda,sass > /tmp/$tag.src.csv 2>/dev/null
python tools/ncu_summary.py /tmp/$tag.ncu-rep > gpurun_out/$tag.summary.txt 2>&1
python tools/ncu_lines.py /tmp/$tag.src.csv 40 >> gpurun_out/$tag.summary.txt 2>&1
tail -3 gpurun_out/$tag.log
