# ncu --set full capture of the fused Gram kernel (one launch) + source-page CSV
# usage: bash tools/gpu_ncu.sh <tag> <devtime args...>
tag=$1; shift
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_kernel|gemm_dp_kernel" -s 1 -c 1 \
  -o gpurun_out/$tag python tools/devtime.py "$@" > gpurun_out/$tag.log 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/$tag.src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/$tag.ncu-rep > gpurun_out/$tag.summary.txt 2>&1
python tools/ncu_stalls.py gpurun_out/$tag.src.csv 30 >> gpurun_out/$tag.summary.txt 2>&1
tail -5 gpurun_out/$tag.log
