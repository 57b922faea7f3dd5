# ncu --set full of one launch of a kernel matching a regex: bash tools/gpu_ncu_k.sh <tag> <regex> <devtime args>
tag=$1; rx=$2; shift 2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s 2 -c 1 \
  -o gpurun_out/$tag python tools/devtime.py "$@" > gpurun_out/$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/$tag.ncu-rep > gpurun_out/$tag.summary.txt 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/$tag.raw.csv 2>/dev/null
