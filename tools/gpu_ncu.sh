# ncu --set full capture of ONE Gram-kernel launch + source-page CSV
# usage: SKIP=<launches to skip> bash tools/gpu_ncu.sh <tag> <devtime args...>
# devtime.py launches, per rep: self levels of X and Y (normalised configs
# only, 2 gram_kernel launches), then the Gram. SKIP defaults to 2 for
# normalised configs (c1, c3) so the capture is the Gram, not sk_self_levels.
tag=$1; shift
case "$1" in c1|c3) def=2 ;; *) def=0 ;; esac
skip=${SKIP:-$def}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_kernel|gemm_dp_kernel" -s $skip -c 1 \
  -o gpurun_out/$tag python tools/devtime.py "$@" > gpurun_out/$tag.log 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/$tag.src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/$tag.ncu-rep > gpurun_out/$tag.summary.txt 2>&1
python tools/ncu_stalls.py gpurun_out/$tag.src.csv 30 >> gpurun_out/$tag.summary.txt 2>&1
tail -5 gpurun_out/$tag.log
