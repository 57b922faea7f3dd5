# ncu launch list (device time per kernel launch) of one devtime run
# usage: bash tools/gpu_launches.sh <tag> <devtime args...>
tag=$1; shift
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/$tag.launches.csv python tools/devtime.py "$@" > gpurun_out/$tag.log 2>&1
python tools/ncu_launches.py gpurun_out/$tag.launches.csv > gpurun_out/$tag.launches.txt 2>&1
tail -30 gpurun_out/$tag.launches.txt
