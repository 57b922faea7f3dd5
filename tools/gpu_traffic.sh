# DRAM bytes (read + write) and duration of the full-size c3 / c5 / c2 Gram launch -> gpurun_out/r2_<cfg>_traffic.csv (profiles/traffic.json)
set -x
mkdir -p gpurun_out
for c in c3 c5 c2; do
  case $c in c3) s=2 ;; *) s=0 ;; esac
  n=$( [ $c = c3 ] && echo 8192 || ([ $c = c5 ] && echo 512 || echo 1024) )
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gram_kernel -s $s -c 1 --csv \
    python tools/devtime.py $c $n fp32 1 > gpurun_out/r2_${c}_traffic.csv 2> gpurun_out/r2_${c}_traffic.err
  tail -5 gpurun_out/r2_${c}_traffic.csv
done
