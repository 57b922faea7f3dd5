set -x
mkdir -p gpurun_out
for c in c3 c1 c2 c4 c5; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err
  echo "$c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c3_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r2_c3_bench_launches.log 2>&1
python tools/ncu_launches.py gpurun_out/r2_c3_bench_launches.csv > gpurun_out/r2_c3_bench_launches.txt 2>&1; head -20 gpurun_out/r2_c3_bench_launches.txt
