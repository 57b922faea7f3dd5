# Round-end style refresh: smoke, GPU tests, bench lines for every config, c3 launch list.
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
bash tools/gpu_bench_all.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/c3_bench_launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu \
  > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/c3_bench_launches.csv > gpurun_out/c3_bench_launches.txt
head -6 gpurun_out/c3_bench_launches.txt
