# Launch list of the bench command (c3) and DRAM traffic of the full-size fused Gram launch.
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/c3_bench_launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu \
  > gpurun_out/c3_bench_under_ncu.log 2>&1
python tools/ncu_launches.py gpurun_out/c3_bench_launches.csv > gpurun_out/c3_bench_launches.txt
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:gram_kernel -s 2 -c 1 --csv --log-file gpurun_out/c3_full_traffic.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu > /dev/null 2>&1
cat gpurun_out/c3_bench_launches.txt; grep -E "dram|duration" gpurun_out/c3_full_traffic.csv | cut -c1-250
