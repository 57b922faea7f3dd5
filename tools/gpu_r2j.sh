set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python tools/devtime.py c4 4096 fp32 2 nofix 2>&1 | tail -1
timeout 300 python tools/devtime.py c4 4096 fp32 2 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.err; tail -c 2500 gpurun_out/r2_bench_c3.json
