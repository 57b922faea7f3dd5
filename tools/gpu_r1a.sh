set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -3 gpurun_out/bench_c3.err
cat gpurun_out/bench_c3.json
timeout 200 python tools/devtime.py c5 64 2>&1 | tail -3
timeout 200 python tools/devtime.py c5 128 2>&1 | tail -2
timeout 200 python tools/devtime.py c2 128 2>&1 | tail -2
timeout 200 python tools/devtime.py c4 128 2>&1 | tail -2
timeout 200 python tools/devtime.py c1 64 2>&1 | tail -2
