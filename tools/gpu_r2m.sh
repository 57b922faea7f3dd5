set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python tools/diag_fp64_pair.py c4 2>&1 | tail -3
timeout 300 python tools/devtime.py c4 2048 fp32 2 2>&1 | tail -1
timeout 300 python tools/devtime.py c4 2048 fp32 2 nofix 2>&1 | tail -1
for c in c3 c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err
  echo "$c rc=$?"; tail -c 600 gpurun_out/r2_bench_$c.json
done
