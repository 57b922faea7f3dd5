# One bench line per BASELINE config (c3 is the headline default).
for c in c3 c1 c2 c4 c5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"; tail -2 gpurun_out/bench_$c.err | cut -c1-300
done
