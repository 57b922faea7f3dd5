# Multi-rank bench logic on ONE GPU: torchrun world 2 with gloo collectives
# (both ranks share cuda:0; the all-gather goes through host copies), both
# arms. Exercises the strong-scaling step (sharded_gram) end to end; not a
# scaling measurement.
export BENCH_DIST_BACKEND=gloo
for cfg in "c3 --size 1024" "c1"; do
  for impl in ours reference; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29533 bench.py --gpus 2 --config $cfg --steps 3 --warmup 3 --impl $impl \
      > gpurun_out/world2_${impl}.log 2>&1
    echo "$cfg $impl rc=$?"; grep -c '"metric"' gpurun_out/world2_${impl}.log; tail -1 gpurun_out/world2_${impl}.log | cut -c1-600
  done
done
