# Multi-rank bench logic on ONE GPU: torchrun world 2, gloo for the barrier/max reduce
# (both ranks share cuda:0), both arms. Not a scaling measurement.
export BENCH_DIST_BACKEND=gloo
for impl in ours reference; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --config c1 --steps 3 --warmup 3 --impl $impl \
    > gpurun_out/world2_$impl.log 2>&1
  echo "$impl rc=$?"; grep -c '"metric"' gpurun_out/world2_$impl.log; tail -1 gpurun_out/world2_$impl.log | cut -c1-400
done
