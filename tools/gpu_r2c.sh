set -x
mkdir -p gpurun_out
timeout 900 python tools/fuzz_dump.py 200 gpurun_out/fuzz_dump.npz 2>&1 | tail -5
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c3 --size 1024 --steps 3 --warmup 3 > gpurun_out/world2_c3.log 2>&1; tail -c 1500 gpurun_out/world2_c3.log
BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --config c1 --steps 3 --warmup 3 > gpurun_out/world2_c1.log 2>&1; tail -c 600 gpurun_out/world2_c1.log
