set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp32_pipes tools/microbench/fp32_pipes.cu && /tmp/fp32_pipes > gpurun_out/fp32_pipes.txt 2>&1; cat gpurun_out/fp32_pipes.txt
bash tools/gpu_ncu.sh r2_c3_gram c3 1024 fp32 1
head -40 gpurun_out/r2_c3_gram.summary.txt
