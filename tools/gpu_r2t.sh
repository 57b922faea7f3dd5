nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_pipe tools/microbench/fp64_pipe.cu && /tmp/fp64_pipe > gpurun_out/fp64_pipe.txt 2>&1; cat gpurun_out/fp64_pipe.txt
for r in 1 2; do
for v in vC vE vF; do echo "$v $(SK_LIB_OVERRIDE=ab/$v.so timeout 300 python tools/devtime.py c5 512 fp32 2 nofix 2>&1 | tail -1)"; done
done
