// FP64 pipe microbenchmark: DFMA / DADD throughput per SM per clock.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void bench(double *out, int iters, long long *cyc) {
  double a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001 + i;
  const double x = out[0], y = out[1];
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = MODE == 0 ? fma(x, a[i], y) : a[i] + x;
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.0) out[2] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double *out; long long *cyc;
  cudaMalloc(&out, 64); cudaMemset(out, 0, 64); cudaMalloc(&cyc, 4096 * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 2; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      const int iters = 4096;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (mode == 0) bench<0><<<sms, warps * 32>>>(out, iters, cyc); else bench<1><<<sms, warps * 32>>>(out, iters, cyc);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double ops = (double)warps * 32 * iters * 16;
      printf("%s warps/SM=%2d  lane-ops/clk/SM=%7.2f\n", mode == 0 ? "DFMA" : "DADD", warps, ops / c);
    }
  return 0;
}
