// FP32 pipe throughput for mixes of packed FFMA2 (row-pair point stage) and
// scalar FFMA/FADD (level recursion), as lane-ops per SM per clock
// (FFMA2 = 2 lane-ops). Independent accumulator chains, 8/16 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, float b, u64 c) {
  u64 d, bb; asm("mov.b64 %0, {%1,%1};" : "=l"(bb) : "f"(b));
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(bb), "l"(c)); return d; }
__device__ __forceinline__ float ffma(float a, float b, float c) { float d; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }

template <int NP, int NS>  // per round: NP FFMA2, NS scalar FFMA, interleaved
__global__ void mix(float* out, int iters, long long* cyc) {
  u64 p[8]; float s[16];
  for (int i = 0; i < 8; ++i) p[i] = ((u64)__float_as_uint(1.f + threadIdx.x) << 32) | __float_as_uint(2.f + i);
  for (int i = 0; i < 16; ++i) s[i] = threadIdx.x * 1e-3f + i;
  float y = out[0], z = out[1];
  u64 xp = ((u64)__float_as_uint(y) << 32) | __float_as_uint(z);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int k = 0; k < (NP > NS ? NP : NS); ++k) {
        if (k < NP) p[k & 7] = ffma2(xp, s[(k + r) & 15], p[k & 7]);
        if (k < NS) s[k & 15] = ffma(y, s[(k + 5) & 15], s[k & 15]);
      }
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
  for (int i = 0; i < 8; ++i) acc += __uint_as_float((unsigned)p[i]) + __uint_as_float((unsigned)(p[i] >> 32));
  for (int i = 0; i < 16; ++i) acc += s[i];
  if (acc == 1234.5f) out[2] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NP, int NS>
void run(int warps) {
  float* out; long long* cyc;
  cudaMalloc(&out, 64); cudaMemset(out, 0, 64); cudaMalloc(&cyc, 148 * 8);
  const int iters = 2048;
  mix<NP, NS><<<148, warps * 32>>>(out, iters, cyc); cudaDeviceSynchronize();
  mix<NP, NS><<<148, warps * 32>>>(out, iters, cyc); cudaDeviceSynchronize();
  long long c[148]; cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double lane_ops = (double)iters * 16 * (2 * NP + NS) * warps * 32;
  const double instr = (double)iters * 16 * (NP + NS) * warps;
  printf("FFMA2:FFMA = %d:%-2d warps/SM=%2d  lane-ops/SM/clk = %6.1f   warp-instr/SM/clk = %.2f\n",
         NP, NS, warps, lane_ops / c[0], instr / c[0]);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {8, 16}) {
    run<8, 0>(w); run<0, 16>(w); run<8, 2>(w); run<8, 4>(w); run<8, 8>(w); run<8, 16>(w); run<4, 16>(w);
  }
  return 0;
}
