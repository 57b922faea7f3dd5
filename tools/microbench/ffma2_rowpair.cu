// FFMA2 throughput in the row-pair form used by the Gram kernel's point stage:
//   acc{r, r+1}[c] = fma(x{r, r+1}[k] (reused pair), y[c][k] (scalar broadcast), acc[c])
// compared with plain FFMA, and mixed with the scalar FADD/FFMA recursion and MUFU.EX2.
// Prints lane-FMA ops per SM per clock (FFMA2 = 2 lane ops).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 bc(float y) { u64 d; asm("mov.b64 %0, {%1,%1};" : "=l"(d) : "f"(y)); return d; }
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int MODE>
__global__ void bench(float* out, int iters, long long* cyc) {
  float y[16];
  for (int i = 0; i < 16; ++i) y[i] = out[i + 2] + threadIdx.x * 1e-3f;
  u64 acc[8];
  float s[8];
  for (int i = 0; i < 8; ++i) { acc[i] = 0; s[i] = 0.f; }
  float xa = out[0], xb = out[1];
  u64 xp; asm("mov.b64 %0, {%1,%2};" : "=l"(xp) : "f"(xa), "f"(xb));
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (MODE == 0) {  // 8 FFMA2 row-pair form
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = ffma2(xp, bc(y[(c + k) & 15]), acc[c]);
      } else if (MODE == 1) {  // 16 scalar FFMA, same data
#pragma unroll
        for (int c = 0; c < 8; ++c) { s[c] = fmaf(xa, y[(c + k) & 15], s[c]); y[(c+k)&15] = fmaf(xb, y[(c + k) & 15], s[c]); }
      } else if (MODE == 2) {  // 8 FFMA2 + 4 FADD + 4 FFMA (recursion-like) + 1 MUFU
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = ffma2(xp, bc(y[(c + k) & 15]), acc[c]);
#pragma unroll
        for (int c = 0; c < 4; ++c) { s[c] = s[c] + s[c + 4]; s[c + 4] = fmaf(s[c], xa, s[c + 4]); }
        s[k & 7] = ex2(s[k & 7]);
      }
    }
    if (MODE != 1) { xp ^= 1ull; }
  }
  long long t1 = clock64();
  float r = 0.f;
  for (int i = 0; i < 8; ++i) r += __uint_as_float((unsigned)acc[i]) + __uint_as_float((unsigned)(acc[i] >> 32)) + s[i];
  for (int i = 0; i < 16; ++i) r += y[i];
  if (r == 1234.5f) out[0] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, double lane_ops_per_iter, int warps) {
  float* out; long long* cyc;
  cudaMalloc(&out, 64 * 4); cudaMemset(out, 0, 64 * 4);
  cudaMalloc(&cyc, 148 * 8);
  int iters = 4096;
  bench<MODE><<<148, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  bench<MODE><<<148, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long c[148]; cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double ops = lane_ops_per_iter * iters * warps * 32;
  printf("%-40s warps/SM=%2d  lane-FMA-ops/SM/clk = %.1f\n", name, warps, ops / c[0]);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {8, 16}) {
    run<0>("FFMA2 rowpair x128 (=256 lane ops)", 16 * 8 * 2, w);
    run<1>("FFMA x256", 16 * 16, w);
    run<2>("FFMA2 x128 + 64 FADD/64 FFMA + 16 MUFU", 16 * (16 + 8), w);
  }
  return 0;
}
