// Microbenchmark: per-SM throughput of ex2.approx, cvt.rn.bf16x2.f32 and a mix
// (used to size the attention softmax; results in DESIGN.md).
#include <cstdio>
#include <cuda_bf16.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned pk(float a, float b) { unsigned r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a)); return r; }
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) v[i] = ex2(v[i]) * -0.5f;
      if (MODE == 1) acc += pk(v[i], v[(i + 1) & 7]), v[i] += 1e-7f;
      if (MODE == 2) { v[i] = ex2(v[i]) * -0.5f; if (i & 1) acc += pk(v[i], v[i - 1]); }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  int iters = 4096;
  for (int mode = 0; mode < 3; ++mode)
    for (int threads : {128, 256, 512, 1024}) {
      long long c[148];
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<148, threads>>>(out, cyc, iters);
        if (mode == 1) k<1><<<148, threads>>>(out, cyc, iters);
        if (mode == 2) k<2><<<148, threads>>>(out, cyc, iters);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
      double ops = double(threads) * iters * (mode == 2 ? 8 : 8);
      printf("mode %d (%s) threads %4d: %.2f ops/clk/SM (%.0f cycles)\n", mode, mode == 0 ? "ex2" : mode == 1 ? "cvt.bf16x2" : "ex2+half cvt", threads, ops / c[0], double(c[0]));
    }
  return 0;
}
