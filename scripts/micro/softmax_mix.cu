// Microbenchmark: the K1 softmax inner loop (FFMA2 -> 2x ex2 -> FADD2 -> F2FP)
// from registers, 8 warps per SM (2 per sub-partition), 64 elements per
// thread per "tile": cycles per tile vs the MUFU floor (16384 ex2 / 16 per clk
// = 1024 cycles).
#include <cstdio>
#include <cstdint>
#include "../../paper_2504_14519_b200/csrc/cuda/sm100.cuh"
using namespace sp;
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(float* out, long long* cyc, int tiles) {
  float sv[64];
  for (int i = 0; i < 64; ++i) sv[i] = (threadIdx.x * 64 + i) * 1e-5f - 0.3f;
  const float sl2 = 0.1275f, msub = 0.5f;
  uint32_t acc = 0;
  float l = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int t = 0; t < tiles; ++t) {
    float2 rs[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    const float2 a2 = make_float2(sl2, sl2), n2 = make_float2(-msub - t * 1e-9f, -msub - t * 1e-9f);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        float a, b;
        if (MODE == 0) {
          const float2 xx = ffma2(make_float2(sv[c * 32 + 2 * e], sv[c * 32 + 2 * e + 1]), a2, n2);
          a = fast_exp2(xx.x);
          b = fast_exp2(xx.y);
          rs[e & 3] = fadd2(rs[e & 3], make_float2(a, b));
        } else {
          a = fast_exp2(fmaf(sv[c * 32 + 2 * e], sl2, n2.x));
          b = fast_exp2(fmaf(sv[c * 32 + 2 * e + 1], sl2, n2.x));
          rs[e & 3].x += a;
          rs[e & 3].y += b;
        }
        pk[e] = pack_bf16(a, b);
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) acc ^= pk[e];
    }
    l += rs[0].x + rs[1].x + rs[2].x + rs[3].x + rs[0].y + rs[1].y + rs[2].y + rs[3].y;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 256 * 4); cudaMalloc(&cyc, 148 * 8);
  const int tiles = 1000;
  for (int mode = 0; mode < 2; ++mode) {
    for (int r = 0; r < 2; ++r) {
      if (mode == 0) k<0><<<148, 256>>>(out, cyc, tiles); else k<1><<<148, 256>>>(out, cyc, tiles);
      cudaDeviceSynchronize();
    }
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %.0f cycles per 128x128 tile (MUFU floor 1024)\n", mode, mode ? "scalar" : "fp32x2", double(c) / tiles);
  }
}
