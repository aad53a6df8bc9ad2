// How far can one thread run ahead of the tensor pipe?  Issue G dispatches
// (M=128,N=128,K=16 SS, 64 cyc each) to an idle pipe, time the issue loop
// and the completion (commit + wait).
#include <cstdio>
#include <cstdint>
#include "../../paper_2504_14519_b200/csrc/cuda/sm100.cuh"
using namespace sp;
__global__ void __launch_bounds__(128, 1) k(long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc_bf16_f32(128, 128, false, false);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    int ph = 0;
    for (int g = 1; g <= 32; g *= 2) {
      long long t0 = clock64();
      for (int kk = 0; kk < g; ++kk) {
        const uint32_t o = ((kk & 7) / 4) * 16384 + (kk % 4) * 32;
        umma_bf16_ss(tm, smem_desc_sw128(a + o, 16, 1024), smem_desc_sw128(b + o, 16, 1024), id, kk ? 1u : 0u);
      }
      long long t1 = clock64();
      umma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
      long long t2 = clock64();
      if (blockIdx.x == 0) { out[2 * g] = t1 - t0; out[2 * g + 1] = t2 - t0; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tm); }
}
int main() {
  long long* o; cudaMalloc(&o, 8 * 128);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int i = 0; i < 2; ++i) k<<<148, 128, 80 * 1024>>>(o);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  long long h[128]; cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
  for (int g = 1; g <= 32; g *= 2) printf("G=%2d dispatches: issue loop %5lld cyc, complete %5lld cyc\n", g, h[2 * g], h[2 * g + 1]);
}
