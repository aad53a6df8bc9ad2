// K3: merge of two normalised attention partials over disjoint key sets —
// the reference's merge_partials (proj/src/attention.cpp:63-82) followed by
// finalize (:84-92), restated for (O, LSE) pairs:
//   m = max(lse_a, lse_b); w_x = exp(lse_x - m) (0 for -inf)
//   O = (w_a O_a + w_b O_b) / (w_a + w_b);  lse = m + log(w_a + w_b)
// Rows where both inputs are empty (-inf) stay 0 / -inf (:72-74).
// HBM-bound elementwise kernel: one warp per (row, head), 16-B accesses.
#include <math.h>

#include "errors.hpp"
#include "slimpipe.h"
#include "sm100.cuh"

namespace sp {
namespace {

template <int D>
// oa/la may alias oo/lo (in-place merge, runtime.cpp): no __restrict__ on
// them; each element is read before it is written by the same thread.
__global__ void __launch_bounds__(256) attn_merge_kernel(const __nv_bfloat16* oa, const float* la,
                                                          const __nv_bfloat16* __restrict__ ob,
                                                          const float* __restrict__ lb, int64_t rows, int heads,
                                                          int64_t stride, __nv_bfloat16* oo, float* lo) {
  const int64_t item = int64_t(blockIdx.x) * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (item >= rows * heads) return;
  const int64_t row = item / heads;
  const int h = int(item % heads);
  const float xa = la[int64_t(h) * rows + row], xb = lb[int64_t(h) * rows + row];
  const float m = fmaxf(xa, xb);
  constexpr int kPer = D / 32;  // elements per lane (2 or 4)
  const int64_t base = row * stride + int64_t(h) * D + lane * kPer;
  float wa = 0.f, wb = 0.f;
  if (m != -INFINITY) {
    wa = xa == -INFINITY ? 0.f : __expf(xa - m);
    wb = xb == -INFINITY ? 0.f : __expf(xb - m);
  }
  const float sum = wa + wb;
  const float ca = sum > 0.f ? wa / sum : 0.f, cb = sum > 0.f ? wb / sum : 0.f;
  float out[kPer];
#pragma unroll
  for (int x = 0; x < kPer; ++x)
    out[x] = ca * __bfloat162float(oa[base + x]) + cb * __bfloat162float(ob[base + x]);
#pragma unroll
  for (int x = 0; x < kPer; ++x) oo[base + x] = __float2bfloat16(out[x]);
  if (lane == 0) lo[int64_t(h) * rows + row] = sum > 0.f ? m + __logf(sum) : -INFINITY;
}

}  // namespace
}  // namespace sp

namespace sp {
// Force-load this file's kernels (cudaFuncGetAttributes) — see preload_kernels
int preload_attn_merge() {
  cudaFuncAttributes a;
  if (cudaError_t e = cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(sp::attn_merge_kernel<64>))) return cuda_status(e, "preload sp::attn_merge_kernel<64>");
  if (cudaError_t e = cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(sp::attn_merge_kernel<128>))) return cuda_status(e, "preload sp::attn_merge_kernel<128>");
  return SP_OK;
}
}  // namespace sp

extern "C" int sp_attn_merge(const void* o_a, const float* lse_a, const void* o_b, const float* lse_b, int64_t rows,
                             int heads, int head_dim, int64_t o_stride, void* o_out, float* lse_out,
                             sp_stream_t stream) {
  using namespace sp;
  if (head_dim != 64 && head_dim != 128)
    return set_error(SP_ERR_UNSUPPORTED, "sp_attn_merge: head_dim %d not in {64,128}", head_dim);
  if (rows <= 0 || heads <= 0) return SP_OK;
  const int64_t items = rows * heads;
  const dim3 grid(unsigned((items + 7) / 8));
  auto* A = static_cast<const __nv_bfloat16*>(o_a);
  auto* B = static_cast<const __nv_bfloat16*>(o_b);
  auto* O = static_cast<__nv_bfloat16*>(o_out);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (head_dim == 128)
    attn_merge_kernel<128><<<grid, 256, 0, st>>>(A, lse_a, B, lse_b, rows, heads, o_stride, O, lse_out);
  else
    attn_merge_kernel<64><<<grid, 256, 0, st>>>(A, lse_a, B, lse_b, rows, heads, o_stride, O, lse_out);
  count_launch(1);
  return cuda_status(cudaGetLastError(), "sp_attn_merge launch");
}
