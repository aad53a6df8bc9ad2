// K2: sliced causal attention backward on sm_100a (tcgen05 + TMEM + TMA).
//
// NOT in the reference (it has a forward-only fp64 kernel,
// proj/src/attention.cpp:21-111); exact softmax-attention gradients, pinned
// against the C oracle (oracle/attention_oracle.c:orc_attn_bwd_head), which
// is itself pinned to the reference forward by finite differences.
//
// The step runs backward slices n..1 (reference schedule.cpp:125-126 edges),
// so every call ACCUMULATES dK/dV of the chunks it touches into fp32 chunk
// accumulators; chunk j's gradient is complete when slice j's backward runs.
//
// One CTA = one 128-key tile of one KV head; it loops over every (query head
// of the GQA group, query tile) that attends the tile.  Per pair:
//   S^T  = K Q^T          dP^T = V dO^T            (M=128 keys)
//   P^T  = exp2(S^T*sl2 - lse2[q]) ; dS^T = P^T (dP^T - delta[q]) * scale
//   dV  += P^T dO         dK  += dS^T Q            (TMEM accumulators)
//   dQ   = dS K  (D=64)  or  dQ^T = K^T dS^T (D=128) -> fp32 red.add to dq_acc
// Warp 0 TMA, warp 1 TMEM owner + UMMA issuer, warps 2..5 element math.
// Query tile BQ = 64 for D=128 (TMEM 64+64+64+128+128 cols), 128 for D=64.
#include <math.h>

#include "errors.hpp"
#include "slimpipe.h"
#include "kernels.hpp"
#include "sm100.cuh"

#include <cstdlib>

namespace sp {
namespace {

constexpr int kBK = 128;  // keys per CTA
constexpr int kThreads = 192;

struct BwdParams {
  int q_rows;
  int total_kv;
  int chunk_len;
  int group;
  int causal;
  int n_qtiles;
  float scale;
  float scale_log2;
  const float* lse2;   // [heads][q_rows] lse * log2(e)
  const float* delta;  // [heads][q_rows]
  float* dq;           // [q_rows][heads*D]
  int64_t dq_stride;
  void* dk;            // [acc_rows][kv_heads*D], fp32 or bf16 (AccT)
  void* dv;
  int64_t acc_stride;
  int chunk_row[SP_MAX_CHUNKS];
  int acc_row[SP_MAX_CHUNKS];
};

template <int D>
struct BwdCfg {
  static constexpr int BQ = D == 128 ? 64 : 128;
  static constexpr bool kDqT = D == 128;  // dQ computed transposed (M = D)
  static constexpr int NS = 2;
  // TMEM column map
  static constexpr int kS = 0, kDP = BQ, kDQ = 2 * BQ, kDV = kDQ + (kDqT ? BQ : D), kDK = kDV + D;
  static_assert(kDK + D <= 512, "TMEM budget");
};

template <int D>
struct alignas(1024) BwdSmem {
  static constexpr int BQ = BwdCfg<D>::BQ, NS = BwdCfg<D>::NS;
  __nv_bfloat16 k[kBK * D];
  __nv_bfloat16 v[kBK * D];
  __nv_bfloat16 q[NS][BQ * D];
  __nv_bfloat16 dout[NS][BQ * D];
  __nv_bfloat16 p[kBK * BQ];   // P^T  [keys][BQ] K-major slabs
  __nv_bfloat16 ds[kBK * BQ];  // dS^T [keys][BQ]
  float lse2[NS][BQ];
  float delta[NS][BQ];
  uint64_t kv_full, q_full[NS], q_empty[NS];
  uint64_t sdp_full, sdp_free, pds_ready, pds_free, dq_full, dq_free, acc_done;
  uint32_t tmem_base;
};

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void red_add_f32(float* addr, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(addr), "f"(v) : "memory");
}

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

template <int D, typename AccT>
__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                    const __grid_constant__ BwdParams prm) {
  using Cfg = BwdCfg<D>;
  constexpr int BQ = Cfg::BQ, NS = Cfg::NS;
  constexpr int kSlabQ = BQ * 64;    // elements per [BQ][64] slab
  constexpr int kSlabK = kBK * 64;   // elements per [128][64] slab
  extern __shared__ uint8_t smem_raw[];
  auto& sm = *reinterpret_cast<BwdSmem<D>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int kt = blockIdx.x;  // key tile over the concatenated chunk list
  const int kvh = blockIdx.y;
  const int key0 = kt * kBK;
  const int off = prm.total_kv - prm.q_rows;  // causal alignment offset
  int t_min = 0;
  if (prm.causal) {
    const int num = key0 - off - BQ + 1;
    t_min = num > 0 ? (num + BQ - 1) / BQ : 0;
  }
  const int tiles_per_head = prm.n_qtiles - t_min;
  const int n_pairs = tiles_per_head > 0 ? tiles_per_head * prm.group : 0;
  const int chunk = key0 / prm.chunk_len;
  const int kv_prow = prm.chunk_row[chunk] + key0 % prm.chunk_len;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    mbar_init(&sm.kv_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm.q_full[s], 1);
      mbar_init(&sm.q_empty[s], 1);
    }
    mbar_init(&sm.sdp_full, 1);
    mbar_init(&sm.sdp_free, 128);
    mbar_init(&sm.pds_ready, 128);
    mbar_init(&sm.pds_free, 1);
    mbar_init(&sm.dq_full, 1);
    mbar_init(&sm.dq_free, 128);
    mbar_init(&sm.acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    if (lane == 0 && n_pairs > 0) {
      // ---------------- TMA producer
      mbar_arrive_expect_tx(&sm.kv_full, 2 * kBK * D * 2);
      for (int sl = 0; sl < D / 64; ++sl) {
        tma_load_2d(sm.k + sl * kSlabK, &tm_k, &sm.kv_full, kvh * D + sl * 64, kv_prow);
        tma_load_2d(sm.v + sl * kSlabK, &tm_v, &sm.kv_full, kvh * D + sl * 64, kv_prow);
      }
      for (int j = 0; j < n_pairs; ++j) {
        const int s = j % NS;
        const int h = kvh * prm.group + j / tiles_per_head;
        const int qrow = (t_min + j % tiles_per_head) * BQ;
        mbar_wait(&sm.q_empty[s], ((j / NS) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.q_full[s], 2 * BQ * D * 2 + 2 * BQ * 4);
        for (int sl = 0; sl < D / 64; ++sl) {
          tma_load_2d(sm.q[s] + sl * kSlabQ, &tm_q, &sm.q_full[s], h * D + sl * 64, qrow);
          tma_load_2d(sm.dout[s] + sl * kSlabQ, &tm_do, &sm.q_full[s], h * D + sl * 64, qrow);
        }
        bulk_load(sm.lse2[s], prm.lse2 + int64_t(h) * prm.q_rows + qrow, BQ * 4, &sm.q_full[s]);
        bulk_load(sm.delta[s], prm.delta + int64_t(h) * prm.q_rows + qrow, BQ * 4, &sm.q_full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && n_pairs > 0) {
      // ---------------- UMMA issuer
      constexpr uint32_t id_s = idesc_bf16_f32(kBK, BQ, false, false);   // K Q^T, V dO^T
      constexpr uint32_t id_acc = idesc_bf16_f32(kBK, D, false, true);   // P^T dO, dS^T Q
      constexpr uint32_t id_dq = Cfg::kDqT ? idesc_bf16_f32(D, BQ, true, true)     // K^T dS^T
                                           : idesc_bf16_f32(BQ, D, true, true);    // dS K
      const uint32_t k_a = smem_u32(sm.k), v_a = smem_u32(sm.v), p_a = smem_u32(sm.p), ds_a = smem_u32(sm.ds);
      mbar_wait(&sm.kv_full, 0);
      for (int j = 0; j < n_pairs; ++j) {
        const int s = j % NS;
        const uint32_t q_a = smem_u32(sm.q[s]), do_a = smem_u32(sm.dout[s]);
        mbar_wait(&sm.q_full[s], (j / NS) & 1);
        if (j > 0) mbar_wait(&sm.sdp_free, (j - 1) & 1);
        tc_fence_after();
        // S^T = K Q^T and dP^T = V dO^T (K-major both, K = D)
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t oa = (kk / 4) * (kSlabK * 2) + (kk % 4) * 32;
          const uint32_t ob = (kk / 4) * (kSlabQ * 2) + (kk % 4) * 32;
          umma_bf16_ss(tmem + Cfg::kS, smem_desc_sw128(k_a + oa, 16, 1024), smem_desc_sw128(q_a + ob, 16, 1024),
                       id_s, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t oa = (kk / 4) * (kSlabK * 2) + (kk % 4) * 32;
          const uint32_t ob = (kk / 4) * (kSlabQ * 2) + (kk % 4) * 32;
          umma_bf16_ss(tmem + Cfg::kDP, smem_desc_sw128(v_a + oa, 16, 1024), smem_desc_sw128(do_a + ob, 16, 1024),
                       id_s, kk > 0);
        }
        umma_commit(&sm.sdp_full);
        mbar_wait(&sm.pds_ready, j & 1);
        tc_fence_after();
        // dV += P^T dO ; dK += dS^T Q   (A K-major [keys][BQ], B MN-major [BQ][D])
#pragma unroll
        for (int kk = 0; kk < BQ / 16; ++kk) {
          const uint32_t oa = (kk / 4) * (kSlabK * 2) + (kk % 4) * 32;
          const uint32_t ob = kk * 16 * 128;
          umma_bf16_ss(tmem + Cfg::kDV, smem_desc_sw128(p_a + oa, 16, 1024),
                       smem_desc_sw128(do_a + ob, kSlabQ * 2, 1024), id_acc, (j > 0 || kk > 0) ? 1u : 0u);
          umma_bf16_ss(tmem + Cfg::kDK, smem_desc_sw128(ds_a + oa, 16, 1024),
                       smem_desc_sw128(q_a + ob, kSlabQ * 2, 1024), id_acc, (j > 0 || kk > 0) ? 1u : 0u);
        }
        if (j > 0) mbar_wait(&sm.dq_free, (j - 1) & 1);
        tc_fence_after();
        // dQ (K = 128 keys; both operands MN-major, 16 keys = 2048 B per step)
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk) {
          const uint32_t ok = kk * 16 * 128;
          if constexpr (Cfg::kDqT)  // A = K^T (M = D groups of 64 -> slab stride), B = dS^T (N = BQ)
            umma_bf16_ss(tmem + Cfg::kDQ, smem_desc_sw128(k_a + ok, kSlabK * 2, 1024),
                         smem_desc_sw128(ds_a + ok, kSlabK * 2, 1024), id_dq, kk > 0);
          else  // A = dS (M = BQ = 128 -> two 64-q slabs), B = K (N = D = 64)
            umma_bf16_ss(tmem + Cfg::kDQ, smem_desc_sw128(ds_a + ok, kSlabK * 2, 1024),
                         smem_desc_sw128(k_a + ok, kSlabK * 2, 1024), id_dq, kk > 0);
        }
        umma_commit(&sm.dq_full);
        umma_commit(&sm.q_empty[s]);
        umma_commit(&sm.pds_free);
      }
      umma_commit(&sm.acc_done);
    }
  } else {
    // ---------------- element math, warps 2..5
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // TMEM lane: key row (S^T, dP^T, dV, dK) / d or q row (dQ)
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const uint32_t p_a = smem_u32(sm.p), ds_a = smem_u32(sm.ds);
    const int key_rel = key0 - off + r;  // key position relative to query row 0's limit
    for (int j = 0; j < n_pairs; ++j) {
      const int s = j % NS;
      const int h = kvh * prm.group + j / tiles_per_head;
      const int qrow0 = (t_min + j % tiles_per_head) * BQ;
      const bool need_mask = prm.causal && (key0 + kBK - 1 - off > qrow0);
      mbar_wait(&sm.q_full[s], (j / NS) & 1);
      mbar_wait(&sm.sdp_full, j & 1);
      if (j > 0) mbar_wait(&sm.pds_free, (j - 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int ch = 0; ch < BQ / 32; ++ch) {
        float sv[32], dp[32];
        tmem_ld32(tmem + lane_off + Cfg::kS + ch * 32, sv);
        tmem_ld32(tmem + lane_off + Cfg::kDP + ch * 32, dp);
        tmem_wait_ld();
        uint32_t pk[16], dk[16];
#pragma unroll
        for (int x = 0; x < 32; x += 2) {
          float pp[2], dd[2];
#pragma unroll
          for (int y = 0; y < 2; ++y) {
            const int c = ch * 32 + x + y;
            float p = fast_exp2(fmaf(sv[x + y], prm.scale_log2, -sm.lse2[s][c]));
            if (need_mask && key_rel > qrow0 + c) p = 0.f;
            pp[y] = p;
            dd[y] = p * (dp[x + y] - sm.delta[s][c]) * prm.scale;
          }
          pk[x / 2] = pack_bf16(pp[0], pp[1]);
          dk[x / 2] = pack_bf16(dd[0], dd[1]);
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int c = ch * 32 + g * 8;  // column within [0, BQ)
          const uint32_t o = (c / 64) * (kSlabK * 2) + sw128_offset(r, c % 64);
          st_shared_v4(p_a + o, pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
          st_shared_v4(ds_a + o, dk[4 * g], dk[4 * g + 1], dk[4 * g + 2], dk[4 * g + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(&sm.sdp_free);
      fence_async_smem();
      mbar_arrive(&sm.pds_ready);
      // drain dQ of this pair
      mbar_wait(&sm.dq_full, j & 1);
      tc_fence_after();
      if constexpr (Cfg::kDqT) {  // lane r = d, columns = query rows
        float dq[BQ];
#pragma unroll
        for (int ch = 0; ch < BQ / 32; ++ch) tmem_ld32(tmem + lane_off + Cfg::kDQ + ch * 32, *reinterpret_cast<float(*)[32]>(&dq[ch * 32]));
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&sm.dq_free);
        float* base = prm.dq + int64_t(qrow0) * prm.dq_stride + h * D + r;
#pragma unroll
        for (int c = 0; c < BQ; ++c) red_add_f32(base + int64_t(c) * prm.dq_stride, dq[c]);
      } else {  // lane r = query row, columns = d
        float dq[D];
#pragma unroll
        for (int ch = 0; ch < D / 32; ++ch) tmem_ld32(tmem + lane_off + Cfg::kDQ + ch * 32, *reinterpret_cast<float(*)[32]>(&dq[ch * 32]));
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&sm.dq_free);
        float* base = prm.dq + int64_t(qrow0 + r) * prm.dq_stride + h * D;
#pragma unroll
        for (int c = 0; c < D; c += 4) red_add_v4(base + c, dq[c], dq[c + 1], dq[c + 2], dq[c + 3]);
      }
    }
    // ---------------- dK / dV accumulate into the fp32 chunk accumulators
    if (n_pairs > 0) {
      mbar_wait(&sm.acc_done, 0);
      tc_fence_after();
      const int64_t arow = prm.acc_row[chunk] + key0 % prm.chunk_len + r;
      AccT* dkp = static_cast<AccT*>(prm.dk) + arow * prm.acc_stride + kvh * D;
      AccT* dvp = static_cast<AccT*>(prm.dv) + arow * prm.acc_stride + kvh * D;
#pragma unroll
      for (int ch = 0; ch < D / 32; ++ch) {
        float a[32], b[32];
        tmem_ld32(tmem + lane_off + Cfg::kDK + ch * 32, a);
        tmem_ld32(tmem + lane_off + Cfg::kDV + ch * 32, b);
        tmem_wait_ld();
        acc_add32(dkp + ch * 32, a);
        acc_add32(dvp + ch * 32, b);
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// delta[h][r] = sum_d dO*O (fp32), lse2[h][r] = lse * log2(e).  One warp per (row, head).
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_prep(const __nv_bfloat16* __restrict__ o, int64_t o_stride,
                                                      const __nv_bfloat16* __restrict__ dout, int64_t do_stride,
                                                      const float* __restrict__ lse, int64_t rows, int heads,
                                                      float* __restrict__ lse2, float* __restrict__ delta) {
  const int64_t item = int64_t(blockIdx.x) * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (item >= rows * heads) return;
  const int64_t row = item / heads;
  const int h = int(item % heads);
  constexpr int kPer = D / 32;
  float acc = 0.f;
#pragma unroll
  for (int x = 0; x < kPer; ++x) {
    const int c = h * D + lane * kPer + x;
    acc += __bfloat162float(o[row * o_stride + c]) * __bfloat162float(dout[row * do_stride + c]);
  }
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
  if (lane == 0) {
    delta[int64_t(h) * rows + row] = acc;
    lse2[int64_t(h) * rows + row] = lse[int64_t(h) * rows + row] * 1.4426950408889634f;
  }
}

template <int D, typename AccT>
int launch_bwd(const CUtensorMap& tq, const CUtensorMap& tdo, const CUtensorMap& tk, const CUtensorMap& tv,
               const BwdParams& prm, int k_tiles, int kv_heads, cudaStream_t st) {
  auto kern = attn_bwd_kernel<D, AccT>;
  const size_t smem = sizeof(BwdSmem<D>) + 1024;
  if (int rc = set_smem_once(reinterpret_cast<const void*>(kern), smem, "attn_bwd: set smem")) return rc;
  kern<<<dim3(k_tiles, kv_heads), kThreads, smem, st>>>(tq, tdo, tk, tv, prm);
  count_launch(1);
  return cuda_status(cudaGetLastError(), "attn_bwd launch");
}

}  // namespace
}  // namespace sp

namespace sp {
namespace {
int bwd_check(int64_t q_rows, int n_chunks, int chunk_len, int heads, int kv_heads, int head_dim, int causal,
              int64_t q_stride, int64_t kv_stride, int64_t do_stride) {
  if (head_dim != 64 && head_dim != 128)
    return set_error(SP_ERR_UNSUPPORTED, "sp_attn_bwd: head_dim %d not in {64,128}", head_dim);
  if (q_rows <= 0 || q_rows % 128 || chunk_len <= 0 || chunk_len % 128 || n_chunks <= 0 || n_chunks > SP_MAX_CHUNKS)
    return set_error(SP_ERR_UNSUPPORTED, "sp_attn_bwd: q_rows/chunk_len must be multiples of 128, 0 < n_chunks <= %d",
                     SP_MAX_CHUNKS);
  if (heads <= 0 || kv_heads <= 0 || heads % kv_heads)
    return set_error(SP_ERR_INVALID, "sp_attn_bwd: heads must be a multiple of kv_heads");
  if (q_stride % 8 || kv_stride % 8 || do_stride % 8)
    return set_error(SP_ERR_INVALID, "sp_attn_bwd: strides must be multiples of 8 elements");
  if (causal && int64_t(n_chunks) * chunk_len < q_rows)
    return set_error(SP_ERR_UNSUPPORTED, "sp_attn_bwd: causal needs total_kv >= q_rows");
  return SP_OK;
}
}  // namespace
}  // namespace sp

namespace sp {
// Force-load this file's kernels (cudaFuncGetAttributes) — see preload_kernels
int preload_attn_bwd() {
  cudaFuncAttributes a;
  if (cudaError_t e = cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(sp::attn_bwd_kernel<64, float>))) return cuda_status(e, "preload sp::attn_bwd_kernel<64>");
  if (cudaError_t e = cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(sp::attn_bwd_kernel<64, __nv_bfloat16>))) return cuda_status(e, "preload sp::attn_bwd_kernel<64, bf16>");
  if (cudaError_t e = cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(sp::attn_bwd_prep<64>))) return cuda_status(e, "preload sp::attn_bwd_prep<64>");
  if (cudaError_t e = cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(sp::attn_bwd_prep<128>))) return cuda_status(e, "preload sp::attn_bwd_prep<128>");
  return SP_OK;
}
}  // namespace sp

extern "C" int sp_attn_bwd_prep(const void* o, int64_t o_stride, const void* dout, int64_t do_stride, const float* lse,
                                int64_t q_rows, int heads, int head_dim, float* stats, sp_stream_t stream) {
  using namespace sp;
  if (head_dim != 64 && head_dim != 128)
    return set_error(SP_ERR_UNSUPPORTED, "sp_attn_bwd_prep: head_dim %d not in {64,128}", head_dim);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* lse2 = stats;
  float* delta = stats + int64_t(heads) * q_rows;
  const int64_t items = q_rows * heads;
  const dim3 grid(unsigned((items + 7) / 8));
  auto* O = static_cast<const __nv_bfloat16*>(o);
  auto* dO = static_cast<const __nv_bfloat16*>(dout);
  if (head_dim == 128)
    attn_bwd_prep<128><<<grid, 256, 0, st>>>(O, o_stride, dO, do_stride, lse, q_rows, heads, lse2, delta);
  else
    attn_bwd_prep<64><<<grid, 256, 0, st>>>(O, o_stride, dO, do_stride, lse, q_rows, heads, lse2, delta);
  count_launch(1);
  return cuda_status(cudaGetLastError(), "attn_bwd_prep launch");
}

namespace sp {
// sp_attn_bwd_core with the chunk accumulators' storage type chosen: fp32, or
// bf16 (acc_bf16; the runtime's dkv_bf16 option)
int attn_bwd_core(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                  int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks, int chunk_len,
                  int heads, int kv_heads, int head_dim, int causal, const void* dout, int64_t do_stride,
                  const float* stats, float* dq_acc, void* dk_acc, void* dv_acc, int64_t acc_rows,
                  const int32_t* acc_row, bool acc_bf16, cudaStream_t stream) {
  if (int rc = bwd_check(q_rows, n_chunks, chunk_len, heads, kv_heads, head_dim, causal, q_stride, kv_stride,
                         do_stride))
    return rc;
  cudaStream_t st = stream;
  const float* lse2 = stats;
  const float* delta = stats + int64_t(heads) * q_rows;
  const int64_t total_kv = int64_t(n_chunks) * chunk_len;
  for (int c = 0; c < n_chunks; ++c)
    if (chunk_row[c] < 0 || int64_t(chunk_row[c]) + chunk_len > pool_rows || acc_row[c] < 0 ||
        int64_t(acc_row[c]) + chunk_len > acc_rows)
      return set_error(SP_ERR_INVALID, "sp_attn_bwd: chunk %d outside the pool/accumulator", c);
  if (head_dim == 128)  // attn_bwd_v2.cu
    return attn_bwd_d128(q, q_rows, q_stride, k_pool, v_pool, pool_rows, kv_stride, chunk_row, n_chunks, chunk_len,
                         heads, kv_heads, causal, dout, do_stride, lse2, delta, dq_acc, dk_acc, dv_acc, acc_rows,
                         acc_row, acc_bf16, st);
  BwdParams prm{};
  prm.q_rows = int(q_rows);
  prm.total_kv = int(total_kv);
  prm.chunk_len = chunk_len;
  prm.group = heads / kv_heads;
  prm.causal = causal;
  const int bq = 128;
  prm.n_qtiles = int(q_rows / bq);
  prm.scale = float(1.0 / sqrt(double(head_dim)));
  prm.scale_log2 = float(1.4426950408889634 / sqrt(double(head_dim)));
  prm.lse2 = lse2;
  prm.delta = delta;
  prm.dq = dq_acc;
  prm.dq_stride = int64_t(heads) * head_dim;
  prm.dk = dk_acc;
  prm.dv = dv_acc;
  prm.acc_stride = int64_t(kv_heads) * head_dim;
  for (int c = 0; c < n_chunks; ++c) {
    prm.chunk_row[c] = chunk_row[c];
    prm.acc_row[c] = acc_row[c];
  }
  CUtensorMap tq, tdo, tk, tv;
  if (!make_tmap_bf16(&tq, q, uint64_t(q_stride), uint64_t(q_rows), uint64_t(q_stride), uint32_t(bq)) ||
      !make_tmap_bf16(&tdo, dout, uint64_t(do_stride), uint64_t(q_rows), uint64_t(do_stride), uint32_t(bq)) ||
      !make_tmap_bf16(&tk, k_pool, uint64_t(kv_stride), uint64_t(pool_rows), uint64_t(kv_stride), 128) ||
      !make_tmap_bf16(&tv, v_pool, uint64_t(kv_stride), uint64_t(pool_rows), uint64_t(kv_stride), 128))
    return set_error(SP_ERR_CUDA, "sp_attn_bwd: cuTensorMapEncodeTiled failed (alignment?)");
  const int k_tiles = int(total_kv / 128);
  return acc_bf16 ? launch_bwd<64, __nv_bfloat16>(tq, tdo, tk, tv, prm, k_tiles, kv_heads, st)
                  : launch_bwd<64, float>(tq, tdo, tk, tv, prm, k_tiles, kv_heads, st);
}
}  // namespace sp

extern "C" int sp_attn_bwd_core(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool,
                                const void* v_pool, int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row,
                                int n_chunks, int chunk_len, int heads, int kv_heads, int head_dim, int causal,
                                const void* dout, int64_t do_stride, const float* stats, float* dq_acc, float* dk_acc,
                                float* dv_acc, int64_t acc_rows, const int32_t* acc_row, sp_stream_t stream) {
  return sp::attn_bwd_core(q, q_rows, q_stride, k_pool, v_pool, pool_rows, kv_stride, chunk_row, n_chunks, chunk_len,
                           heads, kv_heads, head_dim, causal, dout, do_stride, stats, dq_acc, dk_acc, dv_acc, acc_rows,
                           acc_row, false, static_cast<cudaStream_t>(stream));
}

extern "C" int sp_attn_bwd(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                           int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks,
                           int chunk_len, int heads, int kv_heads, int head_dim, int causal, const void* o,
                           int64_t o_stride, const void* dout, int64_t do_stride, const float* lse, float* delta_ws,
                           float* dq_acc, float* dk_acc, float* dv_acc, int64_t acc_rows, const int32_t* acc_row,
                           sp_stream_t stream) {
  using namespace sp;
  if (int rc = bwd_check(q_rows, n_chunks, chunk_len, heads, kv_heads, head_dim, causal, q_stride, kv_stride,
                         do_stride))
    return rc;
  if (o_stride % 8) return set_error(SP_ERR_INVALID, "sp_attn_bwd: strides must be multiples of 8 elements");
  if (int rc = sp_attn_bwd_prep(o, o_stride, dout, do_stride, lse, q_rows, heads, head_dim, delta_ws, stream)) return rc;
  return sp_attn_bwd_core(q, q_rows, q_stride, k_pool, v_pool, pool_rows, kv_stride, chunk_row, n_chunks, chunk_len,
                          heads, kv_heads, head_dim, causal, dout, do_stride, delta_ws, dq_acc, dk_acc, dv_acc,
                          acc_rows, acc_row, stream);
}
