// K1: sliced causal attention forward on sm_100a (tcgen05 + TMEM + TMA).
//
// Semantics = reference chunk_attention (proj/src/attention.cpp:94-111) per
// (query head, slice): online softmax over an ordered list of KV chunks,
// scale 1/sqrt(d) (:31), bottom-right causal alignment (:34-35), finalised
// output O = acc / sumexp (:84-92), plus the row log-sum-exp the backward and
// the exchange merge (K3) need.  Chunks live anywhere in a KV pool (the slot
// arena); the kernel walks them through a row table.
//
// One CTA = one 128-row query tile of one head.  Warp roles:
//   warp 0      TMA producer: Q once, then K/V tiles into an NS-deep ring
//   warp 1      TMEM owner + UMMA issuer (one elected lane):
//                 S[b] = Q K^T   (M=128, N=128, K=D)    b = tile parity
//                 O   += P V     (M=128, N=D,   K=128)  P from smem
//   warps 2..5  softmax (one query row per thread, TMEM lane = row):
//                 S -> exp2 -> P (bf16, SW128 smem), lazy O rescale in TMEM
//                 (only when the running max grows by > 8 in log2 units),
//                 final O / l, LSE.
// TMEM: S double buffer (2 x 128 cols) + O (D cols) -> 512-col allocation.
#include <math.h>

#include "errors.hpp"
#include "slimpipe.h"
#include "sm100.cuh"
#include "kernels.hpp"


namespace sp {
namespace {

constexpr int kBM = 128;  // query rows per CTA
constexpr int kBN = 128;  // keys per KV tile
constexpr int kThreads = 192;

struct FwdParams {
  int q_rows;
  int total_kv;
  int chunk_len;
  int group;  // heads / kv_heads
  int causal;
  int kv_valid;        // keys >= kv_valid are masked (padding)
  int64_t causal_off;  // causal: query row r sees keys <= r + causal_off
  float* row_max;      // optional true row max (natural log units of scaled scores)
  float scale_log2;
  __nv_bfloat16* o;
  int64_t o_stride;
  float* lse;
  int chunk_row[SP_MAX_CHUNKS];
};

template <int D, int NS>
struct alignas(1024) FwdSmem {
  __nv_bfloat16 q[kBM * D];
  __nv_bfloat16 k[NS][kBN * D];
  __nv_bfloat16 v[NS][kBN * D];
  __nv_bfloat16 p[kBM * kBN];
  uint64_t q_full;
  uint64_t k_full[NS], k_empty[NS], v_full[NS], v_empty[NS];
  uint64_t s_full[2];
  uint64_t p_full;
  uint64_t o_done;
  uint32_t tmem_base;
};

template <int D, int NS>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ FwdParams prm) {
  extern __shared__ uint8_t smem_raw[];
  auto& sm = *reinterpret_cast<FwdSmem<D, NS>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kSlab = 128 * 64;  // elements per [128][64] slab
  constexpr uint32_t kTileBytes = kBN * D * 2;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int tile = gridDim.x - 1 - blockIdx.x;  // heaviest (longest causal range) first
  const int head = blockIdx.y;
  const int kv_head = head / prm.group;
  const int row0 = tile * kBM;
  int64_t kmax = prm.kv_valid - 1;  // last key visible to some row of the tile
  if (prm.causal) kmax = min(kmax, int64_t(row0) + kBM - 1 + prm.causal_off);
  const int n_tiles = kmax < 0 ? 0 : int(kmax / kBN + 1);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    mbar_init(&sm.s_full[0], 1);
    mbar_init(&sm.s_full[1], 1);
    mbar_init(&sm.p_full, 128);
    mbar_init(&sm.o_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const uint32_t tmem_o = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      mbar_arrive_expect_tx(&sm.q_full, kBM * D * 2);
      for (int sl = 0; sl < D / 64; ++sl) tma_load_2d(sm.q + sl * kSlab, &tm_q, &sm.q_full, head * D + sl * 64, row0);
      for (int j = 0; j < n_tiles; ++j) {
        const int s = j % NS;
        const uint32_t ph = (j / NS) & 1;
        const int key = j * kBN;
        const int prow = prm.chunk_row[key / prm.chunk_len] + key % prm.chunk_len;
        mbar_wait(&sm.k_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&sm.k_full[s], kTileBytes);
        for (int sl = 0; sl < D / 64; ++sl)
          tma_load_2d(sm.k[s] + sl * kSlab, &tm_k, &sm.k_full[s], kv_head * D + sl * 64, prow);
        mbar_wait(&sm.v_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&sm.v_full[s], kTileBytes);
        for (int sl = 0; sl < D / 64; ++sl)
          tma_load_2d(sm.v[s] + sl * kSlab, &tm_v, &sm.v_full[s], kv_head * D + sl * 64, prow);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- UMMA issuer
      constexpr uint32_t idesc_s = idesc_bf16_f32(kBM, kBN, false, false);
      constexpr uint32_t idesc_o = idesc_bf16_f32(kBM, D, false, true);
      const uint32_t q_addr = smem_u32(sm.q);
      const uint32_t p_addr = smem_u32(sm.p);
      auto issue_s = [&](int j) {
        const int s = j % NS;
        mbar_wait(&sm.k_full[s], (j / NS) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sm.k[s]);
        const uint32_t d_tmem = tmem + (j & 1) * 128;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * (kSlab * 2) + (kk % 4) * 32;
          umma_bf16_ss(d_tmem, smem_desc_sw128(q_addr + off, 16, 1024), smem_desc_sw128(k_addr + off, 16, 1024),
                       idesc_s, kk > 0);
        }
        umma_commit(&sm.s_full[j & 1]);
        umma_commit(&sm.k_empty[s]);
      };
      mbar_wait(&sm.q_full, 0);
      tc_fence_after();
      if (n_tiles > 0) issue_s(0);
      for (int j = 0; j < n_tiles; ++j) {
        if (j + 1 < n_tiles) issue_s(j + 1);
        const int s = j % NS;
        mbar_wait(&sm.p_full, j & 1);
        mbar_wait(&sm.v_full[s], (j / NS) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sm.v[s]);
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          const uint32_t a_off = (kk / 4) * (kSlab * 2) + (kk % 4) * 32;
          const uint32_t b_off = kk * 16 * 128;  // 16 key rows of 128 B
          umma_bf16_ss(tmem_o, smem_desc_sw128(p_addr + a_off, 16, 1024),
                       smem_desc_sw128(v_addr + b_off, kSlab * 2, 1024), idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&sm.v_empty[s]);
        umma_commit(&sm.o_done);
      }
    }
  } else {
    // ---------------- softmax warps 2..5
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // row within the tile == TMEM lane
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const uint32_t p_addr = smem_u32(sm.p);
    const float sl2 = prm.scale_log2;
    float m_used = -INFINITY;  // running max, log2 units of scaled scores
    float l = 0.f, m_true = -INFINITY;
    float sv[kBN];
    const int64_t qlim = prm.causal ? min(int64_t(prm.kv_valid) - 1, int64_t(row0 + r) + prm.causal_off)
                                    : int64_t(prm.kv_valid) - 1;
    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(&sm.s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < kBN / 32; ++c)
        tmem_ld32(tmem + lane_off + (j & 1) * 128 + c * 32, *reinterpret_cast<float(*)[32]>(&sv[c * 32]));
      tmem_wait_ld();
      const int64_t lim = qlim - int64_t(j) * kBN;  // columns c > lim are masked
      if (lim < kBN - 1) {
        const int lm = lim < -1 ? -1 : int(lim);
#pragma unroll
        for (int c = 0; c < kBN; ++c)
          if (c > lm) sv[c] = -INFINITY;
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < kBN; ++c) mx = fmaxf(mx, sv[c]);
      m_true = fmaxf(m_true, mx);
      const float cand = mx * sl2;
      const bool grow = cand > m_used + 8.0f;
      float corr = 1.f;
      if (grow) {
        corr = fast_exp2(m_used - cand);  // 0 when m_used == -inf
        m_used = cand;
      }
      const float msub = m_used == -INFINITY ? 0.f : m_used;
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < kBN; ++c) {
        sv[c] = fast_exp2(fmaf(sv[c], sl2, -msub));
        rs += sv[c];
      }
      l = l * corr + rs;
      if (j > 0) {
        mbar_wait(&sm.o_done, (j - 1) & 1);  // PV(j-1) done: P free, O stable
        tc_fence_after();
        if (__any_sync(0xffffffffu, grow)) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            float ov[32];
            tmem_ld32(tmem_o + lane_off + c * 32, ov);
            tmem_wait_ld();
#pragma unroll
            for (int x = 0; x < 32; ++x) ov[x] *= corr;
            tmem_st32(tmem_o + lane_off + c * 32, ov);
          }
          tmem_wait_st();
        }
      }
#pragma unroll
      for (int g = 0; g < kBN / 8; ++g) {
        const int c = g * 8;
        const uint32_t addr = p_addr + (c / 64) * (kSlab * 2) + sw128_offset(r, c % 64);
        st_shared_v4(addr, pack_bf16(sv[c], sv[c + 1]), pack_bf16(sv[c + 2], sv[c + 3]),
                     pack_bf16(sv[c + 4], sv[c + 5]), pack_bf16(sv[c + 6], sv[c + 7]));
      }
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(&sm.p_full);
    }
    // ---------------- epilogue
    const int grow_row = row0 + r;
    __nv_bfloat16* orow = prm.o + int64_t(grow_row) * prm.o_stride + head * D;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    if (n_tiles > 0) {
      mbar_wait(&sm.o_done, (n_tiles - 1) & 1);
      tc_fence_after();
    }
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float ov[32];
      if (n_tiles > 0) {
        tmem_ld32(tmem_o + lane_off + c * 32, ov);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int x = 0; x < 32; ++x) ov[x] = 0.f;
      }
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int x = 0; x < 4; ++x)
        dst[x] = make_uint4(pack_bf16(ov[8 * x] * inv, ov[8 * x + 1] * inv), pack_bf16(ov[8 * x + 2] * inv, ov[8 * x + 3] * inv),
                            pack_bf16(ov[8 * x + 4] * inv, ov[8 * x + 5] * inv), pack_bf16(ov[8 * x + 6] * inv, ov[8 * x + 7] * inv));
    }
    prm.lse[int64_t(head) * prm.q_rows + grow_row] =
        l > 0.f ? (m_used + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
    if (prm.row_max)
      prm.row_max[int64_t(head) * prm.q_rows + grow_row] =
          l > 0.f ? m_true * prm.scale_log2 * 0.69314718055994530942f : -INFINITY;
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int D, int NS>
int launch_fwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const FwdParams& prm, int q_tiles,
               int heads, cudaStream_t stream) {
  auto kern = attn_fwd_kernel<D, NS>;
  const size_t smem = sizeof(FwdSmem<D, NS>) + 1024;
  if (int rc = set_smem_once(reinterpret_cast<const void*>(kern), smem, "attn_fwd: set smem")) return rc;
  kern<<<dim3(q_tiles, heads), kThreads, smem, stream>>>(tq, tk, tv, prm);
  count_launch(1);
  return cuda_status(cudaGetLastError(), "attn_fwd launch");
}

}  // namespace
}  // namespace sp

namespace sp {
namespace {

// Shared by sp_attn_fwd and sp_attn_fwd_masked: validation, then the d=128
// (attn_fwd_v4.cu) or d=64 kernel.
int attn_fwd_dispatch(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                      int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks, int chunk_len,
                      int heads, int kv_heads, int head_dim, const FwdMask& mk, void* o, int64_t o_stride, float* lse,
                      cudaStream_t st) {
  if (head_dim != 64 && head_dim != 128)
    return set_error(SP_ERR_UNSUPPORTED, "sp_attn_fwd: head_dim %d not in {64,128}", head_dim);
  if (q_rows <= 0 || q_rows % 128 || chunk_len <= 0 || chunk_len % 128 || n_chunks < 0 || n_chunks > SP_MAX_CHUNKS)
    return set_error(SP_ERR_UNSUPPORTED, "sp_attn_fwd: q_rows/chunk_len must be multiples of 128, n_chunks <= %d",
                     SP_MAX_CHUNKS);
  if (heads <= 0 || kv_heads <= 0 || heads % kv_heads)
    return set_error(SP_ERR_INVALID, "sp_attn_fwd: heads must be a multiple of kv_heads");
  if (q_stride % 8 || kv_stride % 8 || o_stride % 8 || q_stride < int64_t(heads) * head_dim ||
      kv_stride < int64_t(kv_heads) * head_dim)
    return set_error(SP_ERR_INVALID, "sp_attn_fwd: bad strides");
  const int64_t total_kv = int64_t(n_chunks) * chunk_len;
  if (total_kv > INT32_MAX || mk.kv_valid < 0 || mk.kv_valid > total_kv || !(mk.scale > 0.0))
    return set_error(SP_ERR_INVALID, "sp_attn_fwd: bad key range or scale");
  for (int c = 0; c < n_chunks; ++c)
    if (chunk_row[c] < 0 || int64_t(chunk_row[c]) + chunk_len > pool_rows)
      return set_error(SP_ERR_INVALID, "sp_attn_fwd: chunk %d outside the pool", c);
  if (head_dim == 128)
    return attn_fwd_d128_ps(q, q_rows, q_stride, k_pool, v_pool, pool_rows, kv_stride, chunk_row, n_chunks, chunk_len,
                            heads, kv_heads, mk, o, o_stride, lse, st);
  FwdParams prm{};
  prm.q_rows = int(q_rows);
  prm.total_kv = int(total_kv);
  prm.chunk_len = chunk_len;
  prm.group = heads / kv_heads;
  prm.causal = mk.causal;
  prm.kv_valid = int(mk.kv_valid);
  prm.causal_off = mk.causal_off;
  prm.row_max = mk.row_max;
  prm.scale_log2 = float(1.4426950408889634 * mk.scale);
  prm.o = static_cast<__nv_bfloat16*>(o);
  prm.o_stride = o_stride;
  prm.lse = lse;
  for (int c = 0; c < n_chunks; ++c) prm.chunk_row[c] = chunk_row[c];
  CUtensorMap tq, tk, tv;
  if (!make_tmap_bf16(&tq, q, uint64_t(q_stride), uint64_t(q_rows), uint64_t(q_stride), 128) ||
      !make_tmap_bf16(&tk, k_pool, uint64_t(kv_stride), uint64_t(pool_rows), uint64_t(kv_stride), 128) ||
      !make_tmap_bf16(&tv, v_pool, uint64_t(kv_stride), uint64_t(pool_rows), uint64_t(kv_stride), 128))
    return set_error(SP_ERR_CUDA, "sp_attn_fwd: cuTensorMapEncodeTiled failed (alignment?)");
  return launch_fwd<64, 3>(tq, tk, tv, prm, int(q_rows / 128), heads, st);
}

}  // namespace
}  // namespace sp

namespace sp {
// Force-load this file's kernels (cudaFuncGetAttributes) — see preload_kernels
int preload_attn_fwd() {
  cudaFuncAttributes a;
  if (cudaError_t e = cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(sp::attn_fwd_kernel<64, 3>))) return cuda_status(e, "preload sp::attn_fwd_kernel<64, 3>");
  return SP_OK;
}
}  // namespace sp

extern "C" int sp_attn_fwd(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                           int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks,
                           int chunk_len, int heads, int kv_heads, int head_dim, int causal, void* o,
                           int64_t o_stride, float* lse, sp_stream_t stream) {
  using namespace sp;
  const int64_t total_kv = int64_t(n_chunks) * chunk_len;
  if (causal && total_kv < q_rows)
    return set_error(SP_ERR_UNSUPPORTED, "sp_attn_fwd: causal needs total_kv >= q_rows");
  FwdMask mk;
  mk.causal = causal;
  mk.causal_off = total_kv - q_rows;  // bottom-right aligned, reference attention.cpp:34-35
  mk.kv_valid = total_kv;
  mk.scale = head_dim > 0 ? 1.0 / sqrt(double(head_dim)) : 0.0;  // attention.cpp:31
  return attn_fwd_dispatch(q, q_rows, q_stride, k_pool, v_pool, pool_rows, kv_stride, chunk_row, n_chunks, chunk_len,
                           heads, kv_heads, head_dim, mk, o, o_stride, lse, static_cast<cudaStream_t>(stream));
}

extern "C" int sp_attn_fwd_masked(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool,
                                  const void* v_pool, int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row,
                                  int n_chunks, int chunk_len, int heads, int kv_heads, int head_dim, int causal,
                                  int64_t causal_off, int64_t kv_valid, double scale, void* o, int64_t o_stride,
                                  float* lse, float* row_max, sp_stream_t stream) {
  using namespace sp;
  FwdMask mk;
  mk.causal = causal;
  mk.causal_off = causal_off;
  mk.kv_valid = kv_valid;
  mk.scale = scale;
  mk.row_max = row_max;
  return attn_fwd_dispatch(q, q_rows, q_stride, k_pool, v_pool, pool_rows, kv_stride, chunk_row, n_chunks, chunk_len,
                           heads, kv_heads, head_dim, mk, o, o_stride, lse, static_cast<cudaStream_t>(stream));
}
