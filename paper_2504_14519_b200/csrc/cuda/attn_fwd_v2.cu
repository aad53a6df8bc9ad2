// K1 (head_dim 128): sliced causal attention forward, production path.
// Same semantics as attn_fwd.cu (reference chunk_attention,
// proj/src/attention.cpp:21-111: scale 1/sqrt(d), bottom-right causal,
// finalize O/l, plus the LSE the backward and the exchange merge need).
//
// Organisation (one CTA = 128 query rows of one head):
//   * TMEM: S double buffer (2 x 128 fp32 cols) + two O accumulators
//     O_A, O_B (128 cols each) = 512 cols.
//   * 8 softmax warps: thread (r, half) owns query row r and key columns
//     [64*half, 64*half+64) of every KV tile, with its OWN running max, sum
//     and accumulator O_half (split-KV inside the CTA).  No cross-thread
//     reduction in the loop; the two halves are merged once in the epilogue
//     exactly like the reference merges partials (attention.cpp:63-92).
//     The per-tile softmax critical path is 64 exponentials per thread.
//   * P is written back as packed bf16 over the thread's own S columns and
//     consumed by TS-UMMAs (A from TMEM): O_half += P_half V[half rows].
//   * the MMA warp issues S(j+1) before PV(j), so the tensor core computes the
//     next scores while the softmax of the current tile runs.  tcgen05 ops of
//     one thread execute in order: S(j+1) may overwrite P(j-1) (issued after
//     PV(j-1)); the softmax waits for PV(j-1) (o_ready) only when it must
//     rescale O (lazy rescale: running max grew by > 8 in log2 units).
// Warps: 0 TMA producer, 1 TMEM owner + UMMA issuer, 2-5 half 0, 6-9 half 1.
#include <math.h>

#include "errors.hpp"
#include "kernels.hpp"
#include "sm100.cuh"

#include <cstdlib>

namespace sp {
namespace {

constexpr int D = 128, BM = 128, BN = 128, NK = 3, NV = 2;
constexpr int kThreads = 320;
constexpr int kSoftmax = 256;
constexpr int kSlab = 128 * 64;

struct Params {
  int q_rows, total_kv, chunk_len, group, causal;
  float scale_log2;
  int dbg;    // diagnostics: 1 = MMA ignores P readiness, 2 = + no K/V reloads
  int trace;  // per-tile timeline of CTA (0,0) into g_fwd_trace (diagnostics)
  __nv_bfloat16* o;
  int64_t o_stride;
  float* lse;
  int chunk_row[SP_MAX_CHUNKS];
};

struct alignas(1024) Smem {
  __nv_bfloat16 q[BM * D];
  __nv_bfloat16 k[NK][BN * D];
  __nv_bfloat16 v[NV][BN * D];
};

struct Ctl {
  uint64_t q_full, k_full[NK], k_empty[NK], v_full[NV], v_empty[NV], s_full[2], p_full[2], o_ready;
  float m_half[2][BM], l_half[2][BM];
  uint32_t tmem_base;
};

// 2^x on the FMA/ALU pipes: x = j + f (j = round(x), |f| <= 1/2), 2^f by a
// degree-4 polynomial (rel. err < 5e-5, far below the bf16 rounding of P),
// 2^j added into the exponent bits.  x is clamped at -126 (result ~0).
__device__ __forceinline__ float poly_exp2(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: round-to-nearest in the mantissa
  const int j = __float_as_int(t) - 0x4B400000;
  const float f = x - (t - 12582912.f);
  float p = fmaf(0.0096181291f, f, 0.0555041087f);
  p = fmaf(p, f, 0.2402264923f);
  p = fmaf(p, f, 0.6931471806f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (j << 23));
}

__device__ long long g_fwd_trace[12][1024];
#define TRF(e, j)                                                           \
  do {                                                                      \
    if (tracing && (j) < 1024) g_fwd_trace[e][(j)] = clock64();            \
  } while (0)

template <int kPoly>  // every kPoly-th pair computes its second exponential on the FMA pipe (0: never)
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_d128_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ Params prm) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(16) Ctl ctl;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tile = gridDim.x - 1 - blockIdx.x;  // longest causal ranges first
  const int head = blockIdx.y;
  const int kvh = head / prm.group;
  const int row0 = tile * BM;
  const int n = prm.causal ? (prm.total_kv - prm.q_rows + row0 + BM) / BN : prm.total_kv / BN;
  const bool tracing = prm.trace && blockIdx.x == 0 && blockIdx.y == 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    mbar_init(&ctl.q_full, 1);
    for (int s = 0; s < NK; ++s) {
      mbar_init(&ctl.k_full[s], 1);
      mbar_init(&ctl.k_empty[s], 1);
    }
    for (int s = 0; s < NV; ++s) {
      mbar_init(&ctl.v_full[s], 1);
      mbar_init(&ctl.v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ctl.s_full[b], 1);
      mbar_init(&ctl.p_full[b], kSoftmax);
    }
    mbar_init(&ctl.o_ready, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&ctl.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl.tmem_base;
  auto kv_row = [&](int j) {
    const int key = j * BN;
    return prm.chunk_row[key / prm.chunk_len] + key % prm.chunk_len;
  };

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&ctl.q_full, BM * D * 2);
      for (int sl = 0; sl < 2; ++sl) tma_load_2d(sm.q + sl * kSlab, &tm_q, &ctl.q_full, head * D + sl * 64, row0);
      auto load_k = [&](int j) {
        const int s = j % NK;
        mbar_wait(&ctl.k_empty[s], ((j / NK) & 1) ^ 1);
        mbar_arrive_expect_tx(&ctl.k_full[s], BN * D * 2);
        for (int sl = 0; sl < 2; ++sl)
          tma_load_2d(sm.k[s] + sl * kSlab, &tm_k, &ctl.k_full[s], kvh * D + sl * 64, kv_row(j));
      };
      auto load_v = [&](int j) {
        const int s = j % NV;
        mbar_wait(&ctl.v_empty[s], ((j / NV) & 1) ^ 1);
        mbar_arrive_expect_tx(&ctl.v_full[s], BN * D * 2);
        for (int sl = 0; sl < 2; ++sl)
          tma_load_2d(sm.v[s] + sl * kSlab, &tm_v, &ctl.v_full[s], kvh * D + sl * 64, kv_row(j));
      };
      // consumption order: S(0), S(1), PV(0), S(2), PV(1), ... (K two ahead of V)
      int jk = 0;
      for (; jk < n && jk < 2; ++jk) load_k(jk);
      const int nload = (prm.dbg & 2) ? (n < NV ? n : NV) : n;
      if (prm.dbg & 2) for (; jk < n && jk < NK; ++jk) load_k(jk);
      for (int jv = 0; jv < nload; ++jv) {
        load_v(jv);
        if (jk < n && !(prm.dbg & 2)) load_k(jk++);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = idesc_bf16_f32(BM, BN, false, false);
      constexpr uint32_t id_o = idesc_bf16_f32(BM, D, false, true);
      const uint32_t q_a = smem_u32(sm.q);
      auto issue_s = [&](int j) {
        const int s = j % NK;
        if (!(prm.dbg & 2) || j < NK) mbar_wait(&ctl.k_full[s], (j / NK) & 1);
        TRF(10, j);
        tc_fence_after();
        const uint32_t k_a = smem_u32(sm.k[s]);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t o = (kk / 4) * (kSlab * 2) + (kk % 4) * 32;
          umma_bf16_ss(tmem + (j & 1) * 128, smem_desc_sw128(q_a + o, 16, 1024), smem_desc_sw128(k_a + o, 16, 1024),
                       id_s, kk > 0);
        }
        umma_commit(&ctl.s_full[j & 1]);
        umma_commit(&ctl.k_empty[s]);
      };
      mbar_wait(&ctl.q_full, 0);
      tc_fence_after();
      if (n > 0) issue_s(0);
      for (int j = 0; j < n; ++j) {
        // S(j+1) into the other buffer: softmax(j-1) finished with it (p_full
        // waited in iteration j-1) and P(j-1) is consumed by PV(j-1), issued
        // before this MMA (in-order tcgen05 pipe).
        TRF(0, j);
        if (j + 1 < n && !(prm.dbg & 8)) issue_s(j + 1);
        TRF(1, j);
        if (!(prm.dbg & 1)) mbar_wait(&ctl.p_full[j & 1], (j >> 1) & 1);
        TRF(2, j);
        if (!(prm.dbg & 2) || j < NV) mbar_wait(&ctl.v_full[j % NV], (j / NV) & 1);
        TRF(3, j);
        tc_fence_after();
        const uint32_t v_a = smem_u32(sm.v[j % NV]);
        const uint32_t p_t = tmem + (j & 1) * 128;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // keys [64hf + 16kk, +16)
            if (!(prm.dbg & 4))
            umma_bf16_ts(tmem + 256 + hf * 128, p_t + hf * 64 + kk * 8,
                         smem_desc_sw128(v_a + (hf * 64 + kk * 16) * 128, kSlab * 2, 1024), id_o,
                         (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&ctl.v_empty[j % NV]);
        umma_commit(&ctl.o_ready);
        TRF(4, j);
      }
    }
  } else {
    // ------------------------------------------------ softmax: row r, key half hf
    const int hf = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const uint32_t o_col = tmem + 256 + hf * 128 + lane_off;
    const float sl2 = prm.scale_log2;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < ((prm.dbg & 16) ? 0 : n); ++j) {
      const int b = j & 1;
      const uint32_t s_col = tmem + b * 128 + hf * 64 + lane_off;
      const bool tl = tracing && warp == 2 && lane == 0;
      if (tl) TRF(5, j);
      mbar_wait(&ctl.s_full[b], (j >> 1) & 1);
      if (tl) TRF(6, j);
      tc_fence_after();
      const bool diag = prm.causal && j == n - 1;
      float sv[64];
      tmem_ld32(s_col, *reinterpret_cast<float(*)[32]>(&sv[0]));
      tmem_ld32(s_col + 32, *reinterpret_cast<float(*)[32]>(&sv[32]));
      tmem_wait_ld();
      if (diag) {
#pragma unroll
        for (int x = 0; x < 64; ++x)
          if (hf * 64 + x > r) sv[x] = -INFINITY;
      }
      // tree reduction: 8 independent chains instead of one 64-long FMNMX chain
      float m8[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) m8[x] = fmaxf(sv[x], sv[x + 8]);
#pragma unroll
      for (int x = 16; x < 64; x += 8)
#pragma unroll
        for (int y = 0; y < 8; ++y) m8[y] = fmaxf(m8[y], sv[x + y]);
      const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      if (tl) TRF(7, j);
      const float cand = mx * sl2;
      const bool grow = cand > m_used + 8.0f;
      float corr = 1.f;
      if (grow) {
        corr = fast_exp2(m_used - cand);  // 0 while m_used == -inf
        m_used = cand;
      }
      const float msub = m_used == -INFINITY ? 0.f : m_used;
      if (j > 0 && __any_sync(0xffffffffu, grow)) {
        mbar_wait(&ctl.o_ready, (j - 1) & 1);  // PV(j-1) complete: O stable
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          float ov[32];
          tmem_ld32(o_col + c * 32, ov);
          tmem_wait_ld();
#pragma unroll
          for (int x = 0; x < 32; ++x) ov[x] *= corr;
          tmem_st32(o_col + c * 32, ov);
        }
      }
      float rs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t pk[16];
#pragma unroll
        for (int x = 0; x < 16; ++x) {
          const float a = fast_exp2(fmaf(sv[h * 32 + 2 * x], sl2, -msub));
          const float xc = fmaf(sv[h * 32 + 2 * x + 1], sl2, -msub);
          const float c = (kPoly > 0 && x % (kPoly > 0 ? kPoly : 1) == 0) ? poly_exp2(xc) : fast_exp2(xc);
          rs[(2 * x) & 7] += a;
          rs[(2 * x + 1) & 7] += c;
          pk[x] = pack_bf16(a, c);
        }
        tmem_st16(s_col + h * 16, pk);
      }
      l = l * corr + (((rs[0] + rs[1]) + (rs[2] + rs[3])) + ((rs[4] + rs[5]) + (rs[6] + rs[7])));
      if (tl) TRF(8, j);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&ctl.p_full[b]);
      if (tl) TRF(9, j);
    }
    // ---------------- epilogue: merge the two halves (reference merge_partials)
    ctl.m_half[hf][r] = m_used;
    ctl.l_half[hf][r] = l;
    if (n > 0) {
      mbar_wait(&ctl.o_ready, (n - 1) & 1);
      tc_fence_after();
    }
    named_bar_sync(1, kSoftmax);
    const float ma = ctl.m_half[0][r], mb = ctl.m_half[1][r];
    const float m = fmaxf(ma, mb);
    const float wa = ma == -INFINITY ? 0.f : fast_exp2(ma - m);
    const float wb = mb == -INFINITY ? 0.f : fast_exp2(mb - m);
    const float lt = ctl.l_half[0][r] * wa + ctl.l_half[1][r] * wb;
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    const int qrow = row0 + r;
    __nv_bfloat16* orow = prm.o + int64_t(qrow) * prm.o_stride + head * D + hf * 64;
#pragma unroll
    for (int c = 0; c < 2; ++c) {  // this thread writes output columns [64hf + 32c, +32)
      float oa[32], ob[32];
      if (n > 0) {
        tmem_ld32(tmem + 256 + lane_off + hf * 64 + c * 32, oa);
        tmem_ld32(tmem + 384 + lane_off + hf * 64 + c * 32, ob);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int x = 0; x < 32; ++x) oa[x] = ob[x] = 0.f;
      }
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        float y[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) y[e] = (oa[8 * x + e] * wa + ob[8 * x + e] * wb) * inv;
        dst[x] = make_uint4(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]), pack_bf16(y[4], y[5]), pack_bf16(y[6], y[7]));
      }
    }
    if (hf == 0)
      prm.lse[int64_t(head) * prm.q_rows + qrow] = lt > 0.f ? (m + __log2f(lt)) * 0.69314718055994530942f : -INFINITY;
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

int attn_fwd_d128(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                  int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks, int chunk_len,
                  int heads, int kv_heads, int causal, void* o, int64_t o_stride, float* lse, cudaStream_t st) {
  Params prm{};
  prm.q_rows = int(q_rows);
  prm.total_kv = n_chunks * chunk_len;
  prm.chunk_len = chunk_len;
  prm.group = heads / kv_heads;
  prm.causal = causal;
  prm.scale_log2 = float(1.4426950408889634 / sqrt(double(D)));
  prm.trace = getenv("SP_FWD_TRACE") != nullptr;
  prm.dbg = getenv("SP_FWD_DBG") ? atoi(getenv("SP_FWD_DBG")) : 0;
  prm.o = static_cast<__nv_bfloat16*>(o);
  prm.o_stride = o_stride;
  prm.lse = lse;
  for (int c = 0; c < n_chunks; ++c) prm.chunk_row[c] = chunk_row[c];
  CUtensorMap tq, tk, tv;
  if (!make_tmap_bf16(&tq, q, uint64_t(q_stride), uint64_t(q_rows), uint64_t(q_stride), BM) ||
      !make_tmap_bf16(&tk, k_pool, uint64_t(kv_stride), uint64_t(pool_rows), uint64_t(kv_stride), BN) ||
      !make_tmap_bf16(&tv, v_pool, uint64_t(kv_stride), uint64_t(pool_rows), uint64_t(kv_stride), BN))
    return set_error(SP_ERR_CUDA, "attn_fwd_d128: cuTensorMapEncodeTiled failed (alignment?)");
  const size_t smem = sizeof(Smem) + 1024;
  static const int poly = getenv("SP_POLY") ? atoi(getenv("SP_POLY")) : 0;
  auto kern = poly == 1   ? attn_fwd_d128_kernel<1>
              : poly == 2 ? attn_fwd_d128_kernel<2>
              : poly == 4 ? attn_fwd_d128_kernel<4>
                          : attn_fwd_d128_kernel<0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return cuda_status(e, "attn_fwd_d128: set smem");
  kern<<<dim3(unsigned(q_rows / BM), heads), kThreads, smem, st>>>(tq, tk, tv, prm);
  count_launch(1);
  return cuda_status(cudaGetLastError(), "attn_fwd_d128 launch");
}

int fwd_trace_copy(long long* out) {
  return cuda_status(cudaMemcpyFromSymbol(out, g_fwd_trace, sizeof(long long) * 12 * 1024), "trace copy");
}

}  // namespace sp

extern "C" int sp_debug_fwd_trace(long long* out) { return sp::fwd_trace_copy(out); }
