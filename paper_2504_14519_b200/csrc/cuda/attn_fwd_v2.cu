// K1 (head_dim 128): sliced causal attention forward, two query tiles per CTA,
// P kept in TMEM.  Same semantics as attn_fwd.cu (reference chunk_attention,
// proj/src/attention.cpp:21-111: scale 1/sqrt(d), bottom-right causal,
// finalize O/l, plus LSE); this is the production path for d = 128.
//
// Why: with P staged through shared memory the forward is shared-memory
// bandwidth bound (S = QK^T and O += PV are both SS-UMMAs at 128 B/clk, plus
// the P tile write).  Here:
//   * one CTA owns 256 query rows (two 128-row tiles t = 0, 1) of one head,
//     so every K/V tile loaded by TMA feeds two query tiles;
//   * TMEM: tile t has S_t (128 fp32 cols) and O_t (128 cols); the softmax
//     writes P_t as packed bf16 over the first 64 columns of S_t, and
//     O_t += P_t V is a TS-UMMA (A from TMEM) — no P traffic in smem;
//   * the MMA warp interleaves  PV_0(j-1), S_0(j), PV_1(j-1), S_1(j): while
//     softmax warpgroup 0 works on S_0(j) the tensor core runs tile 1's work
//     and vice versa (ping-pong).  tcgen05 ops of one thread execute in
//     order, so when S_t(j) is complete PV_t(j-1) is complete too: the
//     softmax may rescale O_t in place without another barrier, and S_t(j)
//     may overwrite P_t(j-1).
// Warps: 0 TMA producer, 1 TMEM owner + UMMA issuer, 2-5 softmax tile 0,
// 6-9 softmax tile 1.
#include <math.h>

#include "errors.hpp"
#include "kernels.hpp"
#include "sm100.cuh"

#include <cstdlib>

namespace sp {
namespace {

constexpr int D = 128, BM = 128, BN = 128, NK = 3, NV = 2;
constexpr int kThreads = 320;
constexpr int kSlab = 128 * 64;

struct Params {
  int q_rows, total_kv, chunk_len, group, causal;
  float scale_log2;
  __nv_bfloat16* o;
  int64_t o_stride;
  float* lse;
  int chunk_row[SP_MAX_CHUNKS];
};

struct alignas(1024) Smem {
  __nv_bfloat16 q[2][BM * D];
  __nv_bfloat16 k[NK][BN * D];
  __nv_bfloat16 v[NV][BN * D];
};

struct Ctl {
  uint64_t q_full, k_full[NK], k_empty[NK], v_full[NV], v_empty[NV], s_full[2], p_full[2], o_done[2];
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

// D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

template <int kPolyEvery>  // 1 in 2*kPolyEvery exponentials on the FMA pipe (0: none)
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_d128_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ Params prm) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(16) Ctl ctl;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int block = gridDim.x - 1 - blockIdx.x;  // longest causal ranges first
  const int head = blockIdx.y;
  const int kvh = head / prm.group;
  const int row0 = block * 2 * BM;
  // KV tiles: tile 1 (rows row0+128..) needs n1 tiles, tile 0 needs n1-1 (causal)
  const int off = prm.total_kv - prm.q_rows;
  const int n1 = prm.causal ? (off + row0 + 2 * BM) / BN : prm.total_kv / BN;
  const int n0 = prm.causal ? n1 - 1 : n1;

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
    for (int t = 0; t < 2; ++t) {
      mbar_init(&ctl.s_full[t], 1);
      mbar_init(&ctl.p_full[t], 128);
      mbar_init(&ctl.o_done[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&ctl.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl.tmem_base;
  auto s_col = [&](int t) { return tmem + t * 256; };
  auto o_col = [&](int t) { return tmem + t * 256 + 128; };
  auto kv_row = [&](int j) {
    const int key = j * BN;
    return prm.chunk_row[key / prm.chunk_len] + key % prm.chunk_len;
  };

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&ctl.q_full, 2 * BM * D * 2);
      for (int t = 0; t < 2; ++t)
        for (int sl = 0; sl < 2; ++sl)
          tma_load_2d(sm.q[t] + sl * kSlab, &tm_q, &ctl.q_full, head * D + sl * 64, row0 + t * BM);
      int jk = 0, jv = 0;
      auto load_k = [&](int j) {
        const int s = j % NK;
        mbar_wait(&ctl.k_empty[s], ((j / NK) & 1) ^ 1);
        mbar_arrive_expect_tx(&ctl.k_full[s], BN * D * 2);
        for (int sl = 0; sl < 2; ++sl) tma_load_2d(sm.k[s] + sl * kSlab, &tm_k, &ctl.k_full[s], kvh * D + sl * 64, kv_row(j));
      };
      auto load_v = [&](int j) {
        const int s = j % NV;
        mbar_wait(&ctl.v_empty[s], ((j / NV) & 1) ^ 1);
        mbar_arrive_expect_tx(&ctl.v_full[s], BN * D * 2);
        for (int sl = 0; sl < 2; ++sl) tma_load_2d(sm.v[s] + sl * kSlab, &tm_v, &ctl.v_full[s], kvh * D + sl * 64, kv_row(j));
      };
      // K runs one tile ahead of V (S(j) is issued before PV(j))
      for (; jk < n1 && jk < 1; ++jk) load_k(jk);
      for (; jv < n1; ++jv) {
        if (jk < n1) load_k(jk++);
        load_v(jv);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = idesc_bf16_f32(BM, BN, false, false);
      constexpr uint32_t id_o = idesc_bf16_f32(BM, D, false, true);
      const uint32_t q_a[2] = {smem_u32(sm.q[0]), smem_u32(sm.q[1])};
      auto issue_s = [&](int t, int j) {
        const uint32_t k_a = smem_u32(sm.k[j % NK]);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t o = (kk / 4) * (kSlab * 2) + (kk % 4) * 32;
          umma_bf16_ss(s_col(t), smem_desc_sw128(q_a[t] + o, 16, 1024), smem_desc_sw128(k_a + o, 16, 1024), id_s,
                       kk > 0);
        }
        umma_commit(&ctl.s_full[t]);
      };
      auto issue_pv = [&](int t, int j, int pv_count) {
        const uint32_t v_a = smem_u32(sm.v[j % NV]);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          umma_bf16_ts(o_col(t), s_col(t) + kk * 8, smem_desc_sw128(v_a + kk * 16 * 128, kSlab * 2, 1024), id_o,
                       (pv_count > 0 || kk > 0) ? 1u : 0u);
      };
      mbar_wait(&ctl.q_full, 0);
      int p_seen[2] = {0, 0};  // P tiles consumed per query tile
      for (int j = 0; j <= n1; ++j) {
        const bool has_k = j < n1;
        if (has_k) {
          mbar_wait(&ctl.k_full[j % NK], (j / NK) & 1);
          tc_fence_after();
        }
        if (j > 0) mbar_wait(&ctl.v_full[(j - 1) % NV], ((j - 1) / NV) & 1);
        for (int t = 0; t < 2; ++t) {
          const int nt = t == 0 ? n0 : n1;
          if (j > 0 && j - 1 < nt) {  // O_t += P_t(j-1) V(j-1)
            mbar_wait(&ctl.p_full[t], p_seen[t] & 1);
            tc_fence_after();
            issue_pv(t, j - 1, p_seen[t]);
            ++p_seen[t];
            if (p_seen[t] == nt) umma_commit(&ctl.o_done[t]);
          }
          if (j < nt) issue_s(t, j);
        }
        if (j > 0) umma_commit(&ctl.v_empty[(j - 1) % NV]);
        if (has_k) umma_commit(&ctl.k_empty[j % NK]);
      }
    }
  } else {
    // ------------------------------------------------ softmax, one WG per query tile
    const int t = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const int nt = t == 0 ? n0 : n1;
    const int qrow = row0 + t * BM + r;
    const float sl2 = prm.scale_log2;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nt; ++j) {
      mbar_wait(&ctl.s_full[t], j & 1);
      tc_fence_after();
      // pass 1: row max (S stays in TMEM; re-read in pass 2 — TMEM reads are
      // cheap, registers are not: 10 warps cap the budget at 168/thread)
      const bool diag = prm.causal && j == nt - 1;
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        float sv[32];
        tmem_ld32(s_col(t) + lane_off + c * 32, sv);
        tmem_wait_ld();
#pragma unroll
        for (int x = 0; x < 32; ++x) mx = fmaxf(mx, (diag && c * 32 + x > r) ? -INFINITY : sv[x]);
      }
      const float cand = mx * sl2;
      const bool grow = cand > m_used + 8.0f;
      float corr = 1.f;
      if (grow) {
        corr = fast_exp2(m_used - cand);
        m_used = cand;
      }
      const float msub = m_used == -INFINITY ? 0.f : m_used;
      // O_t is stable here (PV_t(j-1) completed before S_t(j)): lazy rescale in place
      if (j > 0 && __any_sync(0xffffffffu, grow)) {
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          float ov[32];
          tmem_ld32(o_col(t) + lane_off + c * 32, ov);
          tmem_wait_ld();
#pragma unroll
          for (int x = 0; x < 32; ++x) ov[x] *= corr;
          tmem_st32(o_col(t) + lane_off + c * 32, ov);
        }
      }
      float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        float sv[32];
        tmem_ld32(s_col(t) + lane_off + h * 32, sv);
        tmem_wait_ld();
        if (diag) {
#pragma unroll
          for (int x = 0; x < 32; ++x)
            if (h * 32 + x > r) sv[x] = -INFINITY;
        }
        uint32_t pk[16];
#pragma unroll
        for (int x = 0; x < 16; ++x) {
          const float a = fast_exp2(fmaf(sv[2 * x], sl2, -msub));
          const float xb = fmaf(sv[2 * x + 1], sl2, -msub);
          // a share of the exponentials runs on the FMA pipe (MUFU is the
          // other bottleneck of the tile next to the tensor core)
          const float b = (kPolyEvery > 0 && x % (kPolyEvery > 0 ? kPolyEvery : 1) == 0) ? poly_exp2(xb) : fast_exp2(xb);
          rs0 += a;
          rs1 += b;
          pk[x] = pack_bf16(a, b);
        }
        tmem_st16(s_col(t) + lane_off + h * 16, pk);
      }
      const float rs = rs0 + rs1;
      l = l * corr + rs;
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&ctl.p_full[t]);
    }
    // epilogue
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow = prm.o + int64_t(qrow) * prm.o_stride + head * D;
    if (nt > 0) {
      mbar_wait(&ctl.o_done[t], 0);
      tc_fence_after();
    }
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float ov[32];
      if (nt > 0) {
        tmem_ld32(o_col(t) + lane_off + c * 32, ov);
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
    prm.lse[int64_t(head) * prm.q_rows + qrow] = l > 0.f ? (m_used + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
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
  auto kern = poly == 2 ? attn_fwd_d128_kernel<2> : poly == 4 ? attn_fwd_d128_kernel<4> : poly == 8 ? attn_fwd_d128_kernel<8> : attn_fwd_d128_kernel<0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return cuda_status(e, "attn_fwd_d128: set smem");
  kern<<<dim3(unsigned(q_rows / (2 * BM)), heads), kThreads, smem, st>>>(tq, tk, tv, prm);
  count_launch(1);
  return cuda_status(cudaGetLastError(), "attn_fwd_d128 launch");
}

}  // namespace sp
