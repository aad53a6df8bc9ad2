// K1 (head_dim 128): sliced causal attention forward, ping-pong with a
// shared S buffer.  Same semantics as attn_fwd.cu (reference
// chunk_attention, proj/src/attention.cpp:21-111: scale 1/sqrt(d),
// bottom-right causal, finalize O/l, plus the LSE).
//
// The round-1 predecessor kept S_A, S_B, O_A, O_B in TMEM with P written over
// S, so S_X(j+1) could only be computed after PV_X(j) had consumed P_X(j):
// every tile's softmax sat on a serial chain PV + S + softmax (~3.3K cycles
// per KV step of the CTA, measured).  Here the two tiles SHARE one S buffer and
// P gets its own columns:
//   TMEM: S [0,128) | P_A [128,192) P_B [192,256) (bf16, 2 keys/col) |
//         O_A [256,384) O_B [384,512)
// A softmax reads its S into registers (64 per thread, 112-register budget)
// and releases the buffer at once (s_free), so the next S (other tile or
// next KV tile) overlaps its max/exp work; P_X(j+1) waits only for PV_X(j)
// (pv_done).  The UMMA warp is a small dynamic scheduler over two in-order
// streams: S in the order A0 B0 A1 B1 ..., and PV_A / PV_B.
#include <math.h>


#include "errors.hpp"
#include "kernels.hpp"
#include "sm100.cuh"

namespace sp {
namespace {

constexpr int D = 128, BM = 128, BN = 128, NK = 2, NV = 2;
constexpr int kThreads = 640;  // 16 softmax warps + warpgroup 4 (producer, UMMA, 2 idle)
constexpr int kProducerWarp = 16, kMmaWarp = 17, kPvWarp = 18;
// registers: 96/thread at launch (640 threads); warpgroup 4 shrinks to 32 and
// the four softmax warpgroups grow to 112, enough to keep a 64-column S row
// half in registers across the max exchange (one TMEM read of S per tile).
// setmaxnreg sits at the top of each role's branch so ptxas never sees the
// softmax code reachable under the small budget.
constexpr int kRegsSide = 32, kRegsSoftmax = 112;
constexpr int kSlab = 128 * 64;  // elements of one [128 rows][64] SW128 slab

struct Params {
  int q_rows, total_kv, chunk_len, group, causal;
  int kv_valid;         // keys >= kv_valid are masked (padding)
  int64_t causal_off;   // causal: query row r sees keys <= r + causal_off
  float scale_log2;
  __nv_bfloat16* o;
  int64_t o_stride;
  float* lse;
  float* row_max;       // optional [heads][q_rows]: true row max of the scaled scores (natural log units)
  int chunk_row[SP_MAX_CHUNKS];
};

struct alignas(1024) Smem {
  __nv_bfloat16 q[2][BM * D];
  __nv_bfloat16 k[NK][BN * D];
  __nv_bfloat16 v[NV][BN * D];
};

struct Ctl {
  uint64_t q_full, k_full[NK], k_empty[NK], v_full[NV], v_empty[NV], s_full[2], s_free, p_full[2], pv_done[2];
  uint32_t tmem_base;
  float red_m[2][2][2][BM];  // [tile][tile parity][half][row]: partial row max
  float red_l[2][2][BM];     // [tile][half][row]: partial row sum (epilogue)
};

__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_ps_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ Params prm) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(16) Ctl ctl;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int pair = gridDim.x - 1 - blockIdx.x;  // longest causal ranges first
  const int head = blockIdx.y;
  const int kvh = head / prm.group;
  const int row0 = pair * 2 * BM;
  const bool has_b = row0 + BM < prm.q_rows;
  auto n_tiles = [&](int r0) {  // KV tiles holding a key visible to some row of [r0, r0 + BM)
    int64_t kmax = prm.kv_valid - 1;
    if (prm.causal) kmax = min(kmax, int64_t(r0) + BM - 1 + prm.causal_off);
    return kmax < 0 ? 0 : int(kmax / BN + 1);
  };
  const int n_a = n_tiles(row0);
  const int n_b = has_b ? n_tiles(row0 + BM) : 0;
  const int n = n_a > n_b ? n_a : n_b;  // K/V tiles the CTA streams

  if (warp == kProducerWarp && lane == 0) {
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
    for (int x = 0; x < 2; ++x) {
      mbar_init(&ctl.s_full[x], 1);
      mbar_init(&ctl.p_full[x], 256);
      mbar_init(&ctl.pv_done[x], 1);
    }
    mbar_init(&ctl.s_free, 256);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<512>(&ctl.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl.tmem_base;
  auto kv_row = [&](int j) {
    const int key = j * BN;
    return prm.chunk_row[key / prm.chunk_len] + key % prm.chunk_len;
  };

  if (warp >= 16) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegsSide));
  if (warp == kProducerWarp) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&ctl.q_full, (has_b ? 2 : 1) * BM * D * 2);
      for (int x = 0; x < (has_b ? 2 : 1); ++x)
        for (int sl = 0; sl < 2; ++sl)
          tma_load_2d(sm.q[x] + sl * kSlab, &tm_q, &ctl.q_full, head * D + sl * 64, row0 + x * BM);
      // consumption order: S_A(j), S_B(j) read K(j); PV_A(j), PV_B(j) read
      // V(j); S_X(j+1) follows PV_X(j), so K runs two tiles ahead of V.
      auto load_k = [&](int j) {
        const int s = j % NK;
        mbar_wait(&ctl.k_empty[s], ((j / NK) & 1) ^ 1);
        mbar_arrive_expect_tx(&ctl.k_full[s], BN * D * 2);
        for (int sl = 0; sl < 2; ++sl)
          tma_load_2d(sm.k[s] + sl * kSlab, &tm_k, &ctl.k_full[s], kvh * D + sl * 64, kv_row(j));
      };
      int jk = 0;
      for (; jk < n && jk < 2; ++jk) load_k(jk);
      for (int j = 0; j < n; ++j) {
        const int v = j % NV;
        mbar_wait(&ctl.v_empty[v], ((j / NV) & 1) ^ 1);
        mbar_arrive_expect_tx(&ctl.v_full[v], BN * D * 2);
        for (int sl = 0; sl < 2; ++sl)
          tma_load_2d(sm.v[v] + sl * kSlab, &tm_v, &ctl.v_full[v], kvh * D + sl * 64, kv_row(j));
        if (jk < n) load_k(jk++);
      }
    }
  } else if (warp == kMmaWarp || warp == kPvWarp) {
    // Two issuing warps (whole warp each; one elected lane issues): tcgen05
    // issue blocks for about the duration of the group it issues, so a single
    // issuer queues the S of one tile behind the PV of the other; with one
    // warp per stream the tensor pipe is fed from both.  Commits cover the
    // issuing warp's own MMAs, which is all each barrier needs.
    constexpr uint32_t id_s = idesc_bf16_f32(BM, BN, false, false);
    constexpr uint32_t id_o = idesc_bf16_f32(BM, D, false, true);
    mbar_wait(&ctl.q_full, 0);
    if (warp == kMmaWarp) {
      // S stream A0 B0 A1 B1 ... (B may have one more): the shared buffer is
      // free once the previous S has been read; K(j) is released after the
      // last S that reads it
      const int pairs = n_a < n_b ? n_a : n_b;
      const int n_s = n_a + n_b;
      for (int k = 0; k < n_s; ++k) {
        const int x = k < 2 * pairs ? (k & 1) : (n_a > n_b ? 0 : 1);
        const int j = k < 2 * pairs ? (k >> 1) : pairs + (k - 2 * pairs);
        if (k > 0) mbar_wait(&ctl.s_free, (k - 1) & 1);
        mbar_wait(&ctl.k_full[j % NK], (j / NK) & 1);
        tc_fence_after();
        umma_bf16_ss_k128(tmem, smem_desc_sw128(smem_u32(sm.q[x]), 16, 1024),
                          smem_desc_sw128(smem_u32(sm.k[j % NK]), 16, 1024), id_s, 0u);
        umma_commit_warp(&ctl.s_full[x]);
        if (x == 1 || j >= n_b) umma_commit_warp(&ctl.k_empty[j % NK]);
      }
    } else {
      // PV stream A0 B0 A1 B1 ...; V(j) released after the last PV reading it
      for (int j = 0; j < n; ++j) {
        mbar_wait(&ctl.v_full[j % NV], (j / NV) & 1);
        for (int x = 0; x < 2; ++x) {
          if (j >= (x ? n_b : n_a)) continue;
          mbar_wait(&ctl.p_full[x], j & 1);
          tc_fence_after();
          // keys [16kk, +16): P_X of half kk/4 at cols 128 + 64x + 32(kk/4) + 8(kk%4)
          umma_bf16_ts_k128(tmem + 256 + x * 128, tmem + 128 + x * 64, 32,
                            smem_desc_sw128(smem_u32(sm.v[j % NV]), kSlab * 2, 1024), id_o, j > 0 ? 1u : 0u);
          umma_commit_warp(&ctl.pv_done[x]);
        }
        umma_commit_warp(&ctl.v_empty[j % NV]);
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kRegsSoftmax));
    // ------------------------------- softmax: tile x, key half h, query row r
    const int x = warp >> 3;
    const int h = (warp >> 2) & 1;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int nt = x ? n_b : n_a;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const uint32_t s_col = tmem + h * 64 + lane_off;                 // shared S
    const uint32_t p_col = tmem + 128 + x * 64 + h * 32 + lane_off;  // own P
    const uint32_t o_col = tmem + 256 + x * 128 + h * 64 + lane_off;
    const float sl2 = prm.scale_log2;
    float m_used = -INFINITY, l = 0.f, m_true = -INFINITY;
    // last visible key of this thread's row, relative to its key half
    const int64_t qlim = prm.causal ? min(int64_t(prm.kv_valid) - 1, int64_t(row0 + x * BM + r) + prm.causal_off)
                                    : int64_t(prm.kv_valid) - 1;
    for (int j = 0; j < nt; ++j) {
      mbar_wait(&ctl.s_full[x], j & 1);
      tc_fence_after();
      const int64_t lim = qlim - int64_t(j) * BN - h * 64;  // columns e > lim of this half are masked
      // S row half -> registers once (both loads in flight together)
      float sv[64];
      tmem_ld32(s_col, *reinterpret_cast<float(*)[32]>(&sv[0]));
      tmem_ld32(s_col + 32, *reinterpret_cast<float(*)[32]>(&sv[32]));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&ctl.s_free);  // S buffer may take the next tile's scores
      if (lim < 63) {  // the diagonal tile (or padding): per-element mask
        const int lm = lim < -1 ? -1 : int(lim);
#pragma unroll
        for (int e = 0; e < 64; ++e)
          if (e > lm) sv[e] = -INFINITY;
      }
      float m8[8];
#pragma unroll
      for (int y = 0; y < 8; ++y) m8[y] = fmaxf(sv[y], sv[y + 8]);
#pragma unroll
      for (int e = 16; e < 64; e += 8)
#pragma unroll
        for (int y = 0; y < 8; ++y) m8[y] = fmaxf(m8[y], sv[e + y]);
      const float mh =
          fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      // row max shared by the two halves (slot parity j&1: the partner reads
      // slot j&1 before it can reach the barrier of tile j+1)
      ctl.red_m[x][j & 1][h][r] = mh;
      named_bar_sync(1 + x, 256);
      const float mx = fmaxf(mh, ctl.red_m[x][j & 1][h ^ 1][r]);
      m_true = fmaxf(m_true, mx);
      const float cand = mx * sl2;
      const bool grow = cand > m_used + 8.0f;  // identical decision in both halves
      float corr = 1.f;
      if (grow) {
        corr = fast_exp2(m_used - cand);  // 0 while m_used == -inf
        m_used = cand;
      }
      const float msub = m_used == -INFINITY ? 0.f : m_used;
      // O_X and P_X are ours again once PV_X(j-1) has completed
      if (j > 0) {
        mbar_wait(&ctl.pv_done[x], (j - 1) & 1);
        tc_fence_after();
      }
      if (j > 0 && __any_sync(0xffffffffu, grow)) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float ov[16];
          tmem_ld16(o_col + c * 16, ov);
          tmem_wait_ld_dep16(ov);
          uint32_t ow[16];
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const float2 y = fmul2(make_float2(ov[e], ov[e + 1]), make_float2(corr, corr));
            ow[e] = __float_as_uint(y.x);
            ow[e + 1] = __float_as_uint(y.y);
          }
          tmem_st16(o_col + c * 16, ow);
        }
      }
      float2 rs[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const float2 sl2x2 = make_float2(sl2, sl2), nmx2 = make_float2(-msub, -msub);
      // exponentials from registers; bf16 P_X (keys [64h+16q, +16) -> columns
      // p_col + 8q)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t pk[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int i = q * 16 + 2 * e;
          const float2 xx = ffma2(make_float2(sv[i], sv[i + 1]), sl2x2, nmx2);
          const float a = fast_exp2(xx.x);
          const float b = fast_exp2(xx.y);
          rs[e & 3] = fadd2(rs[e & 3], make_float2(a, b));
          pk[e] = pack_bf16(a, b);
        }
        tmem_st8(p_col + q * 8, pk);
      }
      const float2 rr = fadd2(fadd2(rs[0], rs[1]), fadd2(rs[2], rs[3]));
      l = l * corr + (rr.x + rr.y);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&ctl.p_full[x]);
    }
    // ------------------------------------------------------------- epilogue
    ctl.red_l[x][h][r] = l;
    named_bar_sync(1 + x, 256);
    const float lt = l + ctl.red_l[x][h ^ 1][r];
    const int qrow = row0 + x * BM + r;
    if (qrow < prm.q_rows) {
      if (nt > 0) {
        mbar_wait(&ctl.pv_done[x], (nt - 1) & 1);
        tc_fence_after();
      }
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      __nv_bfloat16* orow = prm.o + int64_t(qrow) * prm.o_stride + head * D + h * 64;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float ov[32];
        if (nt > 0) {
          tmem_ld32(o_col + c * 32, ov);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) ov[e] = 0.f;
        }
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          dst[q4] = make_uint4(pack_bf16(ov[8 * q4] * inv, ov[8 * q4 + 1] * inv),
                               pack_bf16(ov[8 * q4 + 2] * inv, ov[8 * q4 + 3] * inv),
                               pack_bf16(ov[8 * q4 + 4] * inv, ov[8 * q4 + 5] * inv),
                               pack_bf16(ov[8 * q4 + 6] * inv, ov[8 * q4 + 7] * inv));
      }
      if (h == 0) {
        prm.lse[int64_t(head) * prm.q_rows + qrow] =
            lt > 0.f ? (m_used + __log2f(lt)) * 0.69314718055994530942f : -INFINITY;
        if (prm.row_max)
          prm.row_max[int64_t(head) * prm.q_rows + qrow] =
              lt > 0.f ? m_true * prm.scale_log2 * 0.69314718055994530942f : -INFINITY;
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

int attn_fwd_d128_ps(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                     int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks, int chunk_len,
                     int heads, int kv_heads, const FwdMask& mk, void* o, int64_t o_stride, float* lse,
                     cudaStream_t st) {
  Params prm{};
  prm.q_rows = int(q_rows);
  prm.total_kv = n_chunks * chunk_len;
  prm.chunk_len = chunk_len;
  prm.group = heads / kv_heads;
  prm.causal = mk.causal;
  prm.kv_valid = int(mk.kv_valid);
  prm.causal_off = mk.causal_off;
  prm.scale_log2 = float(1.4426950408889634 * mk.scale);
  prm.o = static_cast<__nv_bfloat16*>(o);
  prm.o_stride = o_stride;
  prm.lse = lse;
  prm.row_max = mk.row_max;
  for (int c = 0; c < n_chunks; ++c) prm.chunk_row[c] = chunk_row[c];
  CUtensorMap tq, tk, tv;
  if (!make_tmap_bf16(&tq, q, uint64_t(q_stride), uint64_t(q_rows), uint64_t(q_stride), BM) ||
      !make_tmap_bf16(&tk, k_pool, uint64_t(kv_stride), uint64_t(pool_rows), uint64_t(kv_stride), BN) ||
      !make_tmap_bf16(&tv, v_pool, uint64_t(kv_stride), uint64_t(pool_rows), uint64_t(kv_stride), BN))
    return set_error(SP_ERR_CUDA, "attn_fwd_d128_ps: cuTensorMapEncodeTiled failed (alignment?)");
  const size_t smem = sizeof(Smem) + 1024;
  if (int rc = set_smem_once(reinterpret_cast<const void*>(attn_fwd_ps_kernel), smem, "attn_fwd_d128_ps: set smem"))
    return rc;
  const unsigned pairs = unsigned((q_rows + 2 * BM - 1) / (2 * BM));
  attn_fwd_ps_kernel<<<dim3(pairs, heads), kThreads, smem, st>>>(tq, tk, tv, prm);
  count_launch(1);
  return cuda_status(cudaGetLastError(), "attn_fwd_d128_ps launch");
}


// Force-load this file's kernels (cudaFuncGetAttributes) — see preload_kernels
int preload_attn_fwd_v4() {
  cudaFuncAttributes a;
  if (cudaError_t e = cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(attn_fwd_ps_kernel))) return cuda_status(e, "preload attn_fwd_ps_kernel");
  return SP_OK;
}
}  // namespace sp
