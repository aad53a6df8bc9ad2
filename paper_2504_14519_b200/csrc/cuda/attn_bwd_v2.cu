// K2 (head_dim 128): software-pipelined sliced attention backward, sm_100a.
//
// Same math and accumulation contract as attn_bwd.cu (see its header); this
// variant is the production path for d = 128 and is organised to keep the
// tensor pipe busy:
//   * TMEM holds TWO (S^T, dP^T) buffers (2 x 128 cols) + dV (128) + dK (128);
//     the MMA warp issues S/dP of pair j+1 before dV/dK/dQ of pair j, so the
//     element math of pair j+1 overlaps the accumulation MMAs of pair j.
//   * P^T and dS^T go back into TMEM (packed bf16 over the consumed S^T
//     columns): dV += P^T dO and dK += dS^T Q are TS-UMMAs (A from TMEM),
//     which keeps their A operands out of the shared-memory bandwidth this
//     kernel is bound by; dQ^T of pair j lands in its consumed dP^T columns.
//   * two compute warpgroups (8 warps) split every pair's 64 query columns;
//   * dQ leaves through TMA bulk reduce-add (cp.reduce.async.bulk.tensor
//     .add.f32) from an smem stage instead of per-thread global atomics; a
//     dedicated drain warpgroup does TMEM -> smem -> TMA, so the element-math
//     warps never wait on it (it was ~28% of their time per pair).
// Warps: 0 TMA producer, 1 TMEM owner + S/dP issuer, 2..9 element math,
// 10..13 dQ drain, 14 dQ/dV/dK issuer.
#include <math.h>

#include "errors.hpp"
#include "kernels.hpp"
#include "sm100.cuh"


namespace sp {
namespace {

constexpr int D = 128, BQ = 64, BK = 128;
// NWG element-math warpgroups (2: 32 query columns per thread, 4: 16); warps:
// 0 TMA producer, 1 TMEM owner + S/dP issuer, 2 .. 2+4*NWG-1 element math,
// then the 4 dQ drain warps and the dQ/dV/dK issuer
template <int NWG>
struct Roles {
  static constexpr int kEm0 = 2, kDrain0 = 2 + 4 * NWG, kIssueB = kDrain0 + 4;
  static constexpr int kThreads = 32 * (kIssueB + 1);
  static constexpr int kCompute = 128 * NWG;
};
constexpr int kDrain = 128;
constexpr int kSlabQ = BQ * 64, kSlabK = BK * 64;  // elements per slab

struct Params {
  int q_rows, total_kv, chunk_len, group, causal, n_qtiles;
  float scale, scale_log2;
  const float* lse2;
  const float* delta;
  void* dk;  // chunk accumulators: fp32, or bf16 with AccT = __nv_bfloat16
  void* dv;
  int64_t acc_stride;
  int chunk_row[SP_MAX_CHUNKS];
  int acc_row[SP_MAX_CHUNKS];
};

// NS: Q/dO ring depth; NDS: dS^T tiles (2 = element math of pair j never
// waits for the dQ MMA of pair j-1 to finish reading the previous tile)
// STQ: query rows of the dQ staging tile (64 = one TMA reduce per pair, 32 =
// two, in half the shared memory)
template <int NS, int NDS, int STQ>
struct alignas(1024) Smem {
  __nv_bfloat16 k[BK * D];
  __nv_bfloat16 v[BK * D];
  __nv_bfloat16 q[NS][BQ * D];
  __nv_bfloat16 dout[NS][BQ * D];
  __nv_bfloat16 ds[NDS][BK * BQ];
  float stage[STQ * D];  // dQ rows [q][d] on their way to the TMA reduce
};

template <int NS>
struct Ctl {  // statistics and barriers (after the operand tiles)
  float lse2[NS][BQ];
  float delta[NS][BQ];
  uint64_t kv_full, q_full[NS], q_empty[NS], sdp_full[2], pds_ready, pds_free, dq_full[2], dq_free[2], acc_free[2],
      acc_done;
  uint32_t tmem_base;
};

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int NS, int NDS, int STQ, bool kPad, int NWG, typename AccT>
__global__ void __launch_bounds__(Roles<NWG>::kThreads, 1)
    attn_bwd_d128_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                         const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                         const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ Params prm) {
  extern __shared__ uint8_t smem_raw[];
  using SmemT = Smem<NS, NDS, STQ>;
  static_assert(sizeof(SmemT) % 1024 == 0, "operand tiles stay 1024-aligned");
  // kPad: the launch added 1 KB to align the operand tiles; without it the
  // dynamic window must start 1 KB-aligned (it does when the kernel has no
  // static shared memory) — checked, never assumed
  uint8_t* base = kPad ? reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023))
                       : smem_raw;
  if (!kPad && (smem_u32(smem_raw) & 1023u)) __trap();
  auto& sm = *reinterpret_cast<SmemT*>(base);
  auto& ctl = *reinterpret_cast<Ctl<NS>*>(base + sizeof(SmemT));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int kt = blockIdx.x, kvh = blockIdx.y;
  const int key0 = kt * BK;
  const int off = prm.total_kv - prm.q_rows;
  int t_min = 0;
  if (prm.causal) {
    const int num = key0 - off - BQ + 1;
    t_min = num > 0 ? (num + BQ - 1) / BQ : 0;
  }
  const int per_head = prm.n_qtiles - t_min;
  const int n_pairs = per_head > 0 ? per_head * prm.group : 0;
  const int chunk = key0 / prm.chunk_len;
  const int kv_prow = prm.chunk_row[chunk] + key0 % prm.chunk_len;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    tma_prefetch(&tm_dq);
    mbar_init(&ctl.kv_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&ctl.q_full[s], 1);
      mbar_init(&ctl.q_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ctl.sdp_full[b], 1);
      mbar_init(&ctl.dq_full[b], 1);
      mbar_init(&ctl.dq_free[b], kDrain);
      mbar_init(&ctl.acc_free[b], 1);
    }
    mbar_init(&ctl.pds_ready, Roles<NWG>::kCompute);
    mbar_init(&ctl.pds_free, 1);
    mbar_init(&ctl.acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&ctl.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl.tmem_base;
  constexpr uint32_t kDV = 256, kDK = 384;

  auto pair_head = [&](int j) { return kvh * prm.group + j / per_head; };
  auto pair_row = [&](int j) { return (t_min + j % per_head) * BQ; };

  if (warp == 0) {
    if (lane == 0 && n_pairs > 0) {
      mbar_arrive_expect_tx(&ctl.kv_full, 2 * BK * D * 2);
      for (int sl = 0; sl < 2; ++sl) {
        tma_load_2d(sm.k + sl * kSlabK, &tm_k, &ctl.kv_full, kvh * D + sl * 64, kv_prow);
        tma_load_2d(sm.v + sl * kSlabK, &tm_v, &ctl.kv_full, kvh * D + sl * 64, kv_prow);
      }
      for (int j = 0; j < n_pairs; ++j) {
        const int s = j % NS, h = pair_head(j), qrow = pair_row(j);
        mbar_wait(&ctl.q_empty[s], ((j / NS) & 1) ^ 1);
        mbar_arrive_expect_tx(&ctl.q_full[s], 2 * BQ * D * 2 + 2 * BQ * 4);
        for (int sl = 0; sl < 2; ++sl) {
          tma_load_2d(sm.q[s] + sl * kSlabQ, &tm_q, &ctl.q_full[s], h * D + sl * 64, qrow);
          tma_load_2d(sm.dout[s] + sl * kSlabQ, &tm_do, &ctl.q_full[s], h * D + sl * 64, qrow);
        }
        bulk_load(ctl.lse2[s], prm.lse2 + int64_t(h) * prm.q_rows + qrow, BQ * 4, &ctl.q_full[s]);
        bulk_load(ctl.delta[s], prm.delta + int64_t(h) * prm.q_rows + qrow, BQ * 4, &ctl.q_full[s]);
      }
    }
  } else if (warp == 1 || warp == Roles<NWG>::kIssueB) {
    // Two issuing warps, each a whole warp with one elected lane per UMMA
    // (sm100.cuh *_w / umma_commit_warp): warp 1 issues S^T/dP^T, warp 14
    // dQ^T, dV, dK.  tcgen05 issue blocks for about the duration of the group
    // issued, so one issuer serialises the two streams; with two, S/dP of
    // pair j+1 runs while the accumulation MMAs of pair j wait for P/dS.
    // Commits cover the issuing warp's own MMAs.
    if (n_pairs > 0) {
      constexpr uint32_t id_s = idesc_bf16_f32(BK, BQ, false, false);  // K Q^T, V dO^T
      constexpr uint32_t id_acc = idesc_bf16_f32(BK, D, false, true);  // P^T dO, dS^T Q
      constexpr uint32_t id_dq = idesc_bf16_f32(D, BQ, true, true);    // K^T dS^T
      const uint32_t k_a = smem_u32(sm.k), v_a = smem_u32(sm.v);
      // descriptor bases; per-step offsets are added to the low word (address >> 4)
      const uint64_t dk_k = smem_desc_sw128(k_a, 16, 1024), dv_k = smem_desc_sw128(v_a, 16, 1024);
      const uint64_t dk_mn = smem_desc_sw128(k_a, kSlabK * 2, 1024);
      mbar_wait(&ctl.kv_full, 0);
      if (warp == 1) {
        for (int j = 0; j < n_pairs; ++j) {
          const int s = j % NS, b = j & 1;
          mbar_wait(&ctl.q_full[s], (j / NS) & 1);
          if (j >= 2) {  // buffer b: dQ(j-2) drained, dV/dK(j-2) done reading P/dS
            mbar_wait(&ctl.dq_free[b], ((j >> 1) - 1) & 1);
            mbar_wait(&ctl.acc_free[b], ((j >> 1) - 1) & 1);
          }
          tc_fence_after();
          const uint64_t dq_k = smem_desc_sw128(smem_u32(sm.q[s]), 16, 1024);
          const uint64_t ddo_k = smem_desc_sw128(smem_u32(sm.dout[s]), 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t oa = ((kk / 4) * (kSlabK * 2) + (kk % 4) * 32) >> 4;
            const uint32_t ob = ((kk / 4) * (kSlabQ * 2) + (kk % 4) * 32) >> 4;
            umma_bf16_ss_w(tmem + b * 128, dk_k + oa, dq_k + ob, id_s, kk > 0);
            umma_bf16_ss_w(tmem + b * 128 + 64, dv_k + oa, ddo_k + ob, id_s, kk > 0);
          }
          umma_commit_warp(&ctl.sdp_full[b]);
        }
      } else {
        for (int j = 0; j < n_pairs; ++j) {
          const int s = j % NS, b = j & 1;
          mbar_wait(&ctl.pds_ready, j & 1);
          tc_fence_after();
          const uint64_t dq_mn = smem_desc_sw128(smem_u32(sm.q[s]), kSlabQ * 2, 1024);
          const uint64_t dds_mn = smem_desc_sw128(smem_u32(sm.ds[NDS == 1 ? 0 : b]), kSlabK * 2, 1024);
          const uint64_t ddo_mn = smem_desc_sw128(smem_u32(sm.dout[s]), kSlabQ * 2, 1024);
          // dQ^T = K^T dS^T into pair j's (consumed) dP^T columns (K = 128 keys)
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint32_t ok = (kk * 16 * 128) >> 4;
            umma_bf16_ss_w(tmem + b * 128 + 64, dk_mn + ok, dds_mn + ok, id_dq, kk > 0);
          }
          umma_commit_warp(&ctl.dq_full[b]);
          // dV += P^T dO ; dK += dS^T Q   (K = BQ queries), A operands from TMEM:
          // WG w left P^T (packed bf16) at cols 32w+[0,16), dS^T at 32w+[16,32)
#pragma unroll
          for (int kk = 0; kk < BQ / 16; ++kk) {
            const uint32_t pcol = tmem + b * 128 + (kk >> 1) * 32 + (kk & 1) * 8;
            const uint32_t ob = (kk * 16 * 128) >> 4;
            umma_bf16_ts_w(tmem + kDV, pcol, ddo_mn + ob, id_acc, (j > 0 || kk > 0) ? 1u : 0u);
            umma_bf16_ts_w(tmem + kDK, pcol + 16, dq_mn + ob, id_acc, (j > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit_warp(&ctl.q_empty[s]);  // S/dP(j) of warp 1 completed before pds_ready(j)
          umma_commit_warp(&ctl.pds_free);
          umma_commit_warp(&ctl.acc_free[b]);
        }
        umma_commit_warp(&ctl.acc_done);
      }
    }
  } else if (warp < Roles<NWG>::kDrain0) {
    // --------------------------------------------- element math (NWG WGs)
    constexpr int CW = BQ / NWG;     // query columns of every pair per thread
    const int cw = warp - 2;
    const int wg = cw >> 2;          // column group of every pair
    const int quarter = warp & 3;    // TMEM lane quarter
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const int key_rel = key0 - off + r;
    const int c0 = wg * CW;
    // P^T of queries [16kk, +16) sits at column (kk/2)*32 + (kk%2)*8 of the
    // buffer, dS^T 16 columns further (the dV / dK TS-UMMA A layout)
    const uint32_t pcol = NWG == 2 ? uint32_t(wg * 32) : uint32_t((wg >> 1) * 32 + (wg & 1) * 8);

    for (int j = 0; j < n_pairs; ++j) {
      const int s = j % NS, b = j & 1;

      const int qrow0 = pair_row(j);
      const bool need_mask = prm.causal && (key0 + BK - 1 - off > qrow0);
      mbar_wait(&ctl.q_full[s], (j / NS) & 1);
      mbar_wait(&ctl.sdp_full[b], (j >> 1) & 1);
      tc_fence_after();
      float sv[CW], dp[CW];
      if constexpr (CW == 32) {
        tmem_ld32(tmem + lane_off + b * 128 + c0, sv);
        tmem_ld32(tmem + lane_off + b * 128 + 64 + c0, dp);
      } else {
        tmem_ld16(tmem + lane_off + b * 128 + c0, sv);
        tmem_ld16(tmem + lane_off + b * 128 + 64 + c0, dp);
      }
      tmem_wait_ld();
      // P = exp2(S*scale*log2e - lse2), dS = P * (dP - delta) * scale on
      // packed fp32x2 (FFMA2/FMUL2); statistics come from smem 8 columns at a
      // time with 128-bit loads (they are uniform across the warp)
      uint32_t pk[CW / 2], dk[CW / 2];
      // per-query statistics: one coalesced load per warp (lane i holds column
      // c0+i), then warp shuffles -- a broadcast LDS.128 per 4 columns cost 4
      // shared-memory wavefronts and was ~20 % of this kernel's smem traffic
      const float my_nl = -ctl.lse2[s][c0 + (lane % CW)];
      const float my_nd = -ctl.delta[s][c0 + (lane % CW)] * prm.scale;
      const float2 sl2x2 = make_float2(prm.scale_log2, prm.scale_log2);
      const float2 scx2 = make_float2(prm.scale, prm.scale);
#pragma unroll
      for (int x = 0; x < CW; x += 2) {
        const float2 nl = make_float2(__shfl_sync(0xffffffffu, my_nl, x), __shfl_sync(0xffffffffu, my_nl, x + 1));
        const float2 nd = make_float2(__shfl_sync(0xffffffffu, my_nd, x), __shfl_sync(0xffffffffu, my_nd, x + 1));
        const float2 t = ffma2(make_float2(sv[x], sv[x + 1]), sl2x2, nl);
        float p0 = fast_exp2(t.x), p1 = fast_exp2(t.y);
        if (need_mask) {
          if (key_rel > qrow0 + c0 + x) p0 = 0.f;
          if (key_rel > qrow0 + c0 + x + 1) p1 = 0.f;
        }
        const float2 u = ffma2(make_float2(dp[x], dp[x + 1]), scx2, nd);
        const float2 dd = fmul2(u, make_float2(p0, p1));
        pk[x / 2] = pack_bf16(p0, p1);
        dk[x / 2] = pack_bf16(dd.x, dd.y);
      }
      if (NDS == 1 && j > 0) mbar_wait(&ctl.pds_free, (j - 1) & 1);
      const uint32_t ds_a = smem_u32(sm.ds[NDS == 1 ? 0 : b]);
      // P^T / dS^T (packed bf16) over this WG's own S^T columns: A operands of
      // the dV / dK TS-UMMAs; dS^T also to smem: B operand of dQ^T = K^T dS^T.
      if constexpr (CW == 32) {
        tmem_st16(tmem + lane_off + b * 128 + pcol, pk);
        tmem_st16(tmem + lane_off + b * 128 + pcol + 16, dk);
      } else {
        tmem_st8(tmem + lane_off + b * 128 + pcol, pk);
        tmem_st8(tmem + lane_off + b * 128 + pcol + 16, dk);
      }
#pragma unroll
      for (int g = 0; g < CW / 8; ++g)
        st_shared_v4(ds_a + sw128_offset(r, c0 + g * 8), dk[4 * g], dk[4 * g + 1], dk[4 * g + 2], dk[4 * g + 3]);
      tmem_wait_st();
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(&ctl.pds_ready);

    }
    if (n_pairs > 0) {
      // dK / dV (lane r = key, 128 cols each) += into the fp32 chunk accumulators
      mbar_wait(&ctl.acc_done, 0);
      tc_fence_after();
      const int64_t arow = prm.acc_row[chunk] + key0 % prm.chunk_len + r;
      // WG halves: dK then dV; with 4 WGs each takes 64 of the 128 columns
      const bool is_k = wg < NWG / 2;
      const int c_base = NWG == 2 ? 0 : (wg % 2) * 64;
      AccT* dst = static_cast<AccT*>(is_k ? prm.dk : prm.dv) + arow * prm.acc_stride + kvh * D + c_base;
      const uint32_t col = (is_k ? kDK : kDV) + c_base;
#pragma unroll
      for (int ch = 0; ch < D / 32 / (NWG / 2); ++ch) {
        float a[32];
        tmem_ld32(tmem + lane_off + col + ch * 32, a);
        tmem_wait_ld();
        acc_add32(dst + ch * 32, a);
      }
    }
    tc_fence_before();
  } else if (warp < Roles<NWG>::kIssueB) {
    // --------------------------------------------- dQ drain (one warpgroup)
    // dQ^T of pair jj sits in its consumed dP^T columns (lane = head dim d,
    // columns = the pair's 64 queries): TMEM -> registers (frees the columns
    // for the S/dP of pair jj+2) -> smem stage [q][d] -> TMA reduce-add.
    const int quarter = warp & 3;
    const int d = quarter * 32 + lane;
    const int dtid = (warp - Roles<NWG>::kDrain0) * 32 + lane;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    for (int jj = 0; jj < n_pairs; ++jj) {
      const int bb = jj & 1;
      mbar_wait(&ctl.dq_full[bb], (jj >> 1) & 1);
      tc_fence_after();
      float a0[32], a1[32];
      tmem_ld32(tmem + lane_off + bb * 128 + 64, a0);
      tmem_ld32(tmem + lane_off + bb * 128 + 96, a1);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&ctl.dq_free[bb]);
      // [q][d] rows of the stage, STQ queries per TMA reduce (a0: queries
      // 0..31, a1: 32..63 of the pair)
      auto stage_rows = [&](const float(&lo)[32], const float(&hi)[32], int q0) {
        if (dtid == 0) bulk_wait_read<0>();  // the previous reduce has read the stage
        named_bar_sync(1, kDrain);
        const uint32_t st = smem_u32(sm.stage) + uint32_t(d) * 4u;
#pragma unroll
        for (int x = 0; x < 32; ++x) {
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(st + x * D * 4), "f"(lo[x]) : "memory");
          if (STQ == 64) asm volatile("st.shared.f32 [%0], %1;" ::"r"(st + (32 + x) * D * 4), "f"(hi[x]) : "memory");
        }
        fence_async_smem();
        named_bar_sync(2, kDrain);
        if (dtid == 0) {
          tma_reduce_add_2d(&tm_dq, sm.stage, pair_head(jj) * D, pair_row(jj) + q0);
          bulk_commit();
        }
      };
      if (STQ == 64) {
        stage_rows(a0, a1, 0);
      } else {
        stage_rows(a0, a0, 0);
        stage_rows(a1, a1, 32);
      }
    }
    if (dtid == 0) bulk_wait<0>();
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

// Launch the d=128 backward (lse2/delta already prepared by attn_bwd_prep).
int attn_bwd_d128(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                  int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks, int chunk_len,
                  int heads, int kv_heads, int causal, const void* dout, int64_t do_stride, const float* lse2,
                  const float* delta, float* dq_acc, void* dk_acc, void* dv_acc, int64_t acc_rows,
                  const int32_t* acc_row, bool acc_bf16, cudaStream_t st) {
  Params prm{};
  prm.q_rows = int(q_rows);
  prm.total_kv = n_chunks * chunk_len;
  prm.chunk_len = chunk_len;
  prm.group = heads / kv_heads;
  prm.causal = causal;
  prm.n_qtiles = int(q_rows / BQ);
  prm.scale = float(1.0 / sqrt(double(D)));
  prm.scale_log2 = float(1.4426950408889634 / sqrt(double(D)));
  prm.lse2 = lse2;
  prm.delta = delta;
  prm.dk = dk_acc;
  prm.dv = dv_acc;
  prm.acc_stride = int64_t(kv_heads) * D;
  for (int c = 0; c < n_chunks; ++c) {
    prm.chunk_row[c] = chunk_row[c];
    prm.acc_row[c] = acc_row[c];
  }
  // NS = 3 Q/dO stages, one dS tile, 64-row dQ stage: measured best
  // (scripts/k2_ab.py, profiles/r02_k2_ab.json): NS = 2 costs 11-12 %, a 32-row
  // dQ stage (two reduces per pair, what NS = 4 needs to fit 227 KB) 10-13 %,
  // a second dS tile +1 % at most
  constexpr int kNS = 3, kNDS = 1, kSTQ = 64;
  const int stq = kSTQ;
  CUtensorMap tq, tdo, tk, tv, tdq;
  if (!make_tmap_bf16(&tq, q, uint64_t(q_stride), uint64_t(q_rows), uint64_t(q_stride), BQ) ||
      !make_tmap_bf16(&tdo, dout, uint64_t(do_stride), uint64_t(q_rows), uint64_t(do_stride), BQ) ||
      !make_tmap_bf16(&tk, k_pool, uint64_t(kv_stride), uint64_t(pool_rows), uint64_t(kv_stride), BK) ||
      !make_tmap_bf16(&tv, v_pool, uint64_t(kv_stride), uint64_t(pool_rows), uint64_t(kv_stride), BK) ||
      !make_tmap_f32(&tdq, dq_acc, uint64_t(heads) * D, uint64_t(q_rows), uint64_t(heads) * D, D, uint32_t(stq)))
    return set_error(SP_ERR_CUDA, "attn_bwd_d128: cuTensorMapEncodeTiled failed (alignment?)");
  // two element-math warpgroups: four (16 query columns per thread, 736
  // threads) measured 1-3 % slower (profiles/r02_k2_ab.json) — the element
  // math is not what bounds K2
  constexpr int kNWG = 2;
  const size_t smem = sizeof(Smem<kNS, kNDS, kSTQ>) + sizeof(Ctl<kNS>) + 1024;
  auto launch = [&](auto kern) -> int {
    if (int rc = set_smem_once(reinterpret_cast<const void*>(kern), smem, "attn_bwd_d128: set smem")) return rc;
    kern<<<dim3(prm.total_kv / BK, kv_heads), Roles<kNWG>::kThreads, smem, st>>>(tq, tdo, tk, tv, tdq, prm);
    count_launch(1);
    return SP_OK;
  };
  const int rc = acc_bf16 ? launch(attn_bwd_d128_kernel<kNS, kNDS, kSTQ, true, kNWG, __nv_bfloat16>)
                          : launch(attn_bwd_d128_kernel<kNS, kNDS, kSTQ, true, kNWG, float>);
  if (rc) return rc;
  return cuda_status(cudaGetLastError(), "attn_bwd_d128 launch");
}


// Force-load this file's kernels (cudaFuncGetAttributes) — see preload_kernels
int preload_attn_bwd_v2() {
  cudaFuncAttributes a;
  for (const void* k : {reinterpret_cast<const void*>(attn_bwd_d128_kernel<3, 1, 64, true, 2, float>),
                        reinterpret_cast<const void*>(attn_bwd_d128_kernel<3, 1, 64, true, 2, __nv_bfloat16>)})
    if (cudaError_t e = cudaFuncGetAttributes(&a, k)) return cuda_status(e, "preload attn_bwd_d128_kernel");
  return SP_OK;
}
}  // namespace sp
