// The B200 sliced-1F1B step executor: one process (rank) per GPU owning
// pipeline stages s = rank + 1 + c*p, c < v (reference stage_owner,
// schedule.cpp:158-164; v > 1 is interleaved SlimPipe, the stage links then
// form a ring and the last device sends stage c*p+p's output to device 0).
//
// It walks device_order[rank] of gen_slimpipe (bit-exact host planning) and
// executes each pass on the GPU:
//   F(k,i,s):  acquire an arena slot (reference ledger simulator.cpp:324-327),
//              stage input = embedding (s=1) or NCCL recv from s-1; for every
//              layer: RMSNorm -> QKV GEMM -> RoPE (K/V written into the slot's
//              rows of the layer's KV pool) -> K1 sliced attention over the
//              slots of slices 1..i -> O GEMM + residual -> RMSNorm -> gate/up
//              GEMM -> SwiGLU -> down GEMM + residual; send to s+1.
//   BW(k,i,s): recompute of the stage from the stashed input — every op but
//              K1, whose O/LSE the forward stashed in the slot (selective;
//              cfg.recompute = 1: full, K1 again, reference Full
//              checkpointing workload.cpp:100-104), then the layer
//              backward in reverse with K2 accumulating dK/dV of chunks 1..i
//              into fp32 chunk accumulators (complete for chunk i now, since
//              slices n..i+1 ran before: schedule.cpp:125-126), LM head + loss
//              on the last stage, embedding grad on the first; send dX to s-1;
//              release the slot (simulator.cpp:328-331).
// Streams: compute, comm_fwd (activations s->s+1), comm_bwd (gradients
// s->s-1); each direction has its own NCCL communicator so the two never
// block each other.  CUDA events order buffers between the streams.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "errors.hpp"
#include "kernels.hpp"
#include "pipelab/schedule.hpp"
#include "pipelab/simulator.hpp"
#include "slimpipe.h"
#include "transport.hpp"
#include "xplan.hpp"

namespace sp {
namespace {

#define SP_TRY(expr)           \
  do {                         \
    int rc_ = (expr);          \
    if (rc_ != SP_OK) return rc_; \
  } while (0)

#define SP_CUDA(expr) SP_TRY(cuda_status((expr), #expr))

int nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return SP_OK;
  return set_error(SP_ERR_NCCL, "%s: %s", what, ncclGetErrorString(r));
}
#define SP_NCCL(expr) SP_TRY(nccl_status((expr), #expr))

using bf16raw = uint16_t;

struct LayerParams {
  int64_t attn_norm, wqkv, wo, mlp_norm, wgu, wd;
};

struct LayerWs {
  bf16raw *x_in, *xn, *q, *o, *x_mid, *xn2, *gu, *act;
  float *lse, *rstd1, *rstd2;
  bf16raw* o_ws;  // workspace O/LSE (full recompute); o/lse point at the slot's stash otherwise
  float* lse_ws;
};

struct PassTime {
  int pass;
  cudaEvent_t start, end;
};

struct AttnTimer {
  cudaEvent_t a, b;
  double flops;
  int kind;  // 0 fwd, 1 bwd
};

class Runtime {
 public:
  sp_model_config cfg{};
  int rank = 0, p = 1, stage = 1, Lps = 1;  // stage: the current pass's (global) stage
  int v = 1, nst = 1, cur = 0, lbase = 0;   // stages per device, total stages, pass's local chunk, its first layer
  bool first_dev = true, last_dev = true;   // owns stage 1 / stage nst
  // stage receives wait for the compute stream to reach their pass instead
  // of being posted as soon as a ring buffer frees: an NCCL receive kernel
  // spins on its SMs until the data arrives, and early posts kept one
  // spinning per direction for most of the step (measured c2 PP=4:
  // 75.2K -> 78.4K tokens/s).  SP_JIT_RECV=0 restores early posts.
  bool jit_recv = [] {
    const char* e = std::getenv("SP_JIT_RECV");
    return !(e && e[0] == '0');
  }();
  // exchange serves post their receives when the receiving pass starts on
  // this rank's compute stream instead of as soon as the exchange stream
  // reaches them: an NCCL receive kernel spins on its SMs until the sender's
  // data arrives, and a serve queued from the host's run-ahead would spin
  // for most of the step (SP_XSERVE_JIT=0 restores the early post)
  bool xserve_jit = [] {
    const char* e = std::getenv("SP_XSERVE_JIT");
    return !(e && e[0] == '0');
  }();
  int64_t Ls = 0, h = 0, H = 0, qd = 0, kvd = 0, qkv_w = 0;
  pipelab::Schedule sched;
  std::vector<pipelab::PassId> order;
  pipelab::MemoryLedger ledger;

  // parameters (flat)
  int64_t n_params = 0;
  bf16raw* w = nullptr;
  float *master = nullptr, *grad = nullptr, *adam_m = nullptr, *adam_v = nullptr;
  std::vector<LayerParams> lp;
  int64_t emb = -1, final_norm = -1, head = -1;
  int opt_step = 0;

  // ---- vocabulary parallelism (reference place_vocab,
  // simulator.cpp:414-522): every stage holds vocab rows [v0, v0+Vs) of the
  // LM head; per slice, VocabForward broadcasts the last stage's final hidden
  // state and all-reduces the shard softmax statistics, VocabBackward turns
  // them into the shard's dlogits, dW_head and a partial dX reduced onto the
  // last stage.  The collectives run on the world communicator in the order
  // place_vocab puts the vocab passes (identical on every rank).
  bool vp = false;
  int64_t Vs = 0, v0 = 0;
  cudaStream_t s_vocab = nullptr;
  struct VSlot {
    bf16raw* xf = nullptr;  // [Ls, h] final hidden state of the slice
    float* st = nullptr;    // [4][Ls]: local max, global max, Z, T
  };
  std::vector<VSlot> vslots;
  std::vector<int> vfree;
  std::map<std::pair<int, int>, int> vslot_of;
  float *vlogits = nullptr, *vdxf = nullptr;
  bf16raw* vdlog = nullptr;

  // arena: x stash + per-layer K/V pools, `slots` slice-sized slots
  int slots = 0;
  bf16raw* x_pool = nullptr;
  std::vector<bf16raw*> k_pool, v_pool;
  bool stash = true;                // selective recompute: attention O/LSE live in the slot
  std::vector<bf16raw*> o_pool;     // [slots*Ls][qd] per layer
  std::vector<float*> lse_pool;     // [slots][heads][Ls] per layer
  std::vector<int> free_slots;
  std::map<std::pair<int, int>, int> slot_of;
  // activation offload (cfg.offload): a slot's stage input and per-layer O/LSE
  // live in pinned host memory between its F and BW; one device staging set
  // (x_stage, o_stage/l_stage per layer) serves the pass that runs
  bool offload = false;
  bf16raw *hx = nullptr, *ho = nullptr, *x_stage = nullptr;
  float* hl = nullptr;
  std::vector<bf16raw*> o_stage;
  std::vector<float*> l_stage;
  cudaStream_t s_off = nullptr;
  cudaEvent_t ev_x_off = nullptr, ev_x_in = nullptr;
  std::vector<cudaEvent_t> ev_o_off, ev_o_in;
  size_t offload_bytes = 0;
  int slots_in_use = 0, slots_high_water = 0;
  // fp32 dK/dV chunk accumulators (one microbatch, indexed by slice)
  std::vector<void*> dk_acc, dv_acc;  // fp32, or bf16 with cfg.dkv_bf16
  bool dkv_bf16 = false;
  int64_t acc_es = 4;  // accumulator element size
  void* acc_at(void* base, int64_t elems) const { return static_cast<char*>(base) + elems * acc_es; }

  // workspaces
  std::vector<LayerWs> ws;
  bf16raw *x_final = nullptr, *qkv = nullptr, *dqkv = nullptr, *tmp_h = nullptr, *tmp_H = nullptr,
          *tmp_2H = nullptr, *xf = nullptr, *dlogits = nullptr;
  bf16raw* out_buf[2] = {nullptr, nullptr};  // stage outputs (send to s+1)
  bf16raw* gin_buf[2] = {nullptr, nullptr};  // gradients received from s+1
  bf16raw* gout_buf[2] = {nullptr, nullptr}; // gradients sent to s-1 (dx)
  float *rope_cos = nullptr, *rope_sin = nullptr;  // [seq_len][d/2]
  float* norm_ws = nullptr;  // per-block RMSNorm dW partials (deterministic weight gradient)
  int32_t *h_tok = nullptr, *h_tgt = nullptr;  // pinned staging of host inputs
  float* h_loss = nullptr;
  cudaEvent_t ev_staged = nullptr;
  float *dq_acc = nullptr, *delta_ws = nullptr, *logits = nullptr, *rstd_f = nullptr, *loss_dev = nullptr;
  int32_t *tokens = nullptr, *targets = nullptr;

  int device = 0;  // the runtime's GPU: every entry point makes it current (callers may be other threads)
  cudaStream_t comp = nullptr;
  ncclComm_t nc_fwd = nullptr, nc_bwd = nullptr;
  // Stage links: one 2-rank communicator and one stream per (neighbour,
  // direction), split from nc_fwd / nc_bwd, so a send to a busy neighbour
  // never blocks a receive from the other one (no head-of-line blocking).
  // Comm ranks inside a link: lower stage = 0, higher stage = 1.
  std::unique_ptr<Link> l_act_in, l_act_out, l_grad_in, l_grad_out;
  std::unique_ptr<Link> vlink;  // world communicator of the vocabulary collectives
  LoopWorld* loop = nullptr;    // single-GPU loopback world (transport.hpp), or NCCL when null
  cudaStream_t s_act_in = nullptr, s_act_out = nullptr, s_grad_in = nullptr, s_grad_out = nullptr;
  bf16raw* ain_buf[2] = {nullptr, nullptr};  // activations received from s-1 (ring)
  cudaEvent_t ev_ain_free[2]{};
  int ain_idx = 0;
  cudaEvent_t ev_out_free[2]{}, ev_gin_free[2]{}, ev_gout_free[2]{};
  int out_idx = 0, gin_idx = 0, gout_idx = 0;
  std::vector<PassTime> times;
  std::vector<AttnTimer> attn_times;
  // Event pools, created once and re-recorded every step: timing events
  // (pass spans, attention and stage-send timers) in `tpool`, handed out in
  // order from index 0 each step; `xev` is the one sync-only event behind
  // link() and the stream hand-offs (a wait captures the event's state when
  // it is enqueued, so re-recording it at once is safe).
  std::vector<cudaEvent_t> tpool;
  size_t tpool_i = 0;
  cudaEvent_t xev = nullptr;
  struct CommTimer {
    cudaEvent_t a, b;
    int64_t bytes;
  };
  std::vector<CommTimer> comm_times;  // stage sends of the last step

  // ---- attention workload redistribution (reference exchange.cpp /
  // simulator.cpp:56-108): per-pass transfer lists of this rank, two classes
  // (0: forward ticks, 1: backward ticks) each with its own NCCL
  // communicator, copy stream and high-priority remote-compute stream.
  std::map<int, PassX> xplan;
  pipelab::ExchangeAnnotation ann;
  std::unique_ptr<Link> lx[2];
  cudaStream_t cx[2] = {nullptr, nullptr}, rx[2] = {nullptr, nullptr};
  int x_tout = 0, x_cout = 0, x_tin = 0, x_cin = 0;  // per-class maxima (both classes)
  struct XBuf {
    bf16raw *o_rem = nullptr, *rq = nullptr, *rdo = nullptr, *ro = nullptr, *rk = nullptr, *rv = nullptr;
    float *lse_rem = nullptr, *dq_rem = nullptr, *dk_rem = nullptr, *dv_rem = nullptr;
    float *rlse = nullptr, *rstats = nullptr, *rdq = nullptr, *rdk = nullptr, *rdv = nullptr;
  } xb[2];
  int64_t x_bytes_sent = 0;
  cudaEvent_t step_start = nullptr, step_end = nullptr;
  std::atomic<int> enq_pos{-1};  // diagnostics: pass (index in order) the host is enqueuing, -1 idle
  size_t bytes_allocated = 0;
  std::vector<void*> allocations;

  ~Runtime() {
    if (comp) cudaStreamSynchronize(comp);
    destroy_links();
    for (void* a : allocations) cudaFree(a);
    for (cudaEvent_t e : tpool) cudaEventDestroy(e);
    if (xev) cudaEventDestroy(xev);
    if (ev_staged) cudaEventDestroy(ev_staged);
    for (void* hp : {static_cast<void*>(h_tok), static_cast<void*>(h_tgt), static_cast<void*>(h_loss),
                     static_cast<void*>(hx), static_cast<void*>(ho), static_cast<void*>(hl)})
      if (hp) cudaFreeHost(hp);
    for (cudaEvent_t e : {ev_x_off, ev_x_in})
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_o_off) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_o_in) cudaEventDestroy(e);
  }

  // Communicators are torn down in one global order, like warm_links sets
  // them up: NCCL's destroy of a communicator finalizes it with its peers, so
  // two ranks destroying shared communicators in different orders (the ring
  // of v > 1: rank 0 holds the wrap link as its *input*, rank p-1 as its
  // output) wait on each other forever.
  void destroy_links() {
    const bool ring = v > 1;
    std::vector<std::pair<int, int>> mine;
    const int prev_link = first_dev ? (ring ? p - 1 : -1) : rank - 1;
    const int next_link = (!last_dev || ring) ? rank : -1;
    if (prev_link >= 0) mine.emplace_back(prev_link, 0);
    if (next_link >= 0) mine.emplace_back(next_link, 1);
    std::sort(mine.begin(), mine.end());
    for (const auto& lk : mine) {
      if (lk.second == 0) {
        l_act_in.reset();
        l_grad_out.reset();
      } else {
        l_act_out.reset();
        l_grad_in.reset();
      }
    }
    lx[0].reset();
    lx[1].reset();
    vlink.reset();
    if (nc_fwd) ncclCommDestroy(nc_fwd);
    if (nc_bwd) ncclCommDestroy(nc_bwd);
    nc_fwd = nc_bwd = nullptr;
  }

  int timing_event(cudaEvent_t* e) {
    if (tpool_i == tpool.size()) {
      cudaEvent_t ne;
      SP_CUDA(cudaEventCreate(&ne));
      tpool.push_back(ne);
    }
    *e = tpool[tpool_i++];
    return SP_OK;
  }
  // `to` waits for everything enqueued on `from` so far
  int hand_off(cudaStream_t from, cudaStream_t to) {
    SP_CUDA(cudaEventRecord(xev, from));
    SP_CUDA(cudaStreamWaitEvent(to, xev, 0));
    return SP_OK;
  }

  template <class T>
  int alloc(T** ptr, int64_t count) {
    void* raw = nullptr;
    const size_t bytes = size_t(std::max<int64_t>(count, 1)) * sizeof(T);
    SP_CUDA(cudaMalloc(&raw, bytes));
    allocations.push_back(raw);
    bytes_allocated += bytes;
    *ptr = static_cast<T*>(raw);
    return SP_OK;
  }

  bf16raw* W(int64_t off) { return w + off; }
  // arena slot key of slice (k, j) at the current pass's local chunk
  std::pair<int, int> sk(int k, int j) const { return {k, (cur << 20) | j}; }
  float* G(int64_t off) { return grad + off; }

  int init(const sp_model_config& c, const void* ids, LoopWorld* lw = nullptr) {
    cfg = c;
    loop = lw;
    rank = c.rank;
    p = c.pp;
    stage = rank + 1;
    v = c.interleave <= 0 ? 1 : c.interleave;
    nst = p * v;
    first_dev = rank == 0;
    last_dev = rank == p - 1;
    if (v > 1 && (p < 2 || p % 2))
      return set_error(SP_ERR_UNSUPPORTED, "interleave > 1 needs an even pp >= 2 (stage ring links)");
    if (v > 1 && (c.exchange_mode != 0 || c.vocab_parallel))
      return set_error(SP_ERR_UNSUPPORTED, "interleave > 1 runs with exchange off and vocab_parallel 0");
    // the exchange serves peers on the same per-class stream as its own
    // requests; with the vocabulary collectives holding every rank's compute
    // stream at the same pass, a served partial can queue behind a request
    // that waits on that pass (measured: PP=4 stall) — not combined
    if (c.exchange_min_chunks < 0 || c.exchange_skip_last < 0 || c.exchange_skip_last > 1)
      return set_error(SP_ERR_INVALID, "exchange_min_chunks must be >= 0 and exchange_skip_last 0 or 1");
    if (c.vocab_parallel && c.exchange_mode != 0 && c.pp > 1)
      return set_error(SP_ERR_UNSUPPORTED, "vocab_parallel runs with exchange off");
    if (c.layers % nst) return set_error(SP_ERR_INVALID, "layers (%d) must divide by pp*v (%d)", c.layers, nst);
    if (c.seq_len % c.slices) return set_error(SP_ERR_INVALID, "run: seq_len must be divisible by slices");
    if (c.hidden != c.heads * c.head_dim) return set_error(SP_ERR_INVALID, "hidden != heads * head_dim");
    Lps = c.layers / nst;
    Ls = c.seq_len / c.slices;
    if (c.recompute < 0 || c.recompute > 2) return set_error(SP_ERR_INVALID, "recompute must be 0, 1 or 2");
    stash = c.recompute != 1;  // 2 (auto) is settled in alloc_arena once the parameters are resident
    if (c.offload < 0 || c.offload > 1) return set_error(SP_ERR_INVALID, "offload must be 0 or 1");
    offload = c.offload == 1;
    if (c.dkv_bf16 < 0 || c.dkv_bf16 > 1) return set_error(SP_ERR_INVALID, "dkv_bf16 must be 0 or 1");
    dkv_bf16 = c.dkv_bf16 == 1;
    acc_es = dkv_bf16 ? 2 : 4;
    h = c.hidden;
    H = c.ffn_hidden;
    qd = int64_t(c.heads) * c.head_dim;
    kvd = int64_t(c.kv_heads) * c.head_dim;
    qkv_w = qd + 2 * kvd;
    if (Ls % 128) return set_error(SP_ERR_UNSUPPORTED, "slice length must be a multiple of 128");
    if (c.slices > SP_MAX_CHUNKS)  // the attention kernels carry one chunk-table entry per slice
      return set_error(SP_ERR_UNSUPPORTED, "slices (%d) above SP_MAX_CHUNKS (%d)", c.slices, SP_MAX_CHUNKS);

    pipelab::GenConfig gc;
    gc.p = p;
    gc.v = v;
    gc.m = c.microbatches;
    gc.n = c.slices;
    gc.seq_len = c.seq_len;
    try {
      sched = pipelab::gen_slimpipe(gc);
    } catch (const std::exception& e) {
      return set_error(SP_ERR_INVALID, "%s", e.what());
    }
    const pipelab::Diagnostics diag = pipelab::validate_schedule(sched);
    if (!diag.ok()) return set_error(SP_ERR_RUNTIME, "schedule invalid: %s", diag.first()->message.c_str());
    order = sched.device_order[rank];
    ledger = pipelab::ledger_from_order(sched, pipelab::unit_memory_model(p, v, c.slices));
    if (v > 1) SP_TRY(check_ring_order());
    slots = int(ledger.per_device[rank].chunk_pool_size);
    if (c.exchange_mode != 0 && p > 1) {
      if (c.head_dim != 128 && c.head_dim != 64) return set_error(SP_ERR_UNSUPPORTED, "exchange: head_dim");
      pipelab::CostModel cm;
      cm.beta_attn = 1.0;  // any beta > 0 gives the identical plan (plan depends on slice indices only)
      ann = pipelab::apply_exchange(sched, cm, pipelab::ExchangeMode(c.exchange_mode));
      build_xplan();
    }
    if (c.vocab_parallel && p > 1) {
      if (c.vocab % p || (c.vocab / p) % 4)
        return set_error(SP_ERR_INVALID, "vocab_parallel: vocab (%d) must split into p shards of a multiple of 4",
                         c.vocab);
      vp = true;
      Vs = c.vocab / p;
      v0 = int64_t(rank) * Vs;
      // Base-simulation costs normalised so pass times are O(1): place_vocab
      // compares anchors against pass ends with a fixed 1e-9 slack, which
      // vanishes below one ulp once times reach ~1e7 (raw per-pair costs at
      // 4K+ tokens) and then orders VF(k,i) before its own F(k,i,p).
      pipelab::SimInputs in;
      in.cost.alpha_linear = 1.0 / double(c.seq_len);
      in.cost.beta_attn = 1.0 / (double(c.seq_len) * double(c.seq_len));
      in.seq_len = c.seq_len;
      try {
        sched = pipelab::place_vocab(sched, true, in);  // appends vocab passes: F/BW pass ids unchanged
      } catch (const std::exception& e) {
        return set_error(SP_ERR_INVALID, "%s", e.what());
      }
      const pipelab::Diagnostics vd = pipelab::validate_schedule(sched);
      if (!vd.ok()) return set_error(SP_ERR_RUNTIME, "vocab schedule invalid: %s", vd.first()->message.c_str());
      order = sched.device_order[rank];
      int live = 0, peak = 0;
      for (pipelab::PassId id : order) {
        // the last stage takes the slot at F(k,i,p) (it normalises the output there)
        const auto acq = last_dev ? pipelab::PassKind::Forward : pipelab::PassKind::VocabForward;
        if (sched.passes[id].kind == acq) peak = std::max(peak, ++live);
        if (sched.passes[id].kind == pipelab::PassKind::VocabBackward) --live;
      }
      vslots.resize(std::max(peak, 1));
    } else if (c.vocab_parallel < 0 || c.vocab_parallel > 1) {
      return set_error(SP_ERR_INVALID, "vocab_parallel must be 0 or 1");
    }

    SP_CUDA(cudaGetDevice(&device));  // host-side validation above runs without a GPU
    SP_TRY(preload_kernels());        // before any communication (transport.cu)
    SP_CUDA(cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking));
    // SP_COMM_PRIORITY=high (experimental, unmeasured): the link
    // and exchange streams get the highest priority, so their NCCL kernels are
    // dispatched ahead of the compute stream's queued attention CTAs instead
    // of after the running K1/K2 launch
    const char* cp = std::getenv("SP_COMM_PRIORITY");
    int prio_lo = 0, prio_hi = 0;
    SP_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    const int comm_prio = (cp && std::strcmp(cp, "high") == 0) ? prio_hi : prio_lo;
    for (cudaStream_t* st : {&s_act_in, &s_act_out, &s_grad_in, &s_grad_out})
      SP_CUDA(cudaStreamCreateWithPriority(st, cudaStreamNonBlocking, comm_prio));
    for (int x = 0; x < 2; ++x) {
      SP_CUDA(cudaEventCreateWithFlags(&ev_out_free[x], cudaEventDisableTiming));
      SP_CUDA(cudaEventCreateWithFlags(&ev_gin_free[x], cudaEventDisableTiming));
      SP_CUDA(cudaEventCreateWithFlags(&ev_gout_free[x], cudaEventDisableTiming));
      SP_CUDA(cudaEventRecord(ev_out_free[x], comp));
      SP_CUDA(cudaEventRecord(ev_gin_free[x], comp));
      SP_CUDA(cudaEventRecord(ev_gout_free[x], comp));
      SP_CUDA(cudaEventCreateWithFlags(&ev_ain_free[x], cudaEventDisableTiming));
      SP_CUDA(cudaEventRecord(ev_ain_free[x], comp));
    }
    SP_CUDA(cudaEventCreate(&step_start));
    SP_CUDA(cudaEventCreate(&step_end));
    SP_CUDA(cudaEventCreateWithFlags(&xev, cudaEventDisableTiming));

    if (p > 1 && loop) SP_TRY(init_loop_links());
    else if (p > 1) SP_TRY(init_nccl_links(ids));
    if (!xplan.empty() || c.exchange_mode != 0) {
      int lo = 0, hi = 0;
      SP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      for (int k = 0; k < 2 && p > 1; ++k) {
        SP_CUDA(cudaStreamCreateWithPriority(&cx[k], cudaStreamNonBlocking, comm_prio));
        SP_CUDA(cudaStreamCreateWithPriority(&rx[k], cudaStreamNonBlocking, hi));
      }
    }
    if (vp) SP_CUDA(cudaStreamCreateWithFlags(&s_vocab, cudaStreamNonBlocking));
    SP_TRY(alloc_params());
    // everything but the arena first, so recompute=auto sizes the O/LSE stash
    // against what is really left
    SP_TRY(alloc_workspace());
    SP_TRY(alloc_exchange());
    SP_TRY(alloc_arena());
    SP_TRY(init_weights(c.seed));
    SP_TRY(warm_gemms());
    SP_CUDA(cudaStreamSynchronize(comp));
    return SP_OK;
  }

  // Run every library GEMM of the step once (same shapes, transposes, output
  // types and beta, on the workspaces) before any communication, so cuBLASLt
  // has chosen and LOADED each kernel: a lazily loaded kernel launched while
  // a receive spins can deadlock (preload_kernels, transport.cu).  The
  // gradient buffers the weight-gradient GEMMs touched are zeroed again.
  int warm_gemms() {
    gemm_autotune(true);
    const int rc = warm_gemms_body();
    gemm_autotune(false);
    return rc;
  }
  int warm_gemms_body() {
    LayerWs& x = ws[0];
    const LayerParams& P = lp[0];
    SP_TRY(gemm(false, true, Ls, qkv_w, h, x.xn, h, W(P.wqkv), h, qkv, qkv_w, false, 1.f, 0.f, comp));
    SP_TRY(gemm(false, true, Ls, h, qd, x.o, qd, W(P.wo), qd, x.x_mid, h, false, 1.f, 1.f, comp, x.x_in));
    SP_TRY(gemm(false, true, Ls, 2 * H, h, x.xn2, h, W(P.wgu), h, x.gu, 2 * H, false, 1.f, 0.f, comp));
    SP_TRY(gemm(false, true, Ls, h, H, x.act, H, W(P.wd), H, x_final, h, false, 1.f, 1.f, comp, x.x_mid));
    SP_TRY(gemm(false, false, Ls, H, h, tmp_h, h, W(P.wd), H, tmp_H, H, false, 1.f, 0.f, comp));
    SP_TRY(gemm(true, false, h, H, Ls, tmp_h, h, x.act, H, G(P.wd), H, true, 1.f, 1.f, comp));
    SP_TRY(gemm(false, false, Ls, h, 2 * H, tmp_2H, 2 * H, W(P.wgu), h, tmp_h, h, false, 1.f, 0.f, comp));
    SP_TRY(gemm(true, false, 2 * H, h, Ls, tmp_2H, 2 * H, x.xn2, h, G(P.wgu), h, true, 1.f, 1.f, comp));
    SP_TRY(gemm(false, false, Ls, qd, h, x_final, h, W(P.wo), qd, tmp_h, qd, false, 1.f, 0.f, comp));
    SP_TRY(gemm(true, false, h, qd, Ls, x_final, h, x.o, qd, G(P.wo), qd, true, 1.f, 1.f, comp));
    SP_TRY(gemm(false, false, Ls, h, qkv_w, dqkv, qkv_w, W(P.wqkv), h, tmp_h, h, false, 1.f, 0.f, comp));
    SP_TRY(gemm(true, false, qkv_w, h, Ls, dqkv, qkv_w, x.xn, h, G(P.wqkv), h, true, 1.f, 1.f, comp));
    if (vp) {
      SP_TRY(gemm(false, true, Ls, Vs, h, vslots[0].xf, h, W(head), h, vlogits, Vs, true, 1.f, 0.f, comp));
      SP_TRY(gemm(false, false, Ls, h, Vs, vdlog, Vs, W(head), h, vdxf, h, true, 1.f, 0.f, comp));
      SP_TRY(gemm(true, false, Vs, h, Ls, vdlog, Vs, vslots[0].xf, h, G(head), h, true, 1.f, 1.f, comp));
    } else if (last_dev) {
      const int64_t V = cfg.vocab;
      SP_TRY(gemm(false, true, Ls, V, h, xf, h, W(head), h, logits, V, true, 1.f, 0.f, comp));
      SP_TRY(gemm(false, false, Ls, h, V, dlogits, V, W(head), h, tmp_h, h, false, 1.f, 0.f, comp));
      SP_TRY(gemm(true, false, V, h, Ls, dlogits, V, xf, h, G(head), h, true, 1.f, 1.f, comp));
    }
    SP_CUDA(cudaMemsetAsync(grad, 0, n_params * 4, comp));
    return SP_OK;
  }

  // Stage links and exchange communicators over NCCL (one process per GPU).
  int init_nccl_links(const void* ids) {
    ncclUniqueId id[SP_NCCL_IDS];
    std::memcpy(id, ids, sizeof id);
    // SP_NCCL_MAX_CTAS=N (diagnostics, default unset = NCCL's choice) caps
    // the CTAs of every stage and exchange communicator's kernels
    ncclConfig_t ccfg = NCCL_CONFIG_INITIALIZER;
    ncclConfig_t* pcfg = nullptr;
    if (const char* mc = std::getenv("SP_NCCL_MAX_CTAS")) {
      ccfg.maxCTAs = std::max(1, std::atoi(mc));
      ccfg.minCTAs = 1;
      pcfg = &ccfg;
    }
    if (pcfg) {
      SP_NCCL(ncclCommInitRankConfig(&nc_fwd, p, id[0], rank, pcfg));
      SP_NCCL(ncclCommInitRankConfig(&nc_bwd, p, id[1], rank, pcfg));
    } else {
      SP_NCCL(ncclCommInitRank(&nc_fwd, p, id[0], rank));
      SP_NCCL(ncclCommInitRank(&nc_bwd, p, id[1], rank));
    }
    // link (r, r+1) comes from split A when r is even, split B when r is odd
    auto split = [&](ncclComm_t parent, int color, int key, ncclComm_t* out) -> int {
      SP_NCCL(ncclCommSplit(parent, color, key, out, pcfg));
      return SP_OK;
    };
    // v > 1 (even p): split B also carries the ring's wrap link (p-1, 0),
    // where rank 0 is the receiving end and so takes link rank 1 (key p)
    const bool ring = v > 1;
    const int colA = rank / 2;  // {0,1} {2,3} ...
    const int colB = ring ? (rank % 2 ? (rank + 1) / 2 : rank / 2) % (p / 2)
                          : (rank == 0 ? NCCL_SPLIT_NOCOLOR : (rank + 1) / 2);  // {1,2} {3,4} ... [{p-1,0}]
    const int keyB = ring && rank == 0 ? p : rank;
    ncclComm_t fa = nullptr, fb = nullptr, ga = nullptr, gb = nullptr;
    SP_TRY(split(nc_fwd, (rank == p - 1 && rank % 2 == 0) ? NCCL_SPLIT_NOCOLOR : colA, rank, &fa));
    SP_TRY(split(nc_fwd, (!ring && rank == p - 1 && rank % 2 == 1) ? NCCL_SPLIT_NOCOLOR : colB, keyB, &fb));
    SP_TRY(split(nc_bwd, (rank == p - 1 && rank % 2 == 0) ? NCCL_SPLIT_NOCOLOR : colA, rank, &ga));
    SP_TRY(split(nc_bwd, (!ring && rank == p - 1 && rank % 2 == 1) ? NCCL_SPLIT_NOCOLOR : colB, keyB, &gb));
    const bool even = rank % 2 == 0;
    if (!last_dev || ring) {  // link to the next stage
      l_act_out = make_nccl_link(even ? fa : fb);
      l_grad_in = make_nccl_link(even ? ga : gb);
    }
    if (!first_dev || ring) {  // link to the previous stage (r-1, r): split A iff r-1 even
      l_act_in = make_nccl_link(even ? fb : fa);
      l_grad_out = make_nccl_link(even ? gb : ga);
    }
    if (!xplan.empty() || cfg.exchange_mode != 0)
      for (int k = 0; k < 2; ++k) {
        ncclComm_t cm = nullptr;
        if (pcfg) SP_NCCL(ncclCommInitRankConfig(&cm, p, id[2 + k], rank, pcfg));
        else SP_NCCL(ncclCommInitRank(&cm, p, id[2 + k], rank));
        lx[k] = make_nccl_link(cm);
      }
    if (vp) {  // the vocabulary collectives run on the world communicator nc_bwd
      vlink = make_nccl_link(nc_bwd);
      nc_bwd = nullptr;
    }
    return warm_links();
  }

  // The same links on the single-GPU loopback transport (every rank a thread
  // of this process): communicator ids 0 activations, 1 gradients, 2/3 the
  // two exchange classes.  Link ranks as in init_nccl_links: the lower stage
  // of a stage link is link rank 0 (the ring's wrap link: device p-1).
  int init_loop_links() {
    if (loop_world_size(loop) != p) return set_error(SP_ERR_INVALID, "loopback world has %d ranks, pp = %d",
                                                     loop_world_size(loop), p);
    // Receives are posted early here: the loopback's waits are one-CTA
    // kernels (nothing like an NCCL receive's SMs to save), and with every
    // rank's streams on one device the extra compute -> receive-stream
    // dependencies of just-in-time posting measured a stall at PP=4 with
    // the exchange on (hardware-queue sharing, §2.3).
    jit_recv = false;
    xserve_jit = false;
    const bool ring = v > 1;
    const int nx = (rank + 1) % p, pv = (rank + p - 1) % p;
    if (!last_dev || ring) {
      l_act_out = make_loop_link(loop, 0, {rank, nx}, 0);
      l_grad_in = make_loop_link(loop, 1, {rank, nx}, 0);
    }
    if (!first_dev || ring) {
      l_act_in = make_loop_link(loop, 0, {pv, rank}, 1);
      l_grad_out = make_loop_link(loop, 1, {pv, rank}, 1);
    }
    std::vector<int> all(static_cast<size_t>(p));
    for (int r = 0; r < p; ++r) all[size_t(r)] = r;
    if (!xplan.empty() || cfg.exchange_mode != 0)
      for (int k = 0; k < 2; ++k) lx[k] = make_loop_link(loop, 2 + k, all, rank);
    if (vp) {  // collectives over p2p (transport.cu); scratch sized now, not inside a step
      vlink = make_loop_link(loop, 4, all, rank);
      SP_TRY(vlink->reserve(Ls * h));
    }
    return SP_OK;
  }

  // NCCL connects peers lazily, at the first send/recv (or collective
  // algorithm) of a communicator, with a host-side handshake that blocks
  // until the peer's host reaches the same communicator.  The step enqueues
  // asynchronously in each rank's own pass order, so first uses would meet in
  // rank-dependent orders — a host-level cycle (the round-1 vocab-parallel /
  // interleaved stall: both ranks blocked inside step enqueue).  Every
  // communicator is therefore exercised here, in one global order:
  //   1. stage links in increasing link index (link (a, a+1) = a; the ring's
  //      wrap link = p-1), activations then gradients — per rank increasing,
  //      so the waits form a chain, never a cycle;
  //   2. the two exchange communicators: one group with every peer;
  //   3. the vocabulary collectives at their real message sizes (the
  //      algorithm, hence the connection, depends on the size).
  int warm_links() {
    cudaStream_t st = comp;
    void* buf = nullptr;
    const size_t big = vp ? size_t(Ls) * size_t(h) * 4 : 4096;
    SP_CUDA(cudaMalloc(&buf, big));
    SP_CUDA(cudaMemsetAsync(buf, 0, big, st));
    char* b = static_cast<char*>(buf);
    auto pair = [&](Link* l, int peer) -> int {
      SP_TRY(l->group_start());
      SP_TRY(l->send(b, 4, ncclUint8, peer, st));
      SP_TRY(l->recv(b + 64, 4, ncclUint8, peer, st));
      return l->group_end();
    };
    const bool ring = v > 1;
    const int prev_link = first_dev ? (ring ? p - 1 : -1) : rank - 1;  // link index of (prev, me)
    const int next_link = (!last_dev || ring) ? rank : -1;              // link index of (me, next)
    std::vector<std::pair<int, int>> mine;  // (link index, 0 = to prev / 1 = to next)
    if (prev_link >= 0) mine.emplace_back(prev_link, 0);
    if (next_link >= 0) mine.emplace_back(next_link, 1);
    std::sort(mine.begin(), mine.end());
    for (const auto& lk : mine) {
      if (lk.second == 0) {
        SP_TRY(pair(l_act_in.get(), 0));
        SP_TRY(pair(l_grad_out.get(), 0));
      } else {
        SP_TRY(pair(l_act_out.get(), 1));
        SP_TRY(pair(l_grad_in.get(), 1));
      }
    }
    for (int k = 0; k < 2; ++k) {
      if (!lx[k]) continue;
      SP_TRY(lx[k]->group_start());
      for (int q = 0; q < p; ++q)
        if (q != rank) {
          SP_TRY(lx[k]->send(b, 4, ncclUint8, q, st));
          SP_TRY(lx[k]->recv(b + 64 + 8 * q, 4, ncclUint8, q, st));
        }
      SP_TRY(lx[k]->group_end());
    }
    if (vp) {
      float* f = static_cast<float*>(buf);
      SP_TRY(vlink->broadcast(buf, Ls * h, ncclBfloat16, p - 1, st));
      SP_TRY(vlink->all_reduce(f, Ls, ncclMax, st));
      SP_TRY(vlink->all_reduce(f, 2 * Ls, ncclSum, st));
      SP_TRY(vlink->reduce(f, Ls * h, p - 1, st));
    }
    SP_CUDA(cudaStreamSynchronize(st));
    SP_CUDA(cudaFree(buf));
    return SP_OK;
  }

  // Interleaved pre-flight (v > 1): every stage link is one FIFO pair of
  // NCCL streams, so the sender's order of F outputs (B input grads) on a
  // link must equal the receiver's order of the passes consuming them; and
  // each local chunk's backward must run a microbatch's slices n..1
  // back to back (one dK/dV accumulator set per chunk).
  int check_ring_order() const {
    using Key = std::tuple<int, int, int>;
    for (int d = 0; d < p; ++d) {
      const int nx = (d + 1) % p;
      std::vector<Key> snd, rcv, gsnd, grcv;
      for (pipelab::PassId id : sched.device_order[d]) {
        const pipelab::Pass& q = sched.passes[id];
        if (q.kind == pipelab::PassKind::Forward && q.stage < nst) snd.emplace_back(q.microbatch, q.slice, q.stage);
        if (q.kind == pipelab::PassKind::BackwardFused && q.stage > 1)
          gsnd.emplace_back(q.microbatch, q.slice, q.stage - 1);
      }
      for (pipelab::PassId id : sched.device_order[nx]) {
        const pipelab::Pass& q = sched.passes[id];
        if (q.kind == pipelab::PassKind::Forward && q.stage > 1) rcv.emplace_back(q.microbatch, q.slice, q.stage - 1);
      }
      for (pipelab::PassId id : sched.device_order[(d + p - 1) % p]) {
        const pipelab::Pass& q = sched.passes[id];
        if (q.kind == pipelab::PassKind::BackwardFused && q.stage < nst)
          grcv.emplace_back(q.microbatch, q.slice, q.stage);
      }
      if (snd != rcv || gsnd != grcv)
        return set_error(SP_ERR_UNSUPPORTED, "interleaved schedule: link %d order differs between its ends", d);
      std::vector<std::vector<std::pair<int, int>>> per(static_cast<size_t>(v));
      for (pipelab::PassId id : sched.device_order[d]) {
        const pipelab::Pass& q = sched.passes[id];
        if (q.kind != pipelab::PassKind::Forward) per[size_t((q.stage - 1) / p)].emplace_back(q.microbatch, q.slice);
      }
      for (const auto& seq : per)
        for (std::size_t x = 0; x < seq.size(); ++x)
          if (seq[x].second != cfg.slices - int(x % cfg.slices) || (x % cfg.slices && seq[x].first != seq[x - 1].first))
            return set_error(SP_ERR_UNSUPPORTED, "interleaved schedule: backward slices of a chunk interleave");
    }
    return SP_OK;
  }

  // Per-pass transfer lists of this rank from the tick plans (xplan.hpp).
  void build_xplan() {
    xplan = exchange_passes(sched, ann, rank, p, cfg.exchange_min_chunks, cfg.exchange_skip_last != 0);
    for (const auto& [pid, px] : xplan) {
      x_tout = std::max(x_tout, int(px.out.size()));
      x_cout = std::max(x_cout, px.out_chunks);
      x_tin = std::max(x_tin, int(px.in.size()));
      x_cin = std::max(x_cin, px.in_chunks);
    }
  }

  int alloc_exchange() {
    if (xplan.empty()) return SP_OK;
    const int64_t a = cfg.heads;
    for (int c = 0; c < 2; ++c) {
      XBuf& b = xb[c];
      if (x_tout > 0) {
        SP_TRY(alloc(&b.o_rem, x_tout * Ls * qd));
        SP_TRY(alloc(&b.lse_rem, x_tout * a * Ls));
        if (c == 1) {
          SP_TRY(alloc(&b.dq_rem, x_tout * Ls * qd));
          SP_TRY(alloc(&b.dk_rem, std::max(1, x_cout) * Ls * kvd));
          SP_TRY(alloc(&b.dv_rem, std::max(1, x_cout) * Ls * kvd));
        }
      }
      if (x_tin > 0) {
        SP_TRY(alloc(&b.rq, x_tin * Ls * qd));
        SP_TRY(alloc(&b.ro, x_tin * Ls * qd));
        SP_TRY(alloc(&b.rlse, x_tin * a * Ls));
        SP_TRY(alloc(&b.rk, std::max(1, x_cin) * Ls * kvd));
        SP_TRY(alloc(&b.rv, std::max(1, x_cin) * Ls * kvd));
        if (c == 1) {
          SP_TRY(alloc(&b.rdo, x_tin * Ls * qd));
          SP_TRY(alloc(&b.rstats, x_tin * 2 * a * Ls));
          SP_TRY(alloc(&b.rdq, x_tin * Ls * qd));
          SP_TRY(alloc(&b.rdk, std::max(1, x_cin) * Ls * kvd));
          SP_TRY(alloc(&b.rdv, std::max(1, x_cin) * Ls * kvd));
        }
      }
    }
    return SP_OK;
  }

  const PassX* pass_x(int pid) const {
    auto it = xplan.find(pid);
    return it == xplan.end() ? nullptr : &it->second;
  }

  int link(cudaStream_t from, cudaStream_t to) { return hand_off(from, to); }

  // A stage message (one [Ls, h] bf16 slice) with CUDA events around the
  // send on its stream: bytes / span is the link rate once the receiver's
  // matching receive is posted (reported by sp_runtime_comm_stats).
  int timed_send(Link* l, const void* buf, int peer, cudaStream_t st) {
    CommTimer t{nullptr, nullptr, Ls * h * 2};
    SP_TRY(timing_event(&t.a));
    SP_TRY(timing_event(&t.b));
    SP_CUDA(cudaEventRecord(t.a, st));
    SP_TRY(l->send(buf, Ls * h, ncclBfloat16, peer, st));
    SP_CUDA(cudaEventRecord(t.b, st));
    comm_times.push_back(t);
    return SP_OK;
  }

  // K chunks then V chunks, one message per chunk (the sender ships them from
  // their arena slots), landing contiguously at the transfer's pool rows.
  int recv_chunks(bf16raw* rk, bf16raw* rv, const XIn& xi, int c) {
    for (std::size_t x = 0; x < xi.chunks.size(); ++x)
      SP_TRY(lx[c]->recv(rk + int64_t(xi.base + x) * Ls * kvd, Ls * kvd, ncclBfloat16, xi.peer, cx[c]));
    for (std::size_t x = 0; x < xi.chunks.size(); ++x)
      SP_TRY(lx[c]->recv(rv + int64_t(xi.base + x) * Ls * kvd, Ls * kvd, ncclBfloat16, xi.peer, cx[c]));
    return SP_OK;
  }
  int send_chunks(int l, int k, const XOut& xo, int c) {
    for (int ch : xo.chunks)
      SP_TRY(lx[c]->send(k_pool[l] + int64_t(slot_of.at(sk(k, ch))) * Ls * kvd, Ls * kvd, ncclBfloat16, xo.peer, cx[c]));
    for (int ch : xo.chunks)
      SP_TRY(lx[c]->send(v_pool[l] + int64_t(slot_of.at(sk(k, ch))) * Ls * kvd, Ls * kvd, ncclBfloat16, xo.peer, cx[c]));
    x_bytes_sent += 2 * int64_t(xo.chunks.size()) * Ls * kvd * 2;
    return SP_OK;
  }

  // Chunks this pass attends itself: {1..i} minus every chunk shipped out;
  // causal iff the diagonal chunk i stays (early plans never ship it,
  // reference exchange.cpp:86-89).
  void own_chunks(int k, int i, const PassX* px, std::vector<int32_t>& rows, std::vector<int32_t>& acc,
                  int& causal) const {
    std::vector<char> shipped(i + 1, 0);
    if (px)
      for (const XOut& xo : px->out)
        for (int ch : xo.chunks) shipped[ch] = 1;
    for (int j = 1; j <= i; ++j)
      if (!shipped[j]) {
        rows.push_back(int32_t(slot_of.at(sk(k, j)) * Ls));
        acc.push_back(int32_t((j - 1) * Ls));
      }
    causal = shipped[i] ? 0 : 1;
  }

  // ---- receiver side: every partial this rank computes for peers in pass px.
  // Posted at pass start on the class's copy / remote-compute streams; per
  // layer and transfer: recv (Q [, dO, stats], K/V chunks) -> attention
  // partial -> send back.  Forward ticks: layers 0..L-1 (forward).  Backward
  // ticks: layers 0..L-1 (the peer's recompute) then L-1..0 (its backward).
  int post_remote(const PassX& px) {
    const int c = px.cls;
    XBuf& b = xb[c];
    const int64_t a = cfg.heads;
    if (xserve_jit) SP_TRY(link(comp, cx[c]));
    auto fwd_layer = [&]() -> int {
      for (std::size_t t = 0; t < px.in.size(); ++t) {
        const XIn& xi = px.in[t];
        const int nc = int(xi.chunks.size());
        SP_TRY(lx[c]->group_start());
        SP_TRY(lx[c]->recv(b.rq + t * Ls * qd, Ls * qd, ncclBfloat16, xi.peer, cx[c]));
        SP_TRY(recv_chunks(b.rk, b.rv, xi, c));
        SP_TRY(lx[c]->group_end());
        SP_TRY(link(cx[c], rx[c]));
        std::vector<int32_t> rows;
        for (int x = 0; x < nc; ++x) rows.push_back(int32_t((xi.base + x) * Ls));
        const int causal = xi.chunks.back() == xi.i_src;
        SP_TRY(sp_attn_fwd(b.rq + t * Ls * qd, Ls, qd, b.rk, b.rv, int64_t(std::max(1, x_cin)) * Ls, kvd, rows.data(),
                           nc, int(Ls), cfg.heads, cfg.kv_heads, cfg.head_dim, causal, b.ro + t * Ls * qd, qd,
                           b.rlse + t * a * Ls, rx[c]));
        SP_TRY(link(rx[c], cx[c]));
        SP_TRY(lx[c]->group_start());
        SP_TRY(lx[c]->send(b.ro + t * Ls * qd, Ls * qd, ncclBfloat16, xi.peer, cx[c]));
        SP_TRY(lx[c]->send(b.rlse + t * a * Ls, a * Ls, ncclFloat32, xi.peer, cx[c]));
        SP_TRY(lx[c]->group_end());
      }
      return SP_OK;
    };
    auto bwd_layer = [&]() -> int {
      for (std::size_t t = 0; t < px.in.size(); ++t) {
        const XIn& xi = px.in[t];
        const int nc = int(xi.chunks.size());
        SP_TRY(lx[c]->group_start());
        SP_TRY(lx[c]->recv(b.rq + t * Ls * qd, Ls * qd, ncclBfloat16, xi.peer, cx[c]));
        SP_TRY(lx[c]->recv(b.rdo + t * Ls * qd, Ls * qd, ncclBfloat16, xi.peer, cx[c]));
        SP_TRY(lx[c]->recv(b.rstats + t * 2 * a * Ls, 2 * a * Ls, ncclFloat32, xi.peer, cx[c]));
        SP_TRY(recv_chunks(b.rk, b.rv, xi, c));
        SP_TRY(lx[c]->group_end());
        SP_TRY(link(cx[c], rx[c]));
        std::vector<int32_t> rows;
        for (int x = 0; x < nc; ++x) rows.push_back(int32_t((xi.base + x) * Ls));
        const int causal = xi.chunks.back() == xi.i_src;
        float* dq = b.rdq + t * Ls * qd;
        float* dk = b.rdk + int64_t(xi.base) * Ls * kvd;
        float* dv = b.rdv + int64_t(xi.base) * Ls * kvd;
        SP_CUDA(cudaMemsetAsync(dq, 0, Ls * qd * 4, rx[c]));
        SP_CUDA(cudaMemsetAsync(dk, 0, nc * Ls * kvd * 4, rx[c]));
        SP_CUDA(cudaMemsetAsync(dv, 0, nc * Ls * kvd * 4, rx[c]));
        SP_TRY(sp_attn_bwd_core(b.rq + t * Ls * qd, Ls, qd, b.rk, b.rv, int64_t(std::max(1, x_cin)) * Ls, kvd,
                                rows.data(), nc, int(Ls), cfg.heads, cfg.kv_heads, cfg.head_dim, causal,
                                b.rdo + t * Ls * qd, qd, b.rstats + t * 2 * a * Ls, dq, b.rdk, b.rdv,
                                int64_t(std::max(1, x_cin)) * Ls, rows.data(), rx[c]));
        SP_TRY(link(rx[c], cx[c]));
        SP_TRY(lx[c]->group_start());
        SP_TRY(lx[c]->send(dq, Ls * qd, ncclFloat32, xi.peer, cx[c]));
        SP_TRY(lx[c]->send(dk, nc * Ls * kvd, ncclFloat32, xi.peer, cx[c]));
        SP_TRY(lx[c]->send(dv, nc * Ls * kvd, ncclFloat32, xi.peer, cx[c]));
        SP_TRY(lx[c]->group_end());
      }
      return SP_OK;
    };
    // backward ticks: the peer's recompute needs the forward partials again
    // only under full recompute (selective reuses its stashed O/LSE)
    if (c == 0 || !stash)
      for (int l = 0; l < Lps; ++l) SP_TRY(fwd_layer());
    if (c == 1)
      for (int l = Lps - 1; l >= 0; --l) SP_TRY(bwd_layer());
    return SP_OK;
  }

  int alloc_params() {
    auto take = [&](int64_t n) {
      const int64_t off = n_params;
      n_params += (n + 127) / 128 * 128;
      return off;
    };
    lp.resize(size_t(v) * Lps);  // local chunk c's layers at [c*Lps, (c+1)*Lps)
    for (int l = 0; l < v * Lps; ++l) {
      lp[l].attn_norm = take(h);
      lp[l].wqkv = take(qkv_w * h);
      lp[l].wo = take(h * qd);
      lp[l].mlp_norm = take(h);
      lp[l].wgu = take(2 * H * h);
      lp[l].wd = take(h * H);
    }
    if (first_dev) emb = take(int64_t(cfg.vocab) * h);
    if (last_dev) final_norm = take(h);
    if (vp) head = take(Vs * h);  // this stage's vocab shard
    else if (last_dev) head = take(int64_t(cfg.vocab) * h);
    SP_TRY(alloc(&w, n_params));
    SP_TRY(alloc(&master, n_params));
    SP_TRY(alloc(&grad, n_params));
    SP_TRY(alloc(&adam_m, n_params));
    SP_TRY(alloc(&adam_v, n_params));
    SP_CUDA(cudaMemsetAsync(grad, 0, n_params * 4, comp));
    SP_CUDA(cudaMemsetAsync(adam_m, 0, n_params * 4, comp));
    SP_CUDA(cudaMemsetAsync(adam_v, 0, n_params * 4, comp));
    return SP_OK;
  }

  int init_weights(uint64_t seed) {
    const float std_w = 0.02f;
    uint64_t tag = seed * 1000003ull + uint64_t(rank + 1) * 7919ull;
    auto normal = [&](int64_t off, int64_t n) {
      return init_params(master + off, w + off, n, ++tag, std_w, 0.f, 0, comp);
    };
    auto ones = [&](int64_t off, int64_t n) { return init_params(master + off, w + off, n, ++tag, 0.f, 1.f, 1, comp); };
    for (int l = 0; l < v * Lps; ++l) {
      SP_TRY(ones(lp[l].attn_norm, h));
      SP_TRY(normal(lp[l].wqkv, qkv_w * h));
      SP_TRY(normal(lp[l].wo, h * qd));
      SP_TRY(ones(lp[l].mlp_norm, h));
      SP_TRY(normal(lp[l].wgu, 2 * H * h));
      SP_TRY(normal(lp[l].wd, h * H));
    }
    if (emb >= 0) SP_TRY(normal(emb, int64_t(cfg.vocab) * h));
    if (final_norm >= 0) SP_TRY(ones(final_norm, h));
    if (head >= 0) SP_TRY(normal(head, (vp ? Vs : int64_t(cfg.vocab)) * h));
    return SP_OK;
  }

  int alloc_arena() {
    const int64_t rows = int64_t(slots) * Ls;
    if (offload) SP_TRY(alloc(&x_stage, Ls * h));
    else SP_TRY(alloc(&x_pool, rows * h));
    k_pool.assign(Lps, nullptr);
    v_pool.assign(Lps, nullptr);
    dk_acc.assign(size_t(v) * Lps, nullptr);  // per local chunk and layer
    dv_acc.assign(size_t(v) * Lps, nullptr);
    const int64_t acc_rows = int64_t(cfg.slices) * Ls;
    for (int l = 0; l < Lps; ++l) {
      SP_TRY(alloc(&k_pool[l], rows * kvd));
      SP_TRY(alloc(&v_pool[l], rows * kvd));
    }
    for (int l = 0; l < v * Lps; ++l) {
      // byte buffers of acc_es-sized elements
      SP_TRY(alloc(reinterpret_cast<char**>(&dk_acc[l]), acc_rows * kvd * acc_es));
      SP_TRY(alloc(reinterpret_cast<char**>(&dv_acc[l]), acc_rows * kvd * acc_es));
      SP_CUDA(cudaMemsetAsync(dk_acc[l], 0, acc_rows * kvd * acc_es, comp));
      SP_CUDA(cudaMemsetAsync(dv_acc[l], 0, acc_rows * kvd * acc_es, comp));
    }
    if (cfg.recompute == 2) {  // auto: stash O/LSE only if it fits beside everything allocated so far
      size_t free_b = 0, total_b = 0;
      SP_CUDA(cudaMemGetInfo(&free_b, &total_b));
      // (offloaded: the device keeps one pass's staging, the slots live on the host)
      const double stash_b = double(Lps) * (offload ? Ls : rows) * (qd * 2 + double(cfg.heads) * 4);
      const double margin = 2.0 * double(1 << 30);  // cuBLASLt workspaces, NCCL buffers, allocator slack
      stash = stash_b + margin < double(free_b);
    }
    if (stash && offload) {
      o_stage.assign(Lps, nullptr);
      l_stage.assign(Lps, nullptr);
      for (int l = 0; l < Lps; ++l) {
        SP_TRY(alloc(&o_stage[l], Ls * qd));
        SP_TRY(alloc(&l_stage[l], int64_t(cfg.heads) * Ls));
      }
    } else if (stash) {
      o_pool.assign(Lps, nullptr);
      lse_pool.assign(Lps, nullptr);
      const size_t n_before = allocations.size();
      int rc = SP_OK;
      for (int l = 0; l < Lps && rc == SP_OK; ++l) {
        rc = alloc(&o_pool[l], rows * qd);
        if (rc == SP_OK) rc = alloc(&lse_pool[l], rows * cfg.heads);
      }
      if (rc != SP_OK) {
        if (cfg.recompute != 2) return rc;
        // auto: the estimate was optimistic -> full recompute instead of failing
        cudaGetLastError();
        while (allocations.size() > n_before) {
          cudaFree(allocations.back());
          allocations.pop_back();
        }
        o_pool.clear();
        lse_pool.clear();
        stash = false;
      }
    }
    if (offload) {  // the host side of the slots, and the copy stream / events
      auto host = [&](void** p, size_t bytes) -> int {
        SP_CUDA(cudaHostAlloc(p, std::max<size_t>(bytes, 16), cudaHostAllocDefault));
        offload_bytes += bytes;
        return SP_OK;
      };
      SP_TRY(host(reinterpret_cast<void**>(&hx), size_t(rows) * size_t(h) * 2));
      if (stash) {
        SP_TRY(host(reinterpret_cast<void**>(&ho), size_t(slots) * Lps * size_t(Ls) * size_t(qd) * 2));
        SP_TRY(host(reinterpret_cast<void**>(&hl), size_t(slots) * Lps * size_t(cfg.heads) * size_t(Ls) * 4));
      }
      SP_CUDA(cudaStreamCreateWithFlags(&s_off, cudaStreamNonBlocking));
      for (cudaEvent_t* e : {&ev_x_off, &ev_x_in}) {
        SP_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        SP_CUDA(cudaEventRecord(*e, s_off));
      }
      ev_o_off.assign(Lps, nullptr);
      ev_o_in.assign(Lps, nullptr);
      for (int l = 0; l < Lps; ++l)
        for (cudaEvent_t* e : {&ev_o_off[l], &ev_o_in[l]}) {
          SP_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
          SP_CUDA(cudaEventRecord(*e, s_off));
        }
    }
    free_slots.clear();
    for (int s = slots - 1; s >= 0; --s) free_slots.push_back(s);  // pop_back -> lowest first
    return SP_OK;
  }

  // offload helpers: a slot's host copies
  bf16raw* host_x(int slot) { return hx + int64_t(slot) * Ls * h; }
  bf16raw* host_o(int slot, int l) { return ho + (int64_t(slot) * Lps + l) * Ls * qd; }
  float* host_l(int slot, int l) { return hl + (int64_t(slot) * Lps + l) * cfg.heads * Ls; }

  int alloc_workspace() {
    ws.resize(Lps);
    for (int l = 0; l < Lps; ++l) {
      LayerWs& x = ws[l];
      SP_TRY(alloc(&x.x_in, Ls * h));
      SP_TRY(alloc(&x.xn, Ls * h));
      SP_TRY(alloc(&x.q, Ls * qd));
      SP_TRY(alloc(&x.o_ws, Ls * qd));
      x.o = x.o_ws;
      SP_TRY(alloc(&x.x_mid, Ls * h));
      SP_TRY(alloc(&x.xn2, Ls * h));
      SP_TRY(alloc(&x.gu, Ls * 2 * H));
      SP_TRY(alloc(&x.act, Ls * H));
      SP_TRY(alloc(&x.lse_ws, int64_t(cfg.heads) * Ls));
      x.lse = x.lse_ws;
      SP_TRY(alloc(&x.rstd1, Ls));
      SP_TRY(alloc(&x.rstd2, Ls));
    }
    SP_TRY(alloc(&x_final, Ls * h));
    SP_TRY(alloc(&qkv, Ls * qkv_w));
    SP_TRY(alloc(&dqkv, Ls * qkv_w));
    SP_TRY(alloc(&tmp_h, Ls * std::max(h, qd)));
    SP_TRY(alloc(&tmp_H, Ls * H));
    SP_TRY(alloc(&tmp_2H, Ls * 2 * H));
    for (int x = 0; x < 2; ++x) {
      if (!first_dev || v > 1) SP_TRY(alloc(&ain_buf[x], Ls * h));
      SP_TRY(alloc(&out_buf[x], Ls * h));
      SP_TRY(alloc(&gin_buf[x], Ls * h));
      SP_TRY(alloc(&gout_buf[x], Ls * h));
    }
    SP_TRY(alloc(&rope_cos, cfg.seq_len * (cfg.head_dim / 2)));
    SP_TRY(alloc(&rope_sin, cfg.seq_len * (cfg.head_dim / 2)));
    SP_TRY(rope_table(rope_cos, rope_sin, cfg.seq_len, cfg.head_dim, double(cfg.rope_theta), comp));
    SP_TRY(alloc(&dq_acc, Ls * qd));
    SP_TRY(alloc(&norm_ws, rmsnorm_dw_ws_floats(Ls, int(h))));
    SP_TRY(alloc(&delta_ws, 2 * int64_t(cfg.heads) * Ls));
    SP_TRY(alloc(&loss_dev, 1));
    SP_TRY(alloc(&tokens, int64_t(cfg.microbatches) * cfg.seq_len));
    SP_TRY(alloc(&targets, int64_t(cfg.microbatches) * cfg.seq_len));
    const size_t tok_bytes = size_t(cfg.microbatches) * size_t(cfg.seq_len) * 4;
    SP_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_tok), tok_bytes, cudaHostAllocDefault));
    SP_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_tgt), tok_bytes, cudaHostAllocDefault));
    SP_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_loss), 4, cudaHostAllocDefault));
    SP_CUDA(cudaEventCreateWithFlags(&ev_staged, cudaEventDisableTiming));
    SP_CUDA(cudaEventRecord(ev_staged, comp));
    if (last_dev) {
      SP_TRY(alloc(&xf, Ls * h));
      SP_TRY(alloc(&rstd_f, Ls));
      if (!vp) {
        SP_TRY(alloc(&logits, Ls * int64_t(cfg.vocab)));
        SP_TRY(alloc(&dlogits, Ls * int64_t(cfg.vocab)));
      }
    }
    if (vp) {
      for (VSlot& v : vslots) {
        SP_TRY(alloc(&v.xf, Ls * h));
        SP_TRY(alloc(&v.st, 4 * Ls));
      }
      vfree.clear();
      for (int x = int(vslots.size()) - 1; x >= 0; --x) vfree.push_back(x);
      SP_TRY(alloc(&vlogits, Ls * Vs));
      SP_TRY(alloc(&vdlog, Ls * Vs));
      SP_TRY(alloc(&vdxf, Ls * h));
    }
    return SP_OK;
  }

  // -------------------------------------------------------------- passes
  std::vector<int32_t> chunk_rows(int k, int i) const {
    std::vector<int32_t> rows;
    for (int j = 1; j <= i; ++j) rows.push_back(int32_t(slot_of.at(sk(k, j)) * Ls));
    return rows;
  }

  double attn_flops(int n_chunks, int causal) const {  // forward FLOPs
    const double keys = causal ? double(n_chunks - 1) * Ls + (Ls + 1) / 2.0 : double(n_chunks) * Ls;
    return 4.0 * cfg.head_dim * double(Ls) * keys * cfg.heads;
  }

  int attn_fwd_timed(int l, const std::vector<int32_t>& rows, int causal, LayerWs& x) {
    AttnTimer t{};
    SP_TRY(timing_event(&t.a));
    SP_TRY(timing_event(&t.b));
    const int nch = int(rows.size());
    t.flops = attn_flops(nch, causal);
    t.kind = 0;
    SP_CUDA(cudaEventRecord(t.a, comp));
    SP_TRY(sp_attn_fwd(x.q, Ls, qd, k_pool[l], v_pool[l], int64_t(slots) * Ls, kvd, rows.data(), nch, int(Ls),
                       cfg.heads, cfg.kv_heads, cfg.head_dim, causal, x.o, qd, x.lse, comp));
    SP_CUDA(cudaEventRecord(t.b, comp));
    attn_times.push_back(t);
    return SP_OK;
  }

  // One layer forward; saves its internals in ws[l]; writes its output to x_out.
  // K1 with the pass's transfers: ship Q (+ KV chunks) to each receiver,
  // attend the retained chunks, merge every returned (O, LSE) partial (K3).
  int attention_forward(int l, int k, int i, LayerWs& x, const PassX* px) {
    std::vector<int32_t> rows, acc;
    int causal = 1;
    own_chunks(k, i, px, rows, acc, causal);
    const bool out = px && !px->out.empty();
    const int c = px ? px->cls : 0;
    const int64_t a = cfg.heads;
    if (out) {
      SP_TRY(link(comp, cx[c]));
      for (const XOut& xo : px->out) {
        SP_TRY(lx[c]->group_start());
        SP_TRY(lx[c]->send(x.q, Ls * qd, ncclBfloat16, xo.peer, cx[c]));
        SP_TRY(send_chunks(l, k, xo, c));
        SP_TRY(lx[c]->group_end());
        x_bytes_sent += Ls * qd * 2;
      }
    }
    SP_TRY(attn_fwd_timed(l, rows, causal, x));
    if (out) {
      XBuf& b = xb[c];
      for (std::size_t t = 0; t < px->out.size(); ++t) {
        SP_TRY(lx[c]->group_start());
        SP_TRY(lx[c]->recv(b.o_rem + t * Ls * qd, Ls * qd, ncclBfloat16, px->out[t].peer, cx[c]));
        SP_TRY(lx[c]->recv(b.lse_rem + t * a * Ls, a * Ls, ncclFloat32, px->out[t].peer, cx[c]));
        SP_TRY(lx[c]->group_end());
      }
      SP_TRY(link(cx[c], comp));
      for (std::size_t t = 0; t < px->out.size(); ++t)
        SP_TRY(sp_attn_merge(x.o, x.lse, b.o_rem + t * Ls * qd, b.lse_rem + t * a * Ls, Ls, cfg.heads, cfg.head_dim, qd,
                             x.o, x.lse, comp));
    }
    return SP_OK;
  }

  // attention output of layer l for slice (k, i): the slot's stash or the workspace
  void bind_attn_out(int l, int slot) {
    LayerWs& x = ws[l];
    if (stash && offload) {
      x.o = o_stage[l];
      x.lse = l_stage[l];
      return;
    }
    x.o = stash ? o_pool[l] + int64_t(slot) * Ls * qd : x.o_ws;
    x.lse = stash ? lse_pool[l] + int64_t(slot) * cfg.heads * Ls : x.lse_ws;
  }

  int layer_forward(int l, int k, int i, bf16raw* x_out, const PassX* px, bool recompute) {
    LayerWs& x = ws[l];
    const LayerParams& P = lp[lbase + l];
    const int slot = slot_of.at(sk(k, i));
    bind_attn_out(l, slot);
    const int64_t pos0 = int64_t(i - 1) * Ls;
    SP_TRY(rmsnorm_fwd(x.x_in, W(P.attn_norm), x.xn, x.rstd1, Ls, int(h), cfg.norm_eps, comp));
    SP_TRY(gemm(false, true, Ls, qkv_w, h, x.xn, h, W(P.wqkv), h, qkv, qkv_w, false, 1.f, 0.f, comp));
    SP_TRY(rope_qkv_fwd(qkv, Ls, cfg.heads, cfg.kv_heads, cfg.head_dim, pos0, rope_cos, rope_sin, x.q, qd,
                        k_pool[l] + int64_t(slot) * Ls * kvd, v_pool[l] + int64_t(slot) * Ls * kvd, kvd, comp));
    const bool staged = stash && offload;
    if (!(recompute && stash)) {
      if (staged) SP_CUDA(cudaStreamWaitEvent(comp, ev_o_off[l], 0));  // last pass's copy-out of o_stage[l]
      SP_TRY(attention_forward(l, k, i, x, px));
      if (staged) {  // O/LSE of this slot-layer to the host, overlapping the rest of the pass
        SP_TRY(hand_off(comp, s_off));
        SP_CUDA(cudaMemcpyAsync(host_o(slot, l), x.o, Ls * qd * 2, cudaMemcpyDeviceToHost, s_off));
        SP_CUDA(cudaMemcpyAsync(host_l(slot, l), x.lse, int64_t(cfg.heads) * Ls * 4, cudaMemcpyDeviceToHost, s_off));
        SP_CUDA(cudaEventRecord(ev_o_off[l], s_off));
      }
    } else if (staged) {
      SP_CUDA(cudaStreamWaitEvent(comp, ev_o_in[l], 0));  // the backward's copy-in of this layer's stash
    }
    SP_TRY(gemm(false, true, Ls, h, qd, x.o, qd, W(P.wo), qd, x.x_mid, h, false, 1.f, 1.f, comp, x.x_in));
    SP_TRY(rmsnorm_fwd(x.x_mid, W(P.mlp_norm), x.xn2, x.rstd2, Ls, int(h), cfg.norm_eps, comp));
    SP_TRY(gemm(false, true, Ls, 2 * H, h, x.xn2, h, W(P.wgu), h, x.gu, 2 * H, false, 1.f, 0.f, comp));
    SP_TRY(swiglu_fwd(x.gu, x.act, Ls, int(H), comp));
    SP_TRY(gemm(false, true, Ls, h, H, x.act, H, W(P.wd), H, x_out, h, false, 1.f, 1.f, comp, x.x_mid));
    return SP_OK;
  }

  // Stage forward of slice (k,i) from ws[0].x_in; final output to `out`.
  int stage_forward(int k, int i, bf16raw* out, const PassX* px, bool recompute) {
    for (int l = 0; l < Lps; ++l) SP_TRY(layer_forward(l, k, i, l + 1 < Lps ? ws[l + 1].x_in : out, px, recompute));
    return SP_OK;
  }

  int run_forward(int pid, int k, int i, cudaEvent_t t0) {
    const PassX* px = pass_x(pid);
    if (px && !px->in.empty()) SP_TRY(post_remote(*px));
    if (free_slots.empty()) return set_error(SP_ERR_RUNTIME, "arena exhausted (ledger/schedule mismatch)");
    const int slot = free_slots.back();
    free_slots.pop_back();
    slot_of[sk(k, i)] = slot;
    slots_high_water = std::max(slots_high_water, ++slots_in_use);
    bf16raw* xs = offload ? x_stage : x_pool + int64_t(slot) * Ls * h;
    const int64_t tok0 = int64_t(k - 1) * cfg.seq_len + int64_t(i - 1) * Ls;
    if (offload) SP_CUDA(cudaStreamWaitEvent(comp, ev_x_off, 0));  // the last copy-out of x_stage is done
    if (stage == 1) {
      SP_CUDA(cudaEventRecord(t0, comp));
      SP_TRY(embed_fwd(tokens + tok0, W(emb), xs, Ls, int(h), comp));
    } else {
      // receive into a ring buffer as soon as one is free (decoupled from this
      // rank's compute progress), then copy into the slot at pass start
      const int b = ain_idx;
      ain_idx ^= 1;
      SP_CUDA(cudaStreamWaitEvent(s_act_in, ev_ain_free[b], 0));
      if (jit_recv) SP_TRY(link(comp, s_act_in));  // post the receive only when this pass starts
      SP_TRY(l_act_in->recv(ain_buf[b], Ls * h, ncclBfloat16, 0, s_act_in));
      SP_TRY(link(s_act_in, comp));
      SP_CUDA(cudaEventRecord(t0, comp));  // busy time starts once the input is here
      SP_CUDA(cudaMemcpyAsync(xs, ain_buf[b], Ls * h * 2, cudaMemcpyDeviceToDevice, comp));
      SP_CUDA(cudaEventRecord(ev_ain_free[b], comp));
    }
    SP_CUDA(cudaMemcpyAsync(ws[0].x_in, xs, Ls * h * 2, cudaMemcpyDeviceToDevice, comp));
    if (offload) {  // the stage input to the slot's host copy
      SP_TRY(hand_off(comp, s_off));
      SP_CUDA(cudaMemcpyAsync(host_x(slot), xs, Ls * h * 2, cudaMemcpyDeviceToHost, s_off));
      SP_CUDA(cudaEventRecord(ev_x_off, s_off));
    }
    if (stage < nst) {
      const int b = out_idx;
      out_idx ^= 1;
      SP_CUDA(cudaStreamWaitEvent(comp, ev_out_free[b], 0));
      SP_TRY(stage_forward(k, i, out_buf[b], px, false));
      SP_TRY(hand_off(comp, s_act_out));
      SP_TRY(timed_send(l_act_out.get(), out_buf[b], 1, s_act_out));
      SP_CUDA(cudaEventRecord(ev_out_free[b], s_act_out));
    } else {
      SP_TRY(stage_forward(k, i, x_final, px, false));
      if (vp) {  // x_final is overwritten by later passes: normalise into the slice's vocab slot now
        VSlot* vs = nullptr;
        SP_TRY(vslot_acquire(k, i, &vs));
        SP_TRY(rmsnorm_fwd(x_final, W(final_norm), vs->xf, rstd_f, Ls, int(h), cfg.norm_eps, comp));
      }
    }
    return SP_OK;
  }

  int vslot_acquire(int k, int i, VSlot** out) {
    auto it = vslot_of.find({k, i});
    if (it != vslot_of.end()) {
      *out = &vslots[it->second];
      return SP_OK;
    }
    if (vfree.empty()) return set_error(SP_ERR_RUNTIME, "vocab slots exhausted");
    const int vs_i = vfree.back();
    vfree.pop_back();
    vslot_of[{k, i}] = vs_i;
    *out = &vslots[vs_i];
    return SP_OK;
  }

  int layer_backward(int l, int k, int i, bf16raw* dx, const PassX* px) {
    bind_attn_out(l, slot_of.at(sk(k, i)));
    LayerWs& x = ws[l];
    const LayerParams& P = lp[lbase + l];
    const int64_t pos0 = int64_t(i - 1) * Ls;
    // MLP
    SP_TRY(gemm(false, false, Ls, H, h, dx, h, W(P.wd), H, tmp_H, H, false, 1.f, 0.f, comp));      // d_act
    SP_TRY(gemm(true, false, h, H, Ls, dx, h, x.act, H, G(P.wd), H, true, 1.f, 1.f, comp));         // dWd
    SP_TRY(swiglu_bwd(tmp_H, x.gu, tmp_2H, Ls, int(H), comp));                                      // d_gu
    SP_TRY(gemm(false, false, Ls, h, 2 * H, tmp_2H, 2 * H, W(P.wgu), h, tmp_h, h, false, 1.f, 0.f, comp));  // dxn2
    SP_TRY(gemm(true, false, 2 * H, h, Ls, tmp_2H, 2 * H, x.xn2, h, G(P.wgu), h, true, 1.f, 1.f, comp));    // dWgu
    SP_TRY(rmsnorm_bwd(tmp_h, x.x_mid, W(P.mlp_norm), x.rstd2, dx, dx, G(P.mlp_norm), Ls, int(h), comp, norm_ws));
    // attention output projection
    SP_TRY(gemm(false, false, Ls, qd, h, dx, h, W(P.wo), qd, tmp_h, qd, false, 1.f, 0.f, comp));   // d_o
    SP_TRY(gemm(true, false, h, qd, Ls, dx, h, x.o, qd, G(P.wo), qd, true, 1.f, 1.f, comp));         // dWo
    // K2: sliced attention backward (+ the pass's transfers: the receiver
    // returns dQ and dK/dV partials of the shipped chunks, added here)
    SP_CUDA(cudaMemsetAsync(dq_acc, 0, Ls * qd * 4, comp));
    std::vector<int32_t> rows, acc_rows;
    int causal = 1;
    own_chunks(k, i, px, rows, acc_rows, causal);
    const bool out = px && !px->out.empty();
    const int c = px ? px->cls : 1;
    const int64_t a = cfg.heads;
    SP_TRY(sp_attn_bwd_prep(x.o, qd, tmp_h, qd, x.lse, Ls, cfg.heads, cfg.head_dim, delta_ws, comp));
    if (out) {
      SP_TRY(link(comp, cx[c]));
      for (const XOut& xo : px->out) {
        SP_TRY(lx[c]->group_start());
        SP_TRY(lx[c]->send(x.q, Ls * qd, ncclBfloat16, xo.peer, cx[c]));
        SP_TRY(lx[c]->send(tmp_h, Ls * qd, ncclBfloat16, xo.peer, cx[c]));
        SP_TRY(lx[c]->send(delta_ws, 2 * a * Ls, ncclFloat32, xo.peer, cx[c]));
        SP_TRY(send_chunks(l, k, xo, c));
        SP_TRY(lx[c]->group_end());
        x_bytes_sent += 2 * Ls * qd * 2 + 2 * a * Ls * 4;
      }
    }
    AttnTimer t{};
    SP_TRY(timing_event(&t.a));
    SP_TRY(timing_event(&t.b));
    t.flops = 2.5 * attn_flops(int(rows.size()), causal);
    t.kind = 1;
    SP_CUDA(cudaEventRecord(t.a, comp));
    SP_TRY(attn_bwd_core(x.q, Ls, qd, k_pool[l], v_pool[l], int64_t(slots) * Ls, kvd, rows.data(), int(rows.size()),
                         int(Ls), cfg.heads, cfg.kv_heads, cfg.head_dim, causal, tmp_h, qd, delta_ws, dq_acc,
                         dk_acc[lbase + l], dv_acc[lbase + l], int64_t(cfg.slices) * Ls, acc_rows.data(), dkv_bf16,
                         comp));
    SP_CUDA(cudaEventRecord(t.b, comp));
    attn_times.push_back(t);
    if (out) {
      XBuf& b = xb[c];
      for (std::size_t tt = 0; tt < px->out.size(); ++tt) {
        const XOut& xo = px->out[tt];
        const int64_t nc = int64_t(xo.chunks.size());
        SP_TRY(lx[c]->group_start());
        SP_TRY(lx[c]->recv(b.dq_rem + tt * Ls * qd, Ls * qd, ncclFloat32, xo.peer, cx[c]));
        SP_TRY(lx[c]->recv(b.dk_rem + int64_t(xo.base) * Ls * kvd, nc * Ls * kvd, ncclFloat32, xo.peer, cx[c]));
        SP_TRY(lx[c]->recv(b.dv_rem + int64_t(xo.base) * Ls * kvd, nc * Ls * kvd, ncclFloat32, xo.peer, cx[c]));
        SP_TRY(lx[c]->group_end());
      }
      SP_TRY(link(cx[c], comp));
      for (std::size_t tt = 0; tt < px->out.size(); ++tt) {
        const XOut& xo = px->out[tt];
        SP_TRY(add_f32(dq_acc, b.dq_rem + tt * Ls * qd, Ls * qd, comp));
        for (std::size_t x2 = 0; x2 < xo.chunks.size(); ++x2) {
          const int64_t dst = int64_t(xo.chunks[x2] - 1) * Ls * kvd, src = int64_t(xo.base + x2) * Ls * kvd;
          if (dkv_bf16) {
            SP_TRY(add_to_bf16(acc_at(dk_acc[lbase + l], dst), b.dk_rem + src, Ls * kvd, comp));
            SP_TRY(add_to_bf16(acc_at(dv_acc[lbase + l], dst), b.dv_rem + src, Ls * kvd, comp));
          } else {
            SP_TRY(add_f32(static_cast<float*>(acc_at(dk_acc[lbase + l], dst)), b.dk_rem + src, Ls * kvd, comp));
            SP_TRY(add_f32(static_cast<float*>(acc_at(dv_acc[lbase + l], dst)), b.dv_rem + src, Ls * kvd, comp));
          }
        }
      }
    }
    // chunk i's dK/dV is complete: RoPE backward into d_qkv and reset the rows
    SP_TRY(rope_qkv_bwd(dq_acc, acc_at(dk_acc[lbase + l], pos0 * kvd), acc_at(dv_acc[lbase + l], pos0 * kvd), kvd, Ls,
                        cfg.heads, cfg.kv_heads,
                        cfg.head_dim, pos0, rope_cos, rope_sin, dqkv, 1, comp, dkv_bf16));
    SP_TRY(gemm(false, false, Ls, h, qkv_w, dqkv, qkv_w, W(P.wqkv), h, tmp_h, h, false, 1.f, 0.f, comp));   // dxn
    SP_TRY(gemm(true, false, qkv_w, h, Ls, dqkv, qkv_w, x.xn, h, G(P.wqkv), h, true, 1.f, 1.f, comp));      // dWqkv
    SP_TRY(rmsnorm_bwd(tmp_h, x.x_in, W(P.attn_norm), x.rstd1, dx, dx, G(P.attn_norm), Ls, int(h), comp, norm_ws));
    return SP_OK;
  }

  // VocabForward(k,i): final hidden state of the slice from the last stage
  // (broadcast), logits of this shard, softmax statistics all-reduced.
  int run_vocab_fwd(int k, int i, cudaEvent_t t0) {
    SP_CUDA(cudaEventRecord(t0, comp));
    VSlot* vsp = nullptr;
    SP_TRY(vslot_acquire(k, i, &vsp));  // on the last stage F(k,i,p) already filled xf
    VSlot& vs = *vsp;
    const int64_t tok0 = int64_t(k - 1) * cfg.seq_len + int64_t(i - 1) * Ls;
    SP_TRY(link(comp, s_vocab));
    SP_TRY(vlink->broadcast(vs.xf, Ls * h, ncclBfloat16, p - 1, s_vocab));
    SP_TRY(link(s_vocab, comp));
    SP_TRY(gemm(false, true, Ls, Vs, h, vs.xf, h, W(head), h, vlogits, Vs, true, 1.f, 0.f, comp));
    float* m_loc = vs.st;
    float* m_glob = vs.st + Ls;
    float* zt = vs.st + 2 * Ls;
    SP_TRY(xent_shard_stats(vlogits, targets + tok0, Ls, int(Vs), int(v0), m_loc, m_glob, zt, comp));
    SP_TRY(link(comp, s_vocab));
    SP_TRY(vlink->all_reduce(m_glob, Ls, ncclMax, s_vocab));
    SP_TRY(link(s_vocab, comp));
    SP_TRY(xent_shard_rescale(m_loc, m_glob, zt, Ls, comp));
    SP_TRY(link(comp, s_vocab));
    SP_TRY(vlink->all_reduce(zt, 2 * Ls, ncclSum, s_vocab));
    SP_TRY(link(s_vocab, comp));
    return SP_OK;
  }

  // VocabBackward(k,i): shard dlogits (softmax - onehot), dW_head of the
  // shard, partial dX of the final hidden state reduced onto the last stage.
  int run_vocab_bwd(int k, int i, cudaEvent_t t0) {
    SP_CUDA(cudaEventRecord(t0, comp));
    const int vs_i = vslot_of.at({k, i});
    VSlot& vs = vslots[vs_i];
    const int64_t tok0 = int64_t(k - 1) * cfg.seq_len + int64_t(i - 1) * Ls;
    SP_TRY(gemm(false, true, Ls, Vs, h, vs.xf, h, W(head), h, vlogits, Vs, true, 1.f, 0.f, comp));
    const float scale = 1.f / float(int64_t(cfg.microbatches) * cfg.seq_len);
    SP_TRY(xent_shard_grad(vlogits, targets + tok0, Ls, int(Vs), int(v0), vs.st + Ls, vs.st + 2 * Ls, scale, vdlog,
                           last_dev ? loss_dev : nullptr, comp));
    SP_TRY(gemm(false, false, Ls, h, Vs, vdlog, Vs, W(head), h, vdxf, h, true, 1.f, 0.f, comp));  // partial dX
    SP_TRY(gemm(true, false, Vs, h, Ls, vdlog, Vs, vs.xf, h, G(head), h, true, 1.f, 1.f, comp));    // dW shard
    SP_TRY(link(comp, s_vocab));
    SP_TRY(vlink->reduce(vdxf, Ls * h, p - 1, s_vocab));
    SP_TRY(link(s_vocab, comp));
    vfree.push_back(vs_i);
    vslot_of.erase({k, i});
    return SP_OK;
  }

  int run_backward(int pid, int k, int i, cudaEvent_t t0) {
    const PassX* px = pass_x(pid);
    if (px && !px->in.empty()) SP_TRY(post_remote(*px));
    const int slot = slot_of.at(sk(k, i));
    bf16raw* xs = offload ? x_stage : x_pool + int64_t(slot) * Ls * h;
    const int64_t tok0 = int64_t(k - 1) * cfg.seq_len + int64_t(i - 1) * Ls;
    if (offload) {  // bring the slot's stash back (after every earlier use of the staging)
      SP_TRY(hand_off(comp, s_off));
      SP_CUDA(cudaMemcpyAsync(x_stage, host_x(slot), Ls * h * 2, cudaMemcpyHostToDevice, s_off));
      SP_CUDA(cudaEventRecord(ev_x_in, s_off));
      if (stash)
        for (int l = 0; l < Lps; ++l) {
          SP_CUDA(cudaMemcpyAsync(o_stage[l], host_o(slot, l), Ls * qd * 2, cudaMemcpyHostToDevice, s_off));
          SP_CUDA(cudaMemcpyAsync(l_stage[l], host_l(slot, l), int64_t(cfg.heads) * Ls * 4, cudaMemcpyHostToDevice,
                                  s_off));
          SP_CUDA(cudaEventRecord(ev_o_in[l], s_off));
        }
    }
    // gradient input
    bf16raw* dx = nullptr;
    int gb = -1;
    if (stage < nst) {
      gb = gin_idx;
      gin_idx ^= 1;
      dx = gin_buf[gb];
      SP_CUDA(cudaStreamWaitEvent(s_grad_in, ev_gin_free[gb], 0));
      if (jit_recv) SP_TRY(link(comp, s_grad_in));
      SP_TRY(l_grad_in->recv(dx, Ls * h, ncclBfloat16, 1, s_grad_in));
      SP_TRY(hand_off(s_grad_in, comp));
      SP_CUDA(cudaEventRecord(t0, comp));
    } else {
      SP_CUDA(cudaEventRecord(t0, comp));
      dx = gout_buf[gout_idx];  // last stage: dX is produced here, sent from here
    }
    // recompute (Full checkpointing)
    if (offload) SP_CUDA(cudaStreamWaitEvent(comp, ev_x_in, 0));
    SP_CUDA(cudaMemcpyAsync(ws[0].x_in, xs, Ls * h * 2, cudaMemcpyDeviceToDevice, comp));
    bf16raw* top = stage < nst ? tmp_h : x_final;
    if (stage == nst) {
      SP_CUDA(cudaStreamWaitEvent(comp, ev_gout_free[gout_idx], 0));
      SP_TRY(stage_forward(k, i, x_final, px, true));
      if (vp) {  // dX of the final hidden state = sum of the shards' partials (VocabBackward, just before)
        SP_TRY(rmsnorm_fwd(x_final, W(final_norm), xf, rstd_f, Ls, int(h), cfg.norm_eps, comp));
        SP_TRY(f32_to_bf16(vdxf, tmp_h, Ls * h, comp));
        SP_TRY(rmsnorm_bwd(tmp_h, x_final, W(final_norm), rstd_f, nullptr, dx, G(final_norm), Ls, int(h), comp, norm_ws));
      }
    }
    if (stage == nst && !vp) {
      // LM head + cross entropy
      const int64_t V = cfg.vocab;
      SP_TRY(rmsnorm_fwd(x_final, W(final_norm), xf, rstd_f, Ls, int(h), cfg.norm_eps, comp));
      SP_TRY(gemm(false, true, Ls, V, h, xf, h, W(head), h, logits, V, true, 1.f, 0.f, comp));
      const float scale = 1.f / float(int64_t(cfg.microbatches) * cfg.seq_len);
      SP_TRY(cross_entropy(logits, targets + tok0, Ls, int(V), scale, dlogits, loss_dev, comp));
      SP_TRY(gemm(false, false, Ls, h, V, dlogits, V, W(head), h, tmp_h, h, false, 1.f, 0.f, comp));  // dxf
      SP_TRY(gemm(true, false, V, h, Ls, dlogits, V, xf, h, G(head), h, true, 1.f, 1.f, comp));        // dWhead
      SP_TRY(rmsnorm_bwd(tmp_h, x_final, W(final_norm), rstd_f, nullptr, dx, G(final_norm), Ls, int(h), comp, norm_ws));
    } else if (stage < nst) {
      SP_TRY(stage_forward(k, i, top, px, true));
    }
    for (int l = Lps - 1; l >= 0; --l) SP_TRY(layer_backward(l, k, i, dx, px));
    if (stage == 1) {
      SP_TRY(embed_bwd(tokens + tok0, dx, G(emb), Ls, int(h), comp));
      if (gb >= 0) SP_CUDA(cudaEventRecord(ev_gin_free[gb], comp));
    } else {
      SP_TRY(hand_off(comp, s_grad_out));
      SP_TRY(timed_send(l_grad_out.get(), dx, 0, s_grad_out));
      if (gb >= 0) {  // middle stage: dx lives in the receive buffer
        SP_CUDA(cudaEventRecord(ev_gin_free[gb], s_grad_out));
      } else {        // last stage: dx lives in gout_buf[gout_idx]
        SP_CUDA(cudaEventRecord(ev_gout_free[gout_idx], s_grad_out));
        gout_idx ^= 1;
      }
    }
    free_slots.push_back(slot);  // LIFO reuse
    slot_of.erase(sk(k, i));
    --slots_in_use;
    return SP_OK;
  }

  int step(const int32_t* tok, const int32_t* tgt, int on_device, int flags, float* loss_out) {
    SP_CUDA(cudaSetDevice(device));
    times.clear();
    attn_times.clear();
    comm_times.clear();
    tpool_i = 0;
    slots_high_water = 0;
    x_bytes_sent = 0;
    const int64_t ntok = int64_t(cfg.microbatches) * cfg.seq_len;
    SP_CUDA(cudaEventRecord(step_start, comp));
    // Host inputs go through pinned staging buffers: a pageable copy would
    // block this thread inside the CUDA driver until the stream drained (and,
    // with loopback ranks sharing one context, stall the other ranks' enqueue).
    const bool need_tok = first_dev && tok, need_tgt = (last_dev || vp) && tgt;
    if (on_device) {
      if (need_tok) SP_CUDA(cudaMemcpyAsync(tokens, tok, ntok * 4, cudaMemcpyDeviceToDevice, comp));
      if (need_tgt) SP_CUDA(cudaMemcpyAsync(targets, tgt, ntok * 4, cudaMemcpyDeviceToDevice, comp));
    } else if (need_tok || need_tgt) {
      SP_CUDA(cudaEventSynchronize(ev_staged));  // the previous step's copies have left the staging buffers
      if (need_tok) {
        std::memcpy(h_tok, tok, size_t(ntok) * 4);
        SP_CUDA(cudaMemcpyAsync(tokens, h_tok, ntok * 4, cudaMemcpyHostToDevice, comp));
      }
      if (need_tgt) {
        std::memcpy(h_tgt, tgt, size_t(ntok) * 4);
        SP_CUDA(cudaMemcpyAsync(targets, h_tgt, ntok * 4, cudaMemcpyHostToDevice, comp));
      }
      SP_CUDA(cudaEventRecord(ev_staged, comp));
    }
    SP_CUDA(cudaMemsetAsync(loss_dev, 0, 4, comp));
    for (pipelab::PassId id : order) {
      const pipelab::Pass& ps = sched.passes[id];
      enq_pos = int(times.size());
      PassTime t{id, nullptr, nullptr};
      if (ps.kind == pipelab::PassKind::Forward || ps.kind == pipelab::PassKind::BackwardFused) {
        stage = ps.stage;
        cur = (stage - 1) / p;
        lbase = cur * Lps;
      }
      SP_TRY(timing_event(&t.start));
      SP_TRY(timing_event(&t.end));
      if (ps.kind == pipelab::PassKind::Forward) SP_TRY(run_forward(id, ps.microbatch, ps.slice, t.start));
      else if (ps.kind == pipelab::PassKind::VocabForward) SP_TRY(run_vocab_fwd(ps.microbatch, ps.slice, t.start));
      else if (ps.kind == pipelab::PassKind::VocabBackward) SP_TRY(run_vocab_bwd(ps.microbatch, ps.slice, t.start));
      else SP_TRY(run_backward(id, ps.microbatch, ps.slice, t.start));
      SP_CUDA(cudaEventRecord(t.end, comp));
      times.push_back(t);
    }
    if (!(flags & SP_STEP_NO_OPTIMIZER)) {
      ++opt_step;
      SP_TRY(adamw(master, w, grad, adam_m, adam_v, n_params, cfg.lr, 0.9f, 0.95f, 1e-8f, 0.1f, opt_step, comp));
      SP_CUDA(cudaMemsetAsync(grad, 0, n_params * 4, comp));
    }
    enq_pos = -1;
    // drain comm streams into the compute stream so step_end covers them
    for (cudaStream_t st : {s_act_in, s_act_out, s_grad_in, s_grad_out}) SP_TRY(hand_off(st, comp));
    if (s_off) SP_TRY(hand_off(s_off, comp));
    for (int c = 0; c < 2; ++c)
      if (cx[c]) {
        SP_TRY(link(cx[c], comp));
        SP_TRY(link(rx[c], comp));
      }
    if (s_vocab) SP_TRY(link(s_vocab, comp));
    SP_CUDA(cudaEventRecord(step_end, comp));
    if (loss_out) {
      SP_CUDA(cudaMemcpyAsync(h_loss, loss_dev, 4, cudaMemcpyDeviceToHost, comp));
      SP_CUDA(cudaStreamSynchronize(comp));
      *loss_out = last_dev ? *h_loss / float(ntok) : 0.f;
    }
    return SP_OK;
  }
};

}  // namespace
}  // namespace sp

using sp::Runtime;

extern "C" {

int sp_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return sp::set_error(SP_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  std::memcpy(out128, &id, sizeof id);
  return SP_OK;
}

int sp_runtime_create(const sp_model_config* cfg, const void* nccl_ids, void** handle) {
  auto rt = std::make_unique<Runtime>();
  const int rc = rt->init(*cfg, nccl_ids);
  if (rc != SP_OK) return rc;
  *handle = rt.release();
  return SP_OK;
}

int sp_runtime_create_loopback(const sp_model_config* cfg, void* world, void** handle) {
  if (!world) return sp::set_error(SP_ERR_INVALID, "loopback world is null");
  auto rt = std::make_unique<Runtime>();
  const int rc = rt->init(*cfg, nullptr, static_cast<sp::LoopWorld*>(world));
  if (rc != SP_OK) return rc;
  *handle = rt.release();
  return SP_OK;
}

int sp_runtime_destroy(void* handle) {
  if (handle) cudaSetDevice(static_cast<Runtime*>(handle)->device);
  delete static_cast<Runtime*>(handle);
  return SP_OK;
}

int sp_runtime_step(void* handle, const int32_t* tokens, const int32_t* targets, int on_device, int flags,
                    float* loss) {
  return static_cast<Runtime*>(handle)->step(tokens, targets, on_device, flags, loss);
}

// Diagnostics: index (in device order) of the first pass whose end event has
// not completed on the compute stream, or -1 when all have; writes that
// pass's (kind, microbatch, slice, stage) to out4.
int sp_runtime_progress(void* handle, int32_t* out4) {
  if (handle) cudaSetDevice(static_cast<Runtime*>(handle)->device);
  Runtime* rt = static_cast<Runtime*>(handle);
  for (std::size_t x = 0; x < rt->times.size(); ++x) {
    if (cudaEventQuery(rt->times[x].end) == cudaErrorNotReady) {
      const pipelab::Pass& q = rt->sched.passes[size_t(rt->times[x].pass)];
      out4[0] = int32_t(q.kind), out4[1] = q.microbatch, out4[2] = q.slice, out4[3] = q.stage;
      return int(x);
    }
  }
  return -1;
}

int sp_runtime_enqueue_position(void* handle) { return static_cast<Runtime*>(handle)->enq_pos.load(); }

int sp_runtime_sync(void* handle) {
  if (handle) cudaSetDevice(static_cast<Runtime*>(handle)->device);
  return sp::cuda_status(cudaStreamSynchronize(static_cast<Runtime*>(handle)->comp), "sync");
}

void* sp_runtime_stream(void* handle) { return static_cast<Runtime*>(handle)->comp; }

// Step time (ms between step_start and step_end) and per-pass busy times.
// out: [0] step ms, then per pass of device_order: pass id, start ms, end ms.
int sp_runtime_timeline(void* handle, double* out, int cap) {
  if (handle) cudaSetDevice(static_cast<Runtime*>(handle)->device);
  Runtime* rt = static_cast<Runtime*>(handle);
  cudaError_t e = cudaEventSynchronize(rt->step_end);
  if (e != cudaSuccess) return sp::cuda_status(e, "timeline");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, rt->step_start, rt->step_end);
  int n = 0;
  if (cap > 0) out[n++] = ms;
  for (const auto& t : rt->times) {
    if (n + 3 > cap) break;
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, rt->step_start, t.start);
    cudaEventElapsedTime(&b, rt->step_start, t.end);
    out[n++] = t.pass;
    out[n++] = a;
    out[n++] = b;
  }
  return n;
}

// Attention kernel timing of the last step: out = {fwd_ms, fwd_flops, fwd_launches,
// bwd_ms, bwd_flops, bwd_launches}.
int sp_runtime_attn_stats(void* handle, double* out6) {
  if (handle) cudaSetDevice(static_cast<Runtime*>(handle)->device);
  Runtime* rt = static_cast<Runtime*>(handle);
  for (int x = 0; x < 6; ++x) out6[x] = 0.0;
  for (const auto& t : rt->attn_times) {
    float ms = 0.f;
    cudaEventSynchronize(t.b);
    cudaEventElapsedTime(&ms, t.a, t.b);
    out6[3 * t.kind] += ms;
    out6[3 * t.kind + 1] += t.flops;
    out6[3 * t.kind + 2] += 1;
  }
  return SP_OK;
}

// Stage sends of the last step: out4 = {messages, bytes, total ms, fastest
// message ms} (CUDA events on the send streams).
int sp_runtime_comm_stats(void* handle, double* out4) {
  if (handle) cudaSetDevice(static_cast<Runtime*>(handle)->device);
  Runtime* rt = static_cast<Runtime*>(handle);
  double n = 0, bytes = 0, ms = 0, best = 0;
  for (const auto& t : rt->comm_times) {
    float x = 0.f;
    cudaError_t e = cudaEventSynchronize(t.b);
    if (e != cudaSuccess) return sp::cuda_status(e, "comm stats");
    cudaEventElapsedTime(&x, t.a, t.b);
    n += 1;
    bytes += double(t.bytes);
    ms += x;
    best = (best == 0 || x < best) ? x : best;
  }
  out4[0] = n, out4[1] = bytes, out4[2] = ms, out4[3] = best;
  return SP_OK;
}

int sp_runtime_exchange_stats(void* handle, int64_t* out3) {
  Runtime* rt = static_cast<Runtime*>(handle);
  int64_t o = 0, i = 0;
  for (const auto& kv : rt->xplan) {
    o += kv.second.out.empty() ? 0 : 1;
    i += kv.second.in.empty() ? 0 : 1;
  }
  out3[0] = o;
  out3[1] = i;
  out3[2] = rt->x_bytes_sent;
  return SP_OK;
}

// {slots, slots_high_water, slot_bytes, ledger_peak_units, bytes_allocated, n_params, layers_per_stage}
int sp_runtime_recompute(void* handle) { return static_cast<Runtime*>(handle)->stash ? 0 : 1; }

long long sp_runtime_offload_bytes(void* handle) {
  return static_cast<long long>(static_cast<Runtime*>(handle)->offload_bytes);
}

int sp_runtime_memory(void* handle, int64_t* out7) {
  Runtime* rt = static_cast<Runtime*>(handle);
  out7[0] = rt->slots;
  out7[1] = rt->slots_high_water;
  // device bytes per slot: K/V per layer, plus the stage input and O/LSE
  // stash unless they are offloaded to the host
  out7[2] = int64_t(rt->Lps) * 2 * rt->Ls * rt->kvd * 2 +
            (rt->offload ? 0
                         : rt->Ls * rt->h * 2 +
                               (rt->stash ? int64_t(rt->Lps) * rt->Ls * (rt->qd * 2 + int64_t(rt->cfg.heads) * 4) : 0));
  out7[3] = rt->ledger.per_device[rt->rank].peak_activation_units;
  out7[4] = int64_t(rt->bytes_allocated);
  out7[5] = rt->n_params;
  out7[6] = rt->Lps;
  return SP_OK;
}

// Copy parameter tensors / gradients between host fp32 buffers and the device.
// which: 0 attn_norm 1 wqkv 2 wo 3 mlp_norm 4 wgu 5 wd 6 embedding 7 final_norm 8 head
// dir: 0 device->host (master weights), 1 host->device (sets master + bf16), 2 grads device->host
int sp_runtime_param(void* handle, int layer, int which, float* host, int64_t count, int dir) {
  if (handle) cudaSetDevice(static_cast<Runtime*>(handle)->device);
  Runtime* rt = static_cast<Runtime*>(handle);
  int64_t off = -1, n = 0;
  const int64_t h = rt->h, H = rt->H;
  if (which <= 5) {
    if (layer < 0 || layer >= rt->v * rt->Lps)  // local index c*Lps + l (stage rank+1+c*p, its layer l)
      return sp::set_error(SP_ERR_INVALID, "layer %d not on this device", layer);
    const sp::LayerParams& P = rt->lp[layer];
    const int64_t offs[6] = {P.attn_norm, P.wqkv, P.wo, P.mlp_norm, P.wgu, P.wd};
    const int64_t ns[6] = {h, rt->qkv_w * h, h * rt->qd, h, 2 * H * h, h * H};
    off = offs[which];
    n = ns[which];
  } else if (which == 6) {
    off = rt->emb, n = int64_t(rt->cfg.vocab) * h;
  } else if (which == 7) {
    off = rt->final_norm, n = h;
  } else if (which == 8) {  // the full head, or this stage's vocab shard under vocab parallelism
    off = rt->head, n = (rt->vp ? rt->Vs : int64_t(rt->cfg.vocab)) * h;
  }
  if (off < 0) return sp::set_error(SP_ERR_INVALID, "parameter %d not on this stage", which);
  if (count != n) return sp::set_error(SP_ERR_INVALID, "parameter size %lld != %lld", (long long)count, (long long)n);
  cudaError_t e;
  if (dir == 0) e = cudaMemcpy(host, rt->master + off, n * 4, cudaMemcpyDeviceToHost);
  else if (dir == 2) e = cudaMemcpy(host, rt->grad + off, n * 4, cudaMemcpyDeviceToHost);
  else {
    e = cudaMemcpy(rt->master + off, host, n * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
      int rc = sp::f32_to_bf16(rt->master + off, rt->w + off, n, rt->comp);
      if (rc) return rc;
      e = cudaStreamSynchronize(rt->comp);
    }
  }
  return sp::cuda_status(e, "sp_runtime_param");
}

}  // extern "C"
