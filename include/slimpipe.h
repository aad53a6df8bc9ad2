/* slimpipe.h — the C-ABI of libslimpipe.so, the B200 SlimPipe step.
 *
 * Two halves:
 *   1. Planning (host C++, behind the pipelab headers in include/pipelab/):
 *      exposed here as JSON-text entry points for the Python host mirror and
 *      the parity tests.  The C++ API itself (gen_slimpipe, validate_schedule,
 *      balance_tick, apply_exchange, simulate, ...) is the drop-in for
 *      reference proj/include/pipelab/{schedule,exchange,simulator,workload}.hpp.
 *   2. Device (sm_100a CUDA + NCCL): the replacements for what the reference
 *      only models —
 *        reference proj/src/attention.cpp:21-111  (chunked online-softmax
 *            attention, fp64, forward only)      -> sp_attn_fwd / sp_attn_bwd /
 *                                                   sp_attn_merge
 *        reference proj/src/simulator.cpp:311-346 (slice memory ledger)
 *                                                -> the runtime's HBM slot arena
 *        reference proj/src/simulator.cpp:156-207, 275-309 (exchange transfers,
 *            CommModel simulator.hpp:23-34)      -> sp_exchange_* + NCCL P2P
 *        reference proj/src/schedule.cpp:102-130 cross-device edges
 *                                                -> stage P2P in sp_runtime_step
 *
 * Conventions: status codes (SP_OK == 0), never exceptions; device pointers
 * are plain addresses of caller-owned buffers; `stream` is a cudaStream_t
 * (0 = legacy default stream); bf16 buffers are passed as void*.
 * One host thread per GPU; handles are not thread-safe.
 */
#ifndef SLIMPIPE_H
#define SLIMPIPE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* sp_stream_t; /* cudaStream_t */

enum {
  SP_OK = 0,
  SP_ERR_INVALID = 1,     /* reference: std::invalid_argument */
  SP_ERR_RUNTIME = 2,     /* reference: std::runtime_error    */
  SP_ERR_CUDA = 3,
  SP_ERR_NCCL = 4,
  SP_ERR_UNSUPPORTED = 5, /* shape outside what the kernels implement */
  SP_ERR_NO_DEVICE = 6
};

const char* sp_status_string(int code);
const char* sp_last_error(void); /* message of the last failing call on this thread */
void sp_free(char* p);
int sp_version(void);
long long sp_launch_count(void);         /* kernels launched by this library so far */
long long sp_library_launch_count(void); /* cuBLASLt GEMM calls so far */
/* GEMM plans so far (JSON list: shape, cuBLASLt candidates, the one kept,
 * its time and the heuristic's first choice's; the runtime times candidates
 * during its create-time warm-up).  Free with sp_free. */
int sp_gemm_plans_json(char** out);

/* ---------------------------------------------------------------- planning
 * scheme: 0 gpipe 1 terapipe 2 1f1b 3 interleaved_1f1b 4 zbv 5 vhalf 6 slimpipe
 * mode:   0 off 1 on 2 early.  *out receives a malloc'd JSON string (free with
 * sp_free) — on error a {"error": kind, "what": message} object. */
int sp_plan_schedule_json(int scheme, int p, int v, int m, int n, char** out);
/* reference schedule.cpp:413-579; mutation 0 none, 1 swap BW(1,2)/BW(1,1) on
 * device 1, 2 drop the last pass of device 2, 3 add a cycle-closing edge */
int sp_plan_validate_json(int p, int v, int m, int n, int mutation, char** out);
/* reference exchange.cpp:10-96 */
int sp_plan_balance_json(const int64_t* loads, const int32_t* devices, int count, int early, char** out);
/* reference simulator.cpp:56-108 */
int sp_plan_exchange_json(int p, int v, int m, int n, int mode, double beta_attn, char** out);
/* The executor's per-pass exchange wiring for one rank (0-based): the plan of
 * sp_plan_exchange_json (v = 1) after the placement filter of sp_model_config
 * (exchange_min_chunks, exchange_skip_last) — JSON list of {pass, kind,
 * microbatch, slice, cls, out: [{peer, base, chunks}], in: [{peer, i_src,
 * base, chunks}]}, exactly what sp_runtime_create builds. */
int sp_exchange_passes_json(int p, int m, int n, int mode, int rank, int min_chunks, int skip_last, char** out);
/* reference workload.cpp:87-141; model={L,h,H,a,g,V,bytes,loss_bytes},
 * par={t,c,p,v}, run={S,m,n,ckpt(0 none,1 selective,2 full)} */
int sp_plan_activation_json(const int64_t* model, const int64_t* par, const int64_t* run, double offload,
                            char** out);
/* reference exchange.cpp:98-111 */
int sp_plan_exchange_volume(int64_t p, int64_t n, int64_t layers, int64_t mh_num, int64_t mh_den, char** out);
/* reference simulator.cpp:110-412; cost={alpha,beta,bwd_in,bwd_w},
 * comm={bandwidth,latency}; mem_rats = 6 (num,den) pairs or NULL (unit model) */
int sp_plan_simulate_json(int p, int v, int m, int n, int mode, const double* cost, const double* comm,
                          int64_t seq_len, const int64_t* mem_rats, char** out);
/* reference simulator.cpp:414-522 (place_vocab) on gen_slimpipe(p, v, m, n),
 * base-simulation costs alpha (per token) and beta (per query-key pair):
 * {"valid", "violations", "order": per device [[kind, microbatch, slice, stage], ...]} */
int sp_plan_vocab_json(int p, int v, int m, int n, int distribute, double alpha, double beta, int64_t seq_len,
                       char** out);
/* reference scenario.cpp:72-193: scenario text -> normalised scenario JSON
 * (strict: unknown fields / bad values are SP_ERR_INVALID) */
int sp_plan_scenario_json(const char* text, char** out);
/* reference gantt.cpp:52-106 on simulate(gen_slimpipe(p,v,m,n)) (inputs as
 * sp_plan_simulate_json, unit memory model); svg != 0: the SVG form */
int sp_plan_gantt_json(int p, int v, int m, int n, int mode, const double* cost, const double* comm,
                       int64_t seq_len, int svg, char** out);
/* the same export for a measured step: per-device CUDA-event spans (counts[d]
 * entries of pass id / start / end, devices concatenated) against the
 * executor's schedule */
/* the reference's metric definitions (simulator.cpp:348-409) on a measured
 * step (inputs as sp_plan_gantt_measured): makespan, bubble, busy, idle, phases */
int sp_plan_metrics_measured(int p, int v, int m, int n, int vocab_parallel, int64_t seq_len, const int32_t* counts,
                             const int32_t* pass_ids, const double* starts, const double* ends, char** out);
int sp_plan_gantt_measured(int p, int v, int m, int n, int vocab_parallel, int64_t seq_len, const int32_t* counts,
                           const int32_t* pass_ids, const double* starts, const double* ends, int svg, char** out);

/* ------------------------------------------------- sliced causal attention
 * Replaces reference attention.cpp:94-111 (chunk_attention) for the
 * multi-head bf16 slice layout of the step:
 *   q      bf16 [q_rows][q_stride]   head h occupies columns [h*d, (h+1)*d)
 *   k_pool bf16 [pool_rows][kv_stride], v_pool likewise; kv head g at [g*d,...)
 *   chunk_row[c] (host array, n_chunks <= SP_MAX_CHUNKS): first pool row of the
 *          c-th KV chunk, in attention order; every chunk has chunk_len rows
 *   causal: query row r attends global key positions
 *          <= n_chunks*chunk_len - q_rows + r (reference attention.cpp:34-35,
 *          bottom-right aligned) — only the last chunk is ever masked
 *   o      bf16 [q_rows][o_stride] normalised output (finalize, :84-92)
 *   lse    fp32 [heads][q_rows]  natural-log row log-sum-exp of the scaled
 *          scores (row_max + log(row_sumexp)); -inf for fully masked rows
 * Query head h reads kv head h / (heads / kv_heads).
 * Requirements: head_dim in {64, 128}; q_rows, chunk_len multiples of 128;
 * strides multiples of 8 elements.  The chunk table travels in kernel
 * parameter space (SP_MAX_CHUNKS entries). */
#define SP_MAX_CHUNKS 256
int sp_attn_fwd(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks, int chunk_len,
                int heads, int kv_heads, int head_dim, int causal, void* o, int64_t o_stride, float* lse,
                sp_stream_t stream);

/* sp_attn_fwd with the mask and scale spelled out — what the pipelab
 * attention API (attention.hpp: arbitrary rows, chunk lengths, head_dim <=
 * 128, chunks at any position) runs after padding to the kernel tiles:
 *   causal: query row r sees keys <= r + causal_off (sp_attn_fwd uses
 *           total_kv - q_rows, reference attention.cpp:34-35);
 *   keys >= kv_valid are masked (padding; kv_valid <= n_chunks*chunk_len);
 *   scale: softmax scale (reference 1/sqrt(d) of the UNPADDED head_dim, :31);
 *   row_max (optional, fp32 [heads][q_rows]): the true row max of the scaled
 *           scores, so the caller can form the reference's unnormalised state
 *           (row_sumexp = exp(lse - row_max), partial = O * row_sumexp). */
int sp_attn_fwd_masked(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                       int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks, int chunk_len,
                       int heads, int kv_heads, int head_dim, int causal, int64_t causal_off, int64_t kv_valid,
                       double scale, void* o, int64_t o_stride, float* lse, float* row_max, sp_stream_t stream);

/* Backward of sp_attn_fwd.  Accumulates (+=) into fp32 buffers:
 *   dq_acc  fp32 [q_rows][heads*head_dim]
 *   dk_acc, dv_acc fp32 pools [acc_rows][kv_heads*head_dim]; chunk c's rows
 *           start at acc_row[c] (host array)
 * delta_ws: fp32 [2][heads][q_rows] scratch (lse*log2e, then rowsum(dO*O)).
 * Runs slices n..1 in the step so a chunk's dK/dV is complete when its own
 * slice's backward runs (reference schedule.cpp:125-126 edge order). */
int sp_attn_bwd(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks, int chunk_len,
                int heads, int kv_heads, int head_dim, int causal, const void* o, int64_t o_stride,
                const void* dout, int64_t do_stride, const float* lse, float* delta_ws, float* dq_acc,
                float* dk_acc, float* dv_acc, int64_t acc_rows, const int32_t* acc_row, sp_stream_t stream);

/* The two halves of sp_attn_bwd, for callers that ship the row statistics to
 * a peer (workload redistribution): prep writes stats = [lse*log2e ; delta]
 * (fp32 [2][heads][q_rows]); core consumes them (no O needed). */
int sp_attn_bwd_prep(const void* o, int64_t o_stride, const void* dout, int64_t do_stride, const float* lse,
                     int64_t q_rows, int heads, int head_dim, float* stats, sp_stream_t stream);
int sp_attn_bwd_core(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                     int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks, int chunk_len,
                     int heads, int kv_heads, int head_dim, int causal, const void* dout, int64_t do_stride,
                     const float* stats, float* dq_acc, float* dk_acc, float* dv_acc, int64_t acc_rows,
                     const int32_t* acc_row, sp_stream_t stream);

/* Online-softmax merge of two normalised partials over disjoint key sets
 * (reference merge_partials attention.cpp:63-82 followed by finalize :84-92):
 *   w_x = exp(lse_x - max), o = (w_a o_a + w_b o_b) / (w_a + w_b),
 *   lse = max + log(w_a + w_b); rows where both are -inf stay 0 / -inf.
 * o_out/lse_out may alias o_a/lse_a. */
int sp_attn_merge(const void* o_a, const float* lse_a, const void* o_b, const float* lse_b, int64_t rows,
                  int heads, int head_dim, int64_t o_stride, void* o_out, float* lse_out, sp_stream_t stream);

/* Host fp64 entry of the pipelab attention API (include/pipelab/attention.hpp,
 * reference attention.hpp:41-61) for one head: q [rows][d], k/v the chunks'
 * rows concatenated, chunk_lens[n_chunks].  streamed = 0: chunk_attention;
 * 1: accumulate_chunk per chunk + finalize.  Runs K1 on the current device.
 * out [rows][d]; row_max / row_sumexp [rows] = the returned state. */
int sp_host_chunk_attention(const double* q, int rows, int d, const double* k, const double* v,
                            const int* chunk_lens, int n_chunks, int causal, int streamed, double* out,
                            double* row_max, double* row_sumexp);

/* ---------------------------------------------------------- step executor
 * One process (rank) per GPU; rank r runs pipeline stage r+1 of
 * gen_slimpipe(p=pp, v=1, m=microbatches, n=slices) (the drop-in planning
 * API) with a Llama-style layer stack (layers/pp layers per stage; the
 * embedding on stage 1, final norm + LM head + cross entropy on stage pp).
 * Weights are bf16 (fp32 master + AdamW), random-initialised N(0, 0.02)
 * from `seed`.  The slot arena holds ledger-peak slots of (stage input +
 * per-layer K/V [+ per-layer attention O/LSE when recompute = 0]) —
 * reference simulator.cpp:311-346. */
typedef struct {
  int32_t layers, hidden, ffn_hidden, heads, kv_heads, head_dim, vocab;
  int32_t microbatches, slices, pp, rank, exchange_mode;
  int64_t seq_len;
  float rope_theta, norm_eps, lr;
  uint64_t seed;
  /* 0 = selective: the forward pass stashes each layer's attention output O
   * and LSE in the slot, the backward pass recomputes everything else (norms,
   * GEMMs, RoPE, SwiGLU) but not K1;  1 = full: only the stage input is
   * stashed and K1 runs again in the backward (reference Full checkpointing,
   * workload.cpp:100-104);  2 = auto: selective when the stash fits in the
   * free HBM left after the rest of the arena, else full
   * (sp_runtime_recompute reports the policy in effect). */
  int32_t recompute;
  /* 1: vocabulary parallelism (pp > 1): the LM head and the cross entropy are
   * split by vocabulary across all stages (reference place_vocab with
   * distribute = true, simulator.cpp:414-522); 0: the last stage owns them. */
  int32_t vocab_parallel;
  /* v, stages per device (interleaved SlimPipe, reference gen_slimpipe with
   * v > 1, schedule.cpp:261-270): device d owns stages d+1, d+1+p, ...;
   * 0 or 1 = one stage per device.  v > 1 needs an even pp >= 2, exchange
   * off and vocab_parallel 0. */
  int32_t interleave;
  /* 1: activation offload (reference offload_ratio, workload.cpp:130-132, at
   * ratio "everything but K/V"): each slot's stage input and — selective
   * recompute — per-layer attention O/LSE go to pinned host memory after the
   * forward pass and come back at its backward; the device arena keeps only
   * the K/V chunks later slices attend to.  0: everything stays in HBM. */
  int32_t offload;
  /* 1: the fp32 dK/dV chunk accumulators are stored in bf16 (sums kept in
   * fp32 inside each backward kernel, rounded once per slice contribution):
   * half their HBM; 0: fp32 storage. */
  int32_t dkv_bf16;
  /* exchange placement (exchange_mode != 0): the executor runs the reference
   * plan's transfers (apply_exchange, simulator.cpp:56-108) except those that
   * move fewer than exchange_min_chunks KV chunks (0 or 1 = keep all) and,
   * with exchange_skip_last = 1, those whose receiver is the last stage —
   * which also runs the LM head and the loss that the plan's attention-only
   * tick loads do not count.  Every rank drops the same transfers. */
  int32_t exchange_min_chunks;
  int32_t exchange_skip_last;
} sp_model_config;

#define SP_STEP_NO_OPTIMIZER 1

#define SP_NCCL_IDS 4
int sp_nccl_unique_id(void* out128);
/* nccl_ids: SP_NCCL_IDS consecutive 128-byte ids, identical on all ranks
 * (stage activations, stage gradients, forward-tick exchange, backward-tick
 * exchange); ignored when pp == 1.  exchange_mode: 0 off, 1 on, 2 early
 * (reference ExchangeMode, simulator.hpp:18) — the per-tick plans of
 * apply_exchange are executed: Q (+ KV chunks, dO and statistics in backward
 * ticks) go to the receiving stage, which returns attention partials. */
int sp_runtime_create(const sp_model_config* cfg, const void* nccl_ids, void** handle);
/* Single-GPU loopback transport (tests, one-GPU boxes): all pp ranks run as
 * host threads of ONE process on the current device; each thread creates
 * its rank's runtime with sp_runtime_create_loopback on a shared world and
 * calls sp_runtime_step concurrently.  Stage links and exchange transfers
 * then move through device-side flags + copy kernels instead of NCCL, with
 * the same send/recv order and group semantics (csrc/host/transport.hpp);
 * the vocabulary collectives run as gathers/broadcasts over it. */
int sp_loopback_create(int ranks, void** world);
int sp_loopback_destroy(void* world);
int sp_loopback_errors(void* world); /* message size mismatches seen so far (0 = none) */
/* transport self-test: 2-rank ping-pong of `iters` x (send/recv + grouped send+recv) */
int sp_loopback_pingpong(void* world, int rank, void* send_buf, void* recv_buf, int64_t bytes, int iters);
/* the same protocol with both ranks enqueued from one host thread */
int sp_loopback_pingpong_1thread(void* world, void* buf0, void* buf1, void* rbuf0, void* rbuf1, int64_t bytes,
                                 int iters);
int sp_runtime_create_loopback(const sp_model_config* cfg, void* world, void** handle);
int sp_runtime_destroy(void* handle);
/* tokens/targets: [microbatches][seq_len] int32 (host, or device when on_device);
 * only stage 1 reads tokens and only the last stage reads targets (< 0 = ignore).
 * *loss (last stage) = mean token cross entropy of the step. */
int sp_runtime_step(void* handle, const int32_t* tokens, const int32_t* targets, int on_device, int flags,
                    float* loss);
int sp_runtime_sync(void* handle);
void* sp_runtime_stream(void* handle);
int sp_runtime_timeline(void* handle, double* out, int cap);
int sp_runtime_attn_stats(void* handle, double* out6);
int sp_runtime_memory(void* handle, int64_t* out7);
int sp_runtime_recompute(void* handle);
/* pinned host bytes holding offloaded activations (0 without offload) */
long long sp_runtime_offload_bytes(void* handle);
/* Diagnostics: position in this rank's pass order of the first pass not yet
 * finished on the compute stream (-1: all done); out4 = kind, microbatch,
 * slice, stage of that pass.  Non-blocking. */
int sp_runtime_progress(void* handle, int32_t* out4);
/* Diagnostics (any thread): index in this rank's pass order of the pass the
 * host is enqueuing inside sp_runtime_step, -1 when it is not in a step. */
int sp_runtime_enqueue_position(void* handle);
int sp_runtime_param(void* handle, int layer, int which, float* host, int64_t count, int dir);
/* {passes with outgoing transfers, passes with incoming transfers, bytes sent
 *  by this rank through the exchange in the last step} */
int sp_runtime_exchange_stats(void* handle, int64_t* out3);
/* Stage sends (activations / gradients) of the last step, timed with CUDA
 * events on their streams: out4 = {messages, bytes, sum of send spans in ms,
 * fastest send in ms}. */
int sp_runtime_comm_stats(void* handle, double* out4);

#ifdef __cplusplus
}
#endif
#endif /* SLIMPIPE_H */
