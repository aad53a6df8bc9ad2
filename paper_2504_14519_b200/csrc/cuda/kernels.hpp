// Internal (C++) launch interface of the device ops used by the step
// executor.  All return SP_* status codes; all run on the given stream.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "slimpipe.h"

namespace sp {

int set_error(int code, const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);
void count_launch(int n = 1);          // kernels of this library
void count_library_launch(int n = 1);  // cuBLASLt calls

// layers.cu
int embed_fwd(const int32_t* tok, const void* table, void* out, int64_t rows, int dim, cudaStream_t st);
int embed_bwd(const int32_t* tok, const void* dy, float* dtable, int64_t rows, int dim, cudaStream_t st);
int rmsnorm_fwd(const void* x, const void* w, void* y, float* rstd, int64_t rows, int dim, float eps, cudaStream_t st);
// dw (may be null) += the weight gradient: with dw_ws (rmsnorm_dw_ws_floats
// floats) in a fixed block order (bitwise reproducible), else by atomics
int rmsnorm_bwd(const void* dy, const void* x, const void* w, const float* rstd, const void* dx_in, void* dx_out,
                float* dw, int64_t rows, int dim, cudaStream_t st, float* dw_ws = nullptr);
int64_t rmsnorm_dw_ws_floats(int64_t rows, int dim);
int rope_table(float* cs, float* sn, int64_t positions, int d, double theta, cudaStream_t st);
int rope_qkv_fwd(const void* qkv, int64_t rows, int heads, int kv_heads, int d, int64_t pos0, const float* cs,
                 const float* sn, void* q_out, int64_t q_stride, void* k_out, void* v_out, int64_t kv_stride,
                 cudaStream_t st);
// dk/dv: fp32, or bf16 when acc_bf16 (the dK/dV chunk accumulators' storage)
int rope_qkv_bwd(const float* dq, void* dk, void* dv, int64_t kv_stride, int64_t rows, int heads, int kv_heads,
                 int d, int64_t pos0, const float* cs, const float* sn, void* dqkv, int zero_kv, cudaStream_t st,
                 bool acc_bf16 = false);
int add_to_bf16(void* dst, const float* src, int64_t n, cudaStream_t st);  // bf16 dst += fp32 src
int swiglu_fwd(const void* gu, void* act, int64_t rows, int H, cudaStream_t st);
int swiglu_bwd(const void* dact, const void* gu, void* dgu, int64_t rows, int H, cudaStream_t st);
int cross_entropy(const float* logits, const int32_t* tgt, int64_t rows, int V, float scale, void* dlogits,
                  float* loss_sum, cudaStream_t st);
int adamw(float* master, void* wbf, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
          float eps, float wd, int step, cudaStream_t st);
int init_params(float* master, void* wbf, int64_t n, uint64_t seed, float stdv, float constant, int use_const,
                cudaStream_t st);
int f32_to_bf16(const float* a, void* b, int64_t n, cudaStream_t st);
// vocabulary-parallel cross entropy over a vocab shard [v0, v0+Vs)
int xent_shard_stats(const float* logits, const int32_t* tgt, int64_t rows, int Vs, int v0, float* m_loc,
                     float* m_glob, float* zt, cudaStream_t st);
int xent_shard_rescale(const float* m_loc, const float* m_glob, float* z, int64_t rows, cudaStream_t st);
int xent_shard_grad(const float* logits, const int32_t* tgt, int64_t rows, int Vs, int v0, const float* m_glob,
                    const float* zt, float scale, void* dlogits, float* loss_sum, cudaStream_t st);
int add_f32(float* dst, const float* src, int64_t n, cudaStream_t st);  // dst += src

// K1 masking / output options (sp_attn_fwd: causal_off = total - q_rows,
// kv_valid = total, scale = 1/sqrt(d), no row_max).
struct FwdMask {
  int causal = 1;
  int64_t causal_off = 0;  // causal: query row r sees keys <= r + causal_off
  int64_t kv_valid = 0;    // keys >= kv_valid (padding) are masked
  double scale = 0.0;      // softmax scale
  float* row_max = nullptr;  // optional fp32 [heads][q_rows]: true row max of the scaled scores
};

// attn_fwd_v4.cu — d=128 forward (two 128-row tiles per CTA, shared S buffer)
int attn_fwd_d128_ps(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                     int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks, int chunk_len,
                     int heads, int kv_heads, const FwdMask& mk, void* o, int64_t o_stride, float* lse,
                     cudaStream_t st);

// load every kernel of the library on the current device now (not lazily at
// first launch, which can deadlock against a spinning receive; transport.cu)
int preload_kernels();
int preload_layers();
int preload_attn_fwd();
int preload_attn_fwd_v4();
int preload_attn_bwd();
int preload_attn_bwd_v2();
int preload_attn_merge();

// cudaFuncAttributeMaxDynamicSharedMemorySize once per (kernel, device)
int set_smem_once(const void* fn, size_t smem, const char* what);

// attn_bwd_v2.cu — pipelined d=128 backward (lse2/delta prepared by the caller)
int attn_bwd_d128(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                  int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks, int chunk_len,
                  int heads, int kv_heads, int causal, const void* dout, int64_t do_stride, const float* lse2,
                  const float* delta, float* dq_acc, void* dk_acc, void* dv_acc, int64_t acc_rows,
                  const int32_t* acc_row, bool acc_bf16, cudaStream_t st);
// sp_attn_bwd_core with fp32 (acc_bf16 = false) or bf16 dK/dV chunk accumulators
int attn_bwd_core(const void* q, int64_t q_rows, int64_t q_stride, const void* k_pool, const void* v_pool,
                  int64_t pool_rows, int64_t kv_stride, const int32_t* chunk_row, int n_chunks, int chunk_len,
                  int heads, int kv_heads, int head_dim, int causal, const void* dout, int64_t do_stride,
                  const float* stats, float* dq_acc, void* dk_acc, void* dv_acc, int64_t acc_rows,
                  const int32_t* acc_row, bool acc_bf16, cudaStream_t stream);

// gemm.cu — row-major GEMMs on cuBLASLt (bf16 inputs, fp32 accumulate).
//   C[M,N] = alpha * op(A) op(B) + beta * C
//   A is [M,K] (or [K,M] when trans_a), B is [K,N] (or [N,K] when trans_b),
//   lda/ldb/ldc are row pitches in elements.  c_f32 selects an fp32 C/D.
//   c_in (optional): read the beta term from c_in instead of C (same layout).
int gemm(bool trans_a, bool trans_b, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const void* B,
         int64_t ldb, void* C, int64_t ldc, bool c_f32, float alpha, float beta, cudaStream_t st,
         const void* c_in = nullptr);
// while on, a GEMM shape seen for the first time times cuBLASLt's top
// candidates on its own operands and keeps the fastest (runtime warm-up only)
void gemm_autotune(bool on);

}  // namespace sp
