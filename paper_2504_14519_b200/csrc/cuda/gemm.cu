// Plain library GEMMs of the layer stack (QKV/O/gate-up/down/LM head and
// their input/weight gradients) on cuBLASLt: bf16 operands, fp32 accumulate,
// bf16 or fp32 output, beta for fused residual adds and in-place fp32 weight
// gradient accumulation.  (The attention contractions, which are the hot
// path, are the hand-written tcgen05 kernels in attn_fwd.cu / attn_bwd.cu.)
#include <cublasLt.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <mutex>
#include <tuple>

#include "kernels.hpp"

namespace sp {
namespace {

struct Plan {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, c = nullptr;
  cublasLtMatmulAlgo_t algo{};
  int chosen = 0, candidates = 1;      // index among the heuristic's candidates
  float ms_chosen = 0.f, ms_first = 0.f;  // timed when autotuned (ms per call)
};

using Key = std::tuple<int, bool, bool, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, bool>;

struct State {
  cublasLtHandle_t lt = nullptr;
  // one workspace per (device, stream): GEMMs on different streams (the
  // vocabulary stream, loopback ranks) never share scratch memory
  std::map<std::pair<int, cudaStream_t>, void*> ws;
  size_t ws_bytes = 64ull << 20;
  std::map<Key, Plan> plans;
  std::mutex mu;
  bool tune = false;  // new plans time the heuristic's top candidates and keep the fastest
};

State& state() {
  static State s;
  return s;
}

int lt_status(cublasStatus_t s, const char* what) {
  if (s == CUBLAS_STATUS_SUCCESS) return SP_OK;
  return set_error(SP_ERR_CUDA, "cuBLASLt %s failed (status %d)", what, int(s));
}

}  // namespace

int gemm(bool trans_a, bool trans_b, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const void* B,
         int64_t ldb, void* C, int64_t ldc, bool c_f32, float alpha, float beta, cudaStream_t st, const void* c_in) {
  if (M <= 0 || N <= 0 || K <= 0) return SP_OK;
  State& S = state();
  std::lock_guard<std::mutex> g(S.mu);
  int dev = 0;
  cudaGetDevice(&dev);
  if (!S.lt)
    if (int rc = lt_status(cublasLtCreate(&S.lt), "create")) return rc;
  void*& ws = S.ws[{dev, st}];
  if (!ws)
    if (int rc = cuda_status(cudaMalloc(&ws, S.ws_bytes), "gemm workspace")) return rc;
  const Key key{dev, trans_a, trans_b, M, N, K, lda, ldb, ldc, c_f32};
  auto it = S.plans.find(key);
  if (it == S.plans.end()) {
    Plan p;
    // Column-major view: C^T[N,M] = op(B)^T[N,K] * op(A)^T[K,M].
    if (int rc = lt_status(cublasLtMatmulDescCreate(&p.op, CUBLAS_COMPUTE_32F, CUDA_R_32F), "desc")) return rc;
    const cublasOperation_t ta = trans_b ? CUBLAS_OP_T : CUBLAS_OP_N;
    const cublasOperation_t tb = trans_a ? CUBLAS_OP_T : CUBLAS_OP_N;
    cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof ta);
    cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof tb);
    cublasLtMatrixLayoutCreate(&p.a, CUDA_R_16BF, trans_b ? K : N, trans_b ? N : K, ldb);
    cublasLtMatrixLayoutCreate(&p.b, CUDA_R_16BF, trans_a ? M : K, trans_a ? K : M, lda);
    cublasLtMatrixLayoutCreate(&p.c, c_f32 ? CUDA_R_32F : CUDA_R_16BF, N, M, ldc);
    cublasLtMatmulPreference_t pref;
    cublasLtMatmulPreferenceCreate(&pref);
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &S.ws_bytes,
                                         sizeof S.ws_bytes);
    constexpr int kCand = 6;
    cublasLtMatmulHeuristicResult_t res[kCand]{};
    int found = 0;
    cublasStatus_t hs =
        cublasLtMatmulAlgoGetHeuristic(S.lt, p.op, p.a, p.b, p.c, p.c, pref, S.tune ? kCand : 1, res, &found);
    cublasLtMatmulPreferenceDestroy(pref);
    if (hs != CUBLAS_STATUS_SUCCESS || found == 0)
      return set_error(SP_ERR_CUDA, "cuBLASLt: no algorithm for %lldx%lldx%lld", (long long)M, (long long)N,
                       (long long)K);
    p.algo = res[0].algo;
    p.candidates = found;
    if (S.tune && found > 1) {
      // autotune (runtime warm-up, before any communication): time every
      // candidate on the call's own operands and keep the fastest
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      float best = 0.f;
      for (int x = 0; x < found; ++x) {
        auto run = [&]() {
          return cublasLtMatmul(S.lt, p.op, &alpha, B, p.a, A, p.b, &beta, c_in ? c_in : C, p.c, C, p.c, &res[x].algo,
                                ws, S.ws_bytes, st);
        };
        if (run() != CUBLAS_STATUS_SUCCESS) continue;
        cudaEventRecord(e0, st);
        for (int r = 0; r < 3; ++r) run();
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 3.f;
        if (x == 0) p.ms_first = ms;
        if (x == 0 || ms < best) {
          best = ms;
          p.algo = res[x].algo;
          p.chosen = x;
        }
      }
      p.ms_chosen = best;
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      if (int rc = cuda_status(cudaGetLastError(), "gemm autotune")) return rc;
    }
    it = S.plans.emplace(key, p).first;
  }
  const Plan& p = it->second;
  count_library_launch();
  // D = alpha op(A) op(B) + beta C_in: the residual input is read in place
  // (no separate copy into the output first)
  return lt_status(cublasLtMatmul(S.lt, p.op, &alpha, B, p.a, A, p.b, &beta, c_in ? c_in : C, p.c, C, p.c, &p.algo, ws,
                                  S.ws_bytes, st),
                   "matmul");
}

void gemm_autotune(bool on) {
  std::lock_guard<std::mutex> g(state().mu);
  state().tune = on;
}

std::string gemm_plans_json() {
  State& S = state();
  std::lock_guard<std::mutex> g(S.mu);
  std::string out = "[";
  for (const auto& [k, p] : S.plans) {
    char buf[256];
    std::snprintf(buf, sizeof buf,
                  "%s{\"M\": %lld, \"N\": %lld, \"K\": %lld, \"trans_a\": %d, \"trans_b\": %d, \"c_f32\": %d, "
                  "\"candidates\": %d, \"chosen\": %d, \"ms_first\": %.4f, \"ms_chosen\": %.4f}",
                  out.size() > 1 ? ", " : "", (long long)std::get<3>(k), (long long)std::get<4>(k),
                  (long long)std::get<5>(k), int(std::get<1>(k)), int(std::get<2>(k)), int(std::get<9>(k)),
                  p.candidates, p.chosen, p.ms_first, p.ms_chosen);
    out += buf;
  }
  return out + "]";
}

}  // namespace sp

extern "C" int sp_gemm_plans_json(char** out) {
  const std::string s = sp::gemm_plans_json();
  *out = static_cast<char*>(std::malloc(s.size() + 1));
  if (!*out) return SP_ERR_RUNTIME;
  std::memcpy(*out, s.c_str(), s.size() + 1);
  return SP_OK;
}
