// pipelab attention API (include/pipelab/attention.hpp) on the B200: the
// reference's fp64 host types in, K1 (sp_attn_fwd, one head) on the current
// CUDA device, fp64 states out.  Reference semantics: attention.cpp:13-111.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>

#include "errors.hpp"
#include "pipelab/attention.hpp"
#include "slimpipe.h"

namespace pipelab {

namespace {

constexpr double kNegInf = -std::numeric_limits<double>::infinity();

uint16_t to_bf16(double x) {  // round to nearest even (via fp32)
  const float f = static_cast<float>(x);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return uint16_t(u >> 16);
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

double from_bf16(uint16_t b) {
  const uint32_t u = uint32_t(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("chunked attention (B200): ") + what + ": " +
                                                 cudaGetErrorString(e));
}

struct DevBuf {  // RAII device allocation
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { cuda_check(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc"); }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// One K1 launch (sp_attn_fwd_masked) for a single head: query [rows][d] over
// `chunks` (keys concatenated in order, key/value widths d / dv <= 128).
// Rows, keys and both widths are zero-padded to the kernel tiles (128 rows /
// keys, 64 or 128 columns); the padded keys are masked (kv_valid), the
// softmax scale is the reference's 1/sqrt(d) (attention.cpp:31) and, when
// `causal`, row r sees concatenated keys <= r + causal_off.  Returns the
// reference state (attention.cpp:13-19 semantics): unnormalised partial
// output, the true row max of the scaled scores, and the row sum of
// exponentials relative to it; rows that see no key stay empty (-inf, 0).
AttnChunkState run_k1(const Mat& q, const std::vector<const KvChunk*>& chunks, bool causal, int64_t causal_off) {
  const int rows = q.rows, d = q.cols;
  const int dv = chunks.empty() ? d : chunks.front()->values.cols;
  int64_t total = 0;
  for (const KvChunk* c : chunks) total += c->keys.rows;
  AttnChunkState st = empty_state(rows, dv);
  if (total == 0 || rows == 0) return st;
  if (d > 128 || dv > 128)
    throw std::invalid_argument("chunked attention (B200): head_dim above 128 is not implemented by K1");
  const int dp = (d <= 64 && dv <= 64) ? 64 : 128;
  const int64_t rows_p = (rows + 127) / 128 * 128, total_p = (total + 127) / 128 * 128;
  if (total_p > (int64_t(1) << 30)) throw std::invalid_argument("chunked attention (B200): too many keys");
  std::vector<uint16_t> hq(size_t(rows_p) * dp, 0), hk(size_t(total_p) * dp, 0), hv(size_t(total_p) * dp, 0);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < d; ++c) hq[size_t(r) * dp + c] = to_bf16(q.at(r, c));
  int64_t pos = 0;
  for (const KvChunk* ch : chunks) {
    for (int r = 0; r < ch->keys.rows; ++r) {
      for (int c = 0; c < d; ++c) hk[size_t(pos + r) * dp + c] = to_bf16(ch->keys.at(r, c));
      for (int c = 0; c < dv; ++c) hv[size_t(pos + r) * dp + c] = to_bf16(ch->values.at(r, c));
    }
    pos += ch->keys.rows;
  }
  DevBuf dq(hq.size() * 2), dk(hk.size() * 2), dvb(hv.size() * 2), dout(hq.size() * 2), dlse(size_t(rows_p) * 4),
      dmax(size_t(rows_p) * 4);
  cuda_check(cudaMemcpy(dq.p, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice), "copy q");
  cuda_check(cudaMemcpy(dk.p, hk.data(), hk.size() * 2, cudaMemcpyHostToDevice), "copy k");
  cuda_check(cudaMemcpy(dvb.p, hv.data(), hv.size() * 2, cudaMemcpyHostToDevice), "copy v");
  const int32_t chunk_row = 0;
  const int rc = sp_attn_fwd_masked(dq.p, rows_p, dp, dk.p, dvb.p, total_p, dp, &chunk_row, 1, int(total_p), 1, 1, dp,
                                    causal ? 1 : 0, causal_off, total, 1.0 / std::sqrt(double(d)), dout.p, dp,
                                    static_cast<float*>(dlse.p), static_cast<float*>(dmax.p), nullptr);
  if (rc != SP_OK) {
    if (rc == SP_ERR_INVALID) throw std::invalid_argument(sp_last_error());
    throw std::runtime_error(sp_last_error());
  }
  std::vector<uint16_t> ho(hq.size());
  std::vector<float> hl(static_cast<size_t>(rows_p)), hm(static_cast<size_t>(rows_p));
  cuda_check(cudaMemcpy(ho.data(), dout.p, ho.size() * 2, cudaMemcpyDeviceToHost), "copy o");
  cuda_check(cudaMemcpy(hl.data(), dlse.p, hl.size() * 4, cudaMemcpyDeviceToHost), "copy lse");
  cuda_check(cudaMemcpy(hm.data(), dmax.p, hm.size() * 4, cudaMemcpyDeviceToHost), "copy row max");
  for (int r = 0; r < rows; ++r) {
    const double lse = hl[size_t(r)], m = hm[size_t(r)];
    if (std::isinf(lse) || std::isinf(m)) continue;  // the row sees no key: stays empty
    const double l = std::exp(lse - m);              // sum of exp(s - m), >= 1
    st.row_max[size_t(r)] = m;
    st.row_sumexp[size_t(r)] = l;
    for (int c = 0; c < dv; ++c) st.partial_output.at(r, c) = from_bf16(ho[size_t(r) * dp + c]) * l;
  }
  return st;
}

}  // namespace

// attention.cpp:13-19
AttnChunkState empty_state(int rows, int head_dim) {
  AttnChunkState st;
  st.partial_output = Mat(rows, head_dim);
  st.row_max.assign(size_t(rows), kNegInf);
  st.row_sumexp.assign(size_t(rows), 0.0);
  return st;
}

// attention.cpp:21-61: one chunk at global key position chunk_pos folded into
// the state; row r sees global keys <= total_kv - rows + r when causal.
void accumulate_chunk(AttnChunkState& st, const Mat& query, const KvChunk& chunk, std::int64_t chunk_pos,
                      std::int64_t total_kv, bool causal) {
  const Mat& k = chunk.keys;
  const Mat& v = chunk.values;
  if (k.cols != query.cols || v.rows != k.rows) throw std::invalid_argument("accumulate_chunk: dimension mismatch");
  if (st.partial_output.rows != query.rows || st.partial_output.cols != v.cols)
    throw std::invalid_argument("accumulate_chunk: state shape mismatch");
  st = merge_partials(st, run_k1(query, {&chunk}, causal, total_kv - query.rows - chunk_pos));
}

// attention.cpp:63-82
AttnChunkState merge_partials(const AttnChunkState& a, const AttnChunkState& b) {
  if (a.empty()) return b;
  if (b.empty()) return a;
  if (a.partial_output.rows != b.partial_output.rows || a.partial_output.cols != b.partial_output.cols)
    throw std::invalid_argument("merge_partials: shape mismatch");
  const int rows = a.partial_output.rows, d = a.partial_output.cols;
  AttnChunkState out = empty_state(rows, d);
  for (int r = 0; r < rows; ++r) {
    const double ma = a.row_max[size_t(r)], mb = b.row_max[size_t(r)];
    const double m = ma > mb ? ma : mb;
    if (m == kNegInf) continue;  // both empty
    const double wa = ma == kNegInf ? 0.0 : std::exp(ma - m);
    const double wb = mb == kNegInf ? 0.0 : std::exp(mb - m);
    out.row_max[size_t(r)] = m;
    out.row_sumexp[size_t(r)] = a.row_sumexp[size_t(r)] * wa + b.row_sumexp[size_t(r)] * wb;
    for (int c = 0; c < d; ++c)
      out.partial_output.at(r, c) = a.partial_output.at(r, c) * wa + b.partial_output.at(r, c) * wb;
  }
  return out;
}

// attention.cpp:84-92
Mat finalize(const AttnChunkState& st) {
  const int rows = st.partial_output.rows, d = st.partial_output.cols;
  Mat o(rows, d);
  for (int r = 0; r < rows; ++r) {
    const double l = st.row_sumexp[size_t(r)];
    if (!(l > 0.0)) continue;
    for (int c = 0; c < d; ++c) o.at(r, c) = st.partial_output.at(r, c) / l;
  }
  return o;
}

// attention.cpp:94-111 — one K1 launch over the whole ordered chunk list
std::pair<Mat, AttnChunkState> chunk_attention(const Mat& query, const std::vector<KvChunk>& chunks, bool causal) {
  std::int64_t total_kv = 0;
  std::vector<const KvChunk*> ptrs;
  for (const KvChunk& c : chunks) {
    if (c.keys.rows != c.values.rows) throw std::invalid_argument("chunk_attention: key/value row mismatch");
    if (c.keys.cols != query.cols || c.values.cols != chunks.front().values.cols)
      throw std::invalid_argument("accumulate_chunk: dimension mismatch");
    total_kv += c.keys.rows;
    ptrs.push_back(&c);
  }
  AttnChunkState st = run_k1(query, ptrs, causal, total_kv - query.rows);
  Mat o = finalize(st);
  return {std::move(o), std::move(st)};
}

}  // namespace pipelab

// C shims for the Python parity tests (one head, fp64, row-major).
extern "C" int sp_host_chunk_attention(const double* q, int rows, int d, const double* k, const double* v,
                                       const int* chunk_lens, int n_chunks, int causal, int streamed, double* out,
                                       double* row_max, double* row_sumexp) {
  try {
    pipelab::Mat qm(rows, d);
    std::memcpy(qm.a.data(), q, sizeof(double) * size_t(rows) * d);
    std::vector<pipelab::KvChunk> chunks(static_cast<size_t>(n_chunks));
    int64_t pos = 0;
    for (int c = 0; c < n_chunks; ++c) {
      chunks[size_t(c)].keys = pipelab::Mat(chunk_lens[c], d);
      chunks[size_t(c)].values = pipelab::Mat(chunk_lens[c], d);
      std::memcpy(chunks[size_t(c)].keys.a.data(), k + pos * d, sizeof(double) * size_t(chunk_lens[c]) * d);
      std::memcpy(chunks[size_t(c)].values.a.data(), v + pos * d, sizeof(double) * size_t(chunk_lens[c]) * d);
      pos += chunk_lens[c];
    }
    pipelab::AttnChunkState st = pipelab::empty_state(rows, d);
    pipelab::Mat o;
    if (streamed) {  // accumulate_chunk per chunk, then finalize (attention.cpp:94-111 loop)
      int64_t cp = 0;
      for (int c = 0; c < n_chunks; ++c) {
        pipelab::accumulate_chunk(st, qm, chunks[size_t(c)], cp, pos, causal != 0);
        cp += chunk_lens[c];
      }
      o = pipelab::finalize(st);
    } else {
      auto r = pipelab::chunk_attention(qm, chunks, causal != 0);
      o = std::move(r.first);
      st = std::move(r.second);
    }
    std::memcpy(out, o.a.data(), sizeof(double) * size_t(rows) * d);
    std::memcpy(row_max, st.row_max.data(), sizeof(double) * size_t(rows));
    std::memcpy(row_sumexp, st.row_sumexp.data(), sizeof(double) * size_t(rows));
    return SP_OK;
  } catch (const std::invalid_argument& e) {
    sp::last_error() = e.what();
    return SP_ERR_INVALID;
  } catch (const std::exception& e) {
    sp::last_error() = e.what();
    return SP_ERR_RUNTIME;
  }
}
