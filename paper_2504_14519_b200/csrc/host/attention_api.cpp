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

void check_head_dim(int d) {
  if (d != 64 && d != 128) throw std::invalid_argument("chunked attention (B200): head_dim must be 64 or 128");
}

// One K1 launch: query [rows][d] over `chunks` (keys concatenated in order),
// bottom-right causal over their total when `causal`.  Returns the state
// (O normalised, row_max = LSE, row_sumexp = 1; fully masked rows empty).
AttnChunkState run_k1(const Mat& q, const std::vector<const KvChunk*>& chunks, bool causal) {
  const int rows = q.rows, d = q.cols;
  check_head_dim(d);
  if (rows % 128) throw std::invalid_argument("chunked attention (B200): query rows must be a multiple of 128");
  int64_t total = 0;
  bool equal = true;
  for (const KvChunk* c : chunks) {
    if (c->keys.rows != c->values.rows) throw std::invalid_argument("chunk_attention: key/value row mismatch");
    if (c->keys.cols != d || c->values.cols != d) throw std::invalid_argument("chunk_attention: head_dim mismatch");
    if (c->keys.rows % 128) throw std::invalid_argument("chunked attention (B200): chunk length must be a multiple of 128");
    equal = equal && c->keys.rows == chunks.front()->keys.rows;
    total += c->keys.rows;
  }
  AttnChunkState st = empty_state(rows, d);
  if (total == 0 || rows == 0) return st;
  if (causal && total < rows) throw std::invalid_argument("chunked attention (B200): causal needs total_kv >= rows");
  // chunk table: the given chunks when equal-length, else 128-row pieces
  const int chunk_len = equal ? chunks.front()->keys.rows : 128;
  const int64_t n_tab = total / chunk_len;
  if (n_tab > SP_MAX_CHUNKS) throw std::invalid_argument("chunked attention (B200): too many chunks");
  std::vector<int32_t> chunk_row(static_cast<size_t>(n_tab));
  for (int64_t c = 0; c < n_tab; ++c) chunk_row[size_t(c)] = int32_t(c * chunk_len);

  std::vector<uint16_t> hq(size_t(rows) * d), hk(size_t(total) * d), hv(size_t(total) * d);
  for (size_t x = 0; x < hq.size(); ++x) hq[x] = to_bf16(q.a[x]);
  size_t off = 0;
  for (const KvChunk* c : chunks) {
    for (size_t x = 0; x < c->keys.a.size(); ++x) {
      hk[off + x] = to_bf16(c->keys.a[x]);
      hv[off + x] = to_bf16(c->values.a[x]);
    }
    off += c->keys.a.size();
  }
  DevBuf dq(hq.size() * 2), dk(hk.size() * 2), dv(hv.size() * 2), dout(hq.size() * 2), dlse(size_t(rows) * 4);
  cuda_check(cudaMemcpy(dq.p, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice), "copy q");
  cuda_check(cudaMemcpy(dk.p, hk.data(), hk.size() * 2, cudaMemcpyHostToDevice), "copy k");
  cuda_check(cudaMemcpy(dv.p, hv.data(), hv.size() * 2, cudaMemcpyHostToDevice), "copy v");
  const int rc = sp_attn_fwd(dq.p, rows, d, dk.p, dv.p, total, d, chunk_row.data(), int(n_tab), chunk_len, 1, 1, d,
                             causal ? 1 : 0, dout.p, d, static_cast<float*>(dlse.p), nullptr);
  if (rc != SP_OK) {
    if (rc == SP_ERR_INVALID) throw std::invalid_argument(sp_last_error());
    throw std::runtime_error(sp_last_error());
  }
  std::vector<uint16_t> ho(hq.size());
  std::vector<float> hl(static_cast<size_t>(rows));
  cuda_check(cudaMemcpy(ho.data(), dout.p, ho.size() * 2, cudaMemcpyDeviceToHost), "copy o");
  cuda_check(cudaMemcpy(hl.data(), dlse.p, hl.size() * 4, cudaMemcpyDeviceToHost), "copy lse");
  for (int r = 0; r < rows; ++r) {
    if (std::isinf(hl[size_t(r)]) && hl[size_t(r)] < 0) continue;  // fully masked: stays empty
    st.row_max[size_t(r)] = hl[size_t(r)];
    st.row_sumexp[size_t(r)] = 1.0;
    for (int c = 0; c < d; ++c) st.partial_output.at(r, c) = from_bf16(ho[size_t(r) * d + c]);
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

// attention.cpp:21-61 — the two visibility cases of the sliced schedule
void accumulate_chunk(AttnChunkState& st, const Mat& query, const KvChunk& chunk, std::int64_t chunk_pos,
                      std::int64_t total_kv, bool causal) {
  const int rows = query.rows, len = chunk.keys.rows;
  if (st.empty()) st = empty_state(rows, query.cols);
  if (st.partial_output.rows != rows || st.partial_output.cols != query.cols)
    throw std::invalid_argument("accumulate_chunk: state shape mismatch");
  const int64_t first_visible_limit = total_kv - rows;  // row 0 sees keys <= this
  bool masked = false;
  if (causal && chunk_pos + len - 1 > first_visible_limit) {
    if (chunk_pos > total_kv - 1) return;  // no row sees any key of this chunk
    if (!(len == rows && chunk_pos + len == total_kv))
      throw std::invalid_argument(
          "accumulate_chunk (B200): a partially visible chunk must be the slice's diagonal chunk");
    masked = true;
  }
  st = merge_partials(st, run_k1(query, {&chunk}, masked));
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
  std::vector<const KvChunk*> ptrs;
  for (const KvChunk& c : chunks) ptrs.push_back(&c);
  AttnChunkState st = run_k1(query, ptrs, causal);
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
    pipelab::AttnChunkState st;
    pipelab::Mat o;
    if (streamed) {  // accumulate_chunk per chunk, then finalize (attention.cpp:94-111 loop)
      int64_t cp = 0;
      for (int c = 0; c < n_chunks; ++c) {
        pipelab::accumulate_chunk(st, qm, chunks[size_t(c)], cp, pos, causal != 0);
        cp += chunk_lens[c];
      }
      if (st.empty()) st = pipelab::empty_state(rows, d);
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
