#pragma once

// Drop-in for the reference's chunked-attention API
// (proj/include/pipelab/attention.hpp:14-61), realised on the
// B200: chunk_attention / accumulate_chunk run K1 (sm_100a tcgen05, bf16
// operands, fp32 softmax statistics) on the current CUDA device; the fp64
// types, signatures, state semantics and exceptions are the reference's:
//   * any query rows, chunk lengths, chunk positions and head widths up to
//     128 (the host pads to the kernel tiles and masks the padding; the scale
//     is 1/sqrt(d) of the real width);
//   * the state is the reference's: unnormalised partial output, the true
//     row max of the scaled scores, and the row sum of exponentials relative
//     to it (the kernel reports its row max next to the log-sum-exp);
//   * operands are rounded to bf16 on the way in, so results agree with the
//     fp64 reference within the bf16 tolerance (rel 2e-2), not to 1e-12.
// merge_partials / finalize are O(rows·d) host arithmetic on the returned
// host states with the reference's formulas (attention.cpp:63-92).
// There is no CPU fallback: without a CUDA device every call throws.

#include <cstdint>
#include <utility>
#include <vector>

namespace pipelab {

struct Mat {
  int rows = 0;
  int cols = 0;
  std::vector<double> a;

  Mat() = default;
  Mat(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
  double& at(int r, int c) { return a[static_cast<size_t>(r) * cols + c]; }
  double at(int r, int c) const { return a[static_cast<size_t>(r) * cols + c]; }
};

struct KvChunk {
  Mat keys;    // chunk_len x head_dim
  Mat values;  // chunk_len x head_dim
};

struct AttnChunkState {
  Mat partial_output;              // exp-weighted (unnormalised) value accumulation
  std::vector<double> row_max;     // stabiliser; -inf until a row sees an unmasked key
  std::vector<double> row_sumexp;  // 0 until a row sees an unmasked key

  bool empty() const { return row_max.empty(); }
};

AttnChunkState empty_state(int rows, int head_dim);

void accumulate_chunk(AttnChunkState& st, const Mat& query, const KvChunk& chunk, std::int64_t chunk_pos,
                      std::int64_t total_kv, bool causal);

AttnChunkState merge_partials(const AttnChunkState& a, const AttnChunkState& b);

Mat finalize(const AttnChunkState& st);

std::pair<Mat, AttnChunkState> chunk_attention(const Mat& query, const std::vector<KvChunk>& chunks, bool causal);

}  // namespace pipelab
