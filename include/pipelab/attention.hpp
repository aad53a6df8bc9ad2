#pragma once

// Drop-in for the reference's chunked-attention API
// (proj/include/pipelab/attention.hpp:14-61), realised on the
// B200: chunk_attention / accumulate_chunk run K1 (sm_100a tcgen05, bf16
// operands, fp32 softmax statistics) on the current CUDA device; the fp64
// types and signatures are the reference's.  Differences, by design:
//   * operands are rounded to bf16 on the way in (results agree with the fp64
//     reference within the bf16 tolerance of the parity tests);
//   * a state's row_max holds the row's log-sum-exp and row_sumexp 1 (any
//     stabiliser is valid for the merge/finalize algebra; fully masked rows
//     keep the reference's -inf / 0);
//   * shapes the kernels do not tile throw std::invalid_argument: head_dim in
//     {64, 128}, query rows and every chunk length multiples of 128, and for
//     accumulate_chunk a chunk that is either fully visible or the diagonal
//     chunk of a slice (rows == chunk length, chunk ends at total_kv) — the
//     two cases of the sliced schedule.  There is no CPU fallback.
// merge_partials / finalize are O(rows·d) host glue with the reference's
// formulas (attention.cpp:63-92).

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
