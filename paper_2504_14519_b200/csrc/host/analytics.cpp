// Closed-form memory / bubble models (drop-in for the reference's
// proj/src/analytics.cpp:11-105; formulas from the SlimPipe paper, Table 1
// and Eq. 1).  Pure functions on exact rationals.
#include "pipelab/analytics.hpp"

#include <stdexcept>

namespace pipelab {

namespace {
bool sliced(Scheme s) { return s == Scheme::SlimPipe || s == Scheme::TeraPipe; }
}  // namespace

// analytics.cpp:11-31
Rat memory_multiplier(Scheme scheme, std::int64_t p, std::int64_t m, std::int64_t n, std::int64_t v) {
  if (scheme == Scheme::SlimPipe) return Rat(1, p) + Rat(2 * (p - 1), n * v * p);  // M_a/p + 2(p-1) slices in flight
  if (scheme == Scheme::GPipe || scheme == Scheme::TeraPipe) return Rat(m, p);     // all m microbatches stashed
  if (scheme == Scheme::OneFOneB || scheme == Scheme::ZBV) return Rat(1);
  if (scheme == Scheme::Interleaved1F1B) return v == 1 ? Rat(1) : Rat(1) + Rat(p - 1, v * p);
  if (scheme == Scheme::VHalf) return Rat(1, 2) + Rat(1, p);
  throw std::invalid_argument("memory_multiplier: unknown scheme");
}

// analytics.cpp:33-36
Rat slim_acc_memory(std::int64_t p, std::int64_t n, const Rat& microbatch_bytes) {
  if (n < p) throw std::invalid_argument("slim_acc_memory: requires n >= p");
  const Rat slices_in_flight = Rat(1) + Rat(2 * (p - 1), n);
  return slices_in_flight * microbatch_bytes / Rat(p);
}

// analytics.cpp:38-67
BubbleBound bubble_bounds(Scheme scheme, std::int64_t p, std::int64_t m, std::int64_t n, std::int64_t v) {
  BubbleBound b;
  if (scheme == Scheme::ZBV) {
    b.interval = std::make_pair(Rat(0), Rat(2 * (p - 1), 3 * m));
  } else if (scheme == Scheme::VHalf) {
    b.interval = std::make_pair(Rat(p, 2 * m), Rat(1, 3) + Rat(p, 2 * m));
  } else {
    // (p-1) / (m * virtual stages * slices): exact for unsliced schemes, an
    // upper bound for the sliced ones (attention-heavy slices only shrink it)
    const std::int64_t virt = scheme == Scheme::Interleaved1F1B || scheme == Scheme::SlimPipe ? v : 1;
    const std::int64_t sl = sliced(scheme) ? n : 1;
    b.exact = Rat(p - 1, sl * virt * m);
    b.upper_bound_only = sliced(scheme);
  }
  return b;
}

// analytics.cpp:69-72
Rat slim_attention_bubble(std::int64_t p, std::int64_t m, std::int64_t n, std::int64_t v) {
  return Rat((p - 1) * p, (n + 1) * n * v * m);
}

// analytics.cpp:74-89
bool scheme_accepts(Scheme scheme, std::int64_t p, std::int64_t m, std::int64_t n, std::int64_t v) {
  if (p < 1 || m < 1 || n < 1 || v < 1) return false;
  switch (scheme) {
    case Scheme::SlimPipe: return n % p == 0;
    case Scheme::TeraPipe: return v == 1;
    case Scheme::GPipe: return v == 1 && n == 1;
    case Scheme::OneFOneB: return v == 1 && n == 1 && m >= p;
    case Scheme::Interleaved1F1B: return n == 1 && (v == 1 ? m >= p : m % p == 0);
    case Scheme::ZBV:
    case Scheme::VHalf: return v == 2 && n == 1 && m >= p;
  }
  return false;
}

// analytics.cpp:91-112
bool memory_form_valid(Scheme scheme, std::int64_t p, std::int64_t m, std::int64_t n, std::int64_t v) {
  if (!scheme_accepts(scheme, p, m, n, v)) return false;
  switch (scheme) {
    case Scheme::SlimPipe: return m * n * v >= n * v + 2 * (p - 1);  // warm-up of n*v + 2(p-1) slices fits
    case Scheme::Interleaved1F1B: return v == 1 || m * v >= p * v + p - 1;
    case Scheme::ZBV: return m >= 2 * p - 1;
    case Scheme::VHalf: return m >= p + 1;
    default: return true;
  }
}

}  // namespace pipelab
