// Closed-form memory / bubble models (drop-in for the reference's
// proj/src/analytics.cpp:11-105; formulas from the SlimPipe paper, Table 1
// and Eq. 1).  Pure functions on exact rationals.
#include "pipelab/analytics.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <sstream>
#include <stdexcept>

#include "pipelab/simulator.hpp"
#include "pipelab/workload.hpp"

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

// ---- closed forms vs simulate() over a grid (reference analytics.cpp:110-193)

namespace {

// simulate() under linear unit costs and the unit memory model: the peak of
// activation units over devices, in M_a, and the bubble fraction
std::pair<Rat, double> simulated_point(Scheme scheme, std::int64_t p, std::int64_t v, std::int64_t m,
                                       std::int64_t n) {
  GenConfig gc;
  gc.p = std::int32_t(p), gc.v = std::int32_t(v), gc.m = std::int32_t(m), gc.n = std::int32_t(n);
  gc.cost.alpha_linear = 1.0;
  gc.cost.beta_attn = 0.0;
  gc.seq_len = n;
  SimInputs in;
  in.cost = gc.cost;
  in.memory = unit_memory_model(p, v, n);
  in.seq_len = n;
  const SimResult r = simulate(generate(scheme, gc), in);
  std::int64_t peak = 0;
  for (const DeviceMemory& dm : r.memory.per_device) peak = std::max(peak, dm.peak_activation_units);
  return {Rat(peak, n * p * v), r.metrics.bubble_fraction};
}

// exact forms must match to 1e-9; upper bounds may not be exceeded; interval
// forms get a ±10 % band
bool bubble_within(const BubbleBound& bb, double simulated, double* closed_out) {
  if (bb.exact) {
    const double c = bb.exact->to_double();
    *closed_out = c;
    return bb.upper_bound_only ? simulated <= c + 1e-9 : std::abs(simulated - c) < 1e-9;
  }
  const double lo = bb.interval->first.to_double(), hi = bb.interval->second.to_double();
  *closed_out = hi;
  return simulated >= 0.9 * lo - 1e-9 && simulated <= 1.1 * hi + 1e-9;
}

}  // namespace

std::vector<CompareRow> compare_report(const std::vector<Scheme>& schemes, const std::vector<std::int64_t>& ps,
                                       const std::vector<std::int64_t>& vs, const std::vector<std::int64_t>& ms,
                                       const std::vector<std::int64_t>& ns_per_p) {
  std::vector<CompareRow> rows;
  for (Scheme scheme : schemes) {
    const bool sliced = scheme == Scheme::SlimPipe || scheme == Scheme::TeraPipe;
    for (std::int64_t p : ps)
      for (std::int64_t v : vs)
        for (std::int64_t m : ms) {
          std::vector<std::int64_t> ns{1};
          if (sliced) {
            ns.clear();
            for (std::int64_t k : ns_per_p) ns.push_back(k * p);
          }
          for (std::int64_t n : ns) {
            if (!scheme_accepts(scheme, p, m, n, v)) continue;
            const auto [sim_mem, sim_bubble] = simulated_point(scheme, p, v, m, n);
            const Rat closed_mem = memory_multiplier(scheme, p, m, n, v);
            CompareRow row{scheme, p, v, m, n, closed_mem.to_double(), 0.0, sim_mem.to_double(), sim_bubble,
                           true, true};
            row.memory_exact = !memory_form_valid(scheme, p, m, n, v) || sim_mem == closed_mem;
            row.within_bound = bubble_within(bubble_bounds(scheme, p, m, n, v), sim_bubble, &row.closed_bubble);
            rows.push_back(row);
          }
        }
  }
  return rows;
}

std::string compare_report_csv(const std::vector<CompareRow>& rows) {
  auto g10 = [](double x) {
    char b[64];
    std::snprintf(b, sizeof b, "%.10g", x);
    return std::string(b);
  };
  std::ostringstream csv;
  csv << "scheme,p,v,m,n,closed_memory,simulated_memory,memory_exact,closed_bubble,simulated_bubble,within_bound\n";
  for (const CompareRow& r : rows)
    csv << to_string(r.scheme) << ',' << r.p << ',' << r.v << ',' << r.m << ',' << r.n << ',' << g10(r.closed_memory)
        << ',' << g10(r.simulated_memory) << ',' << int(r.memory_exact) << ',' << g10(r.closed_bubble) << ','
        << g10(r.simulated_bubble) << ',' << int(r.within_bound) << '\n';
  return csv.str();
}

}  // namespace pipelab
