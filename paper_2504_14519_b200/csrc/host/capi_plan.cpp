// extern "C" planning entry points of libslimpipe.so (declared in
// include/slimpipe.h).  They expose the pipelab planning layer to the Python
// host mirror and the parity tests as JSON text in the neutral format that
// oracle/ref_shim.cpp emits for the reference, so plans can be compared
// byte-for-byte.  Status codes, no exceptions across the ABI.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include "pipelab/analytics.hpp"
#include "pipelab/exchange.hpp"
#include "pipelab/gantt.hpp"
#include "pipelab/scenario.hpp"
#include "pipelab/schedule.hpp"
#include "pipelab/simulator.hpp"
#include "pipelab/workload.hpp"
#include "errors.hpp"
#include "slimpipe.h"
#include "xplan.hpp"

using namespace pipelab;

namespace {

char* to_c(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

std::string escaped(const char* what) {  // for the {"error", "what"} JSON
  std::string s;
  for (const char* c = what; *c; ++c) {
    if (*c == '"' || *c == '\\') s += '\\';
    s += *c;
  }
  return s;
}

template <class F>
int guarded(char** out, F&& body) {
  try {
    *out = to_c(body());
    return SP_OK;
  } catch (const std::invalid_argument& e) {
    sp::last_error() = e.what();
    *out = to_c(std::string("{\"error\":\"invalid_argument\",\"what\":\"") + escaped(e.what()) + "\"}");
    return SP_ERR_INVALID;
  } catch (const std::exception& e) {
    sp::last_error() = e.what();
    *out = to_c(std::string("{\"error\":\"runtime_error\",\"what\":\"") + escaped(e.what()) + "\"}");
    return SP_ERR_RUNTIME;
  }
}

GenConfig gen_cfg(int p, int v, int m, int n) {
  GenConfig c;
  c.p = p;
  c.v = v;
  c.m = m;
  c.n = n;
  c.cost.alpha_linear = 1.0;
  c.cost.beta_attn = 1.0;
  c.seq_len = n;
  return c;
}

std::string q(const Rat& r) { return "\"" + r.str() + "\""; }

std::string g17(double x) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", x);
  return b;
}

template <class C>
void join(std::ostringstream& os, const C& c) {
  bool first = true;
  for (const auto& x : c) {
    os << (first ? "" : ",") << x;
    first = false;
  }
}

void emit_plan(std::ostringstream& os, const ExchangePlan& p) {
  os << "{\"transfers\":[";
  for (std::size_t t = 0; t < p.transfers.size(); ++t) {
    const Transfer& tr = p.transfers[t];
    os << (t ? "," : "") << "{\"src\":" << tr.src << ",\"dst\":" << tr.dst << ",\"chunks\":[";
    join(os, tr.kv_chunk_indices);
    os << "],\"q\":" << int(tr.carries_query) << ",\"o\":" << int(tr.carries_output) << "}";
  }
  os << "],\"loads\":[";
  join(os, p.resulting_loads);
  os << "]}";
}

std::string annotation_json(const ExchangeAnnotation& ann) {
  std::ostringstream os;
  os << "{\"mode\":" << int(ann.mode) << ",\"ticks\":[";
  for (std::size_t t = 0; t < ann.ticks.size(); ++t) {
    const TickPlan& tp = ann.ticks[t];
    os << (t ? "," : "") << "{\"tick\":" << tp.tick << ",\"fwd\":" << int(tp.forward)
       << ",\"junc\":" << int(tp.juncture) << ",\"in\":[";
    for (std::size_t x = 0; x < tp.loads.size(); ++x)
      os << (x ? "," : "") << "[" << tp.loads[x].device << "," << tp.loads[x].kv_chunks << "," << tp.passes[x]
         << "]";
    os << "],\"plan\":";
    emit_plan(os, tp.plan);
    os << "}";
  }
  os << "],\"balanced\":[";
  bool first = true;
  for (const auto& [pid, c] : ann.balanced_chunks) {
    os << (first ? "" : ",") << "[" << pid << "," << c << "]";
    first = false;
  }
  os << "]}";
  return os.str();
}

}  // namespace

extern "C" {

void sp_free(char* p) { std::free(p); }

int sp_plan_schedule_json(int scheme, int p, int v, int m, int n, char** out) {
  return guarded(out, [&] { return schedule_to_json(generate(Scheme(scheme), gen_cfg(p, v, m, n))); });
}

int sp_plan_validate_json(int p, int v, int m, int n, int mutation, char** out) {
  return guarded(out, [&] {
    Schedule s = gen_slimpipe(gen_cfg(p, v, m, n));
    if (mutation == 1) {
      auto& ord = s.device_order[0];
      int a = -1, b = -1;
      for (std::size_t x = 0; x < ord.size(); ++x) {
        const Pass& ps = s.passes[ord[x]];
        if (ps.kind == PassKind::BackwardFused && ps.microbatch == 1) {
          if (ps.slice == 2) a = int(x);
          if (ps.slice == 1) b = int(x);
        }
      }
      if (a >= 0 && b >= 0) std::swap(ord[a], ord[b]);
    } else if (mutation == 2 && s.device_order.size() > 1) {
      s.device_order[1].pop_back();
    } else if (mutation == 3) {
      s.edges.push_back({s.device_order[0][1], s.device_order[0][0]});
    }
    const Diagnostics d = validate_schedule(s);
    std::ostringstream os;
    os << "[";
    for (std::size_t x = 0; x < d.violations.size(); ++x) {
      const Violation& vi = d.violations[x];
      os << (x ? "," : "") << "{\"rule\":\"" << vi.rule << "\",\"message\":\"" << vi.message
         << "\",\"pass\":" << (vi.pass ? *vi.pass : -2) << "}";
    }
    os << "]";
    return os.str();
  });
}

int sp_plan_balance_json(const int64_t* loads, const int32_t* devices, int count, int early, char** out) {
  return guarded(out, [&] {
    std::vector<TickLoad> tl;
    for (int x = 0; x < count; ++x) tl.push_back({devices[x], loads[x]});
    ExchangePlan plan = balance_tick(tl);
    if (early) plan = to_early_exchange(tl, plan);
    std::ostringstream os;
    emit_plan(os, plan);
    return os.str();
  });
}

int sp_plan_exchange_json(int p, int v, int m, int n, int mode, double beta, char** out) {
  return guarded(out, [&] {
    GenConfig c = gen_cfg(p, v, m, n);
    CostModel cm = c.cost;
    cm.beta_attn = beta;
    return annotation_json(apply_exchange(gen_slimpipe(c), cm, ExchangeMode(mode)));
  });
}

int sp_exchange_passes_json(int p, int m, int n, int mode, int rank, int min_chunks, int skip_last, char** out) {
  return guarded(out, [&] {
    if (rank < 0 || rank >= p) throw std::invalid_argument("rank out of range");
    GenConfig c = gen_cfg(p, 1, m, n);
    const Schedule s = gen_slimpipe(c);
    CostModel cm = c.cost;
    cm.beta_attn = 1.0;  // as the runtime: the plan depends on slice indices only
    const auto xp = sp::exchange_passes(s, apply_exchange(s, cm, ExchangeMode(mode)), rank, p, min_chunks,
                                        skip_last != 0);
    std::ostringstream o;
    auto ints = [&](const std::vector<int>& v) {
      o << '[';
      for (std::size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
      o << ']';
    };
    o << '[';
    bool first = true;
    for (const auto& [pid, px] : xp) {
      const Pass& ps = s.passes[pid];
      o << (first ? "" : ",") << "{\"pass\":" << pid << ",\"kind\":\"" << (ps.kind == PassKind::Forward ? "F" : "BW")
        << "\",\"microbatch\":" << ps.microbatch << ",\"slice\":" << ps.slice << ",\"cls\":" << px.cls
        << ",\"out\":[";
      for (std::size_t i = 0; i < px.out.size(); ++i) {
        o << (i ? "," : "") << "{\"peer\":" << px.out[i].peer << ",\"base\":" << px.out[i].base << ",\"chunks\":";
        ints(px.out[i].chunks);
        o << '}';
      }
      o << "],\"in\":[";
      for (std::size_t i = 0; i < px.in.size(); ++i) {
        o << (i ? "," : "") << "{\"peer\":" << px.in[i].peer << ",\"i_src\":" << px.in[i].i_src
          << ",\"base\":" << px.in[i].base << ",\"chunks\":";
        ints(px.in[i].chunks);
        o << '}';
      }
      o << "]}";
      first = false;
    }
    o << ']';
    return o.str();
  });
}

int sp_plan_activation_json(const int64_t* model, const int64_t* par, const int64_t* run, double offload,
                            char** out) {
  return guarded(out, [&] {
    ModelConfig mc;
    mc.layers = model[0];
    mc.hidden = model[1];
    mc.ffn_hidden = model[2];
    mc.heads = model[3];
    mc.query_groups = model[4];
    mc.vocab = model[5];
    mc.bytes_per_element = model[6];
    mc.loss_bytes_per_element = model[7];
    ParallelismConfig pc;
    pc.tp = par[0];
    pc.cp = par[1];
    pc.pp = par[2];
    pc.stages_per_device = par[3];
    RunConfig rc;
    rc.seq_len = run[0];
    rc.microbatches = run[1];
    rc.slices = run[2];
    rc.checkpointing = Checkpointing(run[3]);
    rc.offload_ratio = offload;
    const MemoryModel mm = activation_bytes(mc, pc, rc);
    std::ostringstream os;
    os << "{\"ptl\":" << q(mm.per_token_layer_bytes) << ",\"mh\":" << q(mm.embedding_bytes)
       << ",\"ma\":" << q(mm.microbatch_activation_bytes) << ",\"slice_stage\":" << q(mm.slice_stage_bytes)
       << ",\"logits_slice\":" << q(mm.logits_slice_bytes) << ",\"exchange_slice\":" << q(mm.exchange_slice_bytes)
       << "}";
    return os.str();
  });
}

// Closed forms of analytics.hpp for one (scheme, p, m, n, v): JSON with the
// rationals as "num/den" strings.
int sp_plan_analytics_json(int scheme, int64_t p, int64_t m, int64_t n, int64_t v, int64_t ma_num, int64_t ma_den,
                           char** out) {
  return guarded(out, [&] {
    const Scheme sc = Scheme(scheme);
    std::string j = "{\"accepts\":" + std::string(scheme_accepts(sc, p, m, n, v) ? "true" : "false");
    j += ",\"form_valid\":" + std::string(memory_form_valid(sc, p, m, n, v) ? "true" : "false");
    j += ",\"memory\":" + q(memory_multiplier(sc, p, m, n, v));
    const BubbleBound b = bubble_bounds(sc, p, m, n, v);
    if (b.exact) j += ",\"bubble\":" + q(*b.exact);
    if (b.interval) j += ",\"bubble_lo\":" + q(b.interval->first) + ",\"bubble_hi\":" + q(b.interval->second);
    j += ",\"upper_only\":" + std::string(b.upper_bound_only ? "true" : "false");
    if (sc == Scheme::SlimPipe) {
      j += ",\"attention_bubble\":" + q(slim_attention_bubble(p, m, n, v));
      if (n >= p) j += ",\"acc_memory\":" + q(slim_acc_memory(p, n, Rat(ma_num, ma_den)));
    }
    return j + "}";
  });
}

int sp_plan_exchange_volume(int64_t p, int64_t n, int64_t L, int64_t mh_num, int64_t mh_den, char** out) {
  return guarded(out, [&] {
    return "{\"theta\":" + q(exchange_volume(p, n, L, Rat(mh_num, mh_den))) +
           ",\"bound\":" + q(exchange_volume_bound(p, n, L, Rat(mh_num, mh_den))) + "}";
  });
}

int sp_plan_simulate_json(int p, int v, int m, int n, int mode, const double* cost, const double* comm,
                          int64_t seq_len, const int64_t* mem_rats, char** out) {
  return guarded(out, [&] {
    Schedule s = gen_slimpipe(gen_cfg(p, v, m, n));
    SimInputs in;
    in.cost.alpha_linear = cost[0];
    in.cost.beta_attn = cost[1];
    in.cost.bwd_input_mult = cost[2];
    in.cost.bwd_weight_mult = cost[3];
    in.comm.bandwidth = comm[0];
    in.comm.latency = comm[1];
    in.seq_len = seq_len;
    in.exchange = ExchangeMode(mode);
    if (mem_rats) {
      in.memory.per_token_layer_bytes = Rat(mem_rats[0], mem_rats[1]);
      in.memory.embedding_bytes = Rat(mem_rats[2], mem_rats[3]);
      in.memory.microbatch_activation_bytes = Rat(mem_rats[4], mem_rats[5]);
      in.memory.slice_stage_bytes = Rat(mem_rats[6], mem_rats[7]);
      in.memory.logits_slice_bytes = Rat(mem_rats[8], mem_rats[9]);
      in.memory.exchange_slice_bytes = Rat(mem_rats[10], mem_rats[11]);
    } else {
      in.memory = unit_memory_model(p, v, n);
    }
    const SimResult r = simulate(s, in);
    std::ostringstream os;
    os << "{\"makespan\":" << g17(r.metrics.makespan) << ",\"bubble\":" << g17(r.metrics.bubble_fraction)
       << ",\"busy\":[";
    for (int d = 0; d < p; ++d) os << (d ? "," : "") << g17(r.metrics.device_busy[d]);
    os << "],\"phases\":[";
    for (int d = 0; d < p; ++d) {
      const DevicePhases& ph = r.metrics.phases[d];
      os << (d ? "," : "") << "[" << g17(ph.warmup_idle) << "," << g17(ph.midstream_idle) << ","
         << g17(ph.cooldown_idle) << "]";
    }
    os << "],\"p2p\":[";
    for (int d = 0; d < p; ++d) os << (d ? "," : "") << q(r.metrics.p2p_bytes_sent[d]);
    os << "],\"exchange\":[";
    for (int d = 0; d < p; ++d) os << (d ? "," : "") << q(r.metrics.exchange_bytes[d]);
    os << "],\"exchange_per_mb\":" << q(r.metrics.exchange_bytes_per_microbatch_device)
       << ",\"fticks\":" << r.metrics.forward_ticks << ",\"jticks\":" << r.metrics.juncture_ticks
       << ",\"memory\":[";
    for (int d = 0; d < p; ++d) {
      const DeviceMemory& dm = r.memory.per_device[d];
      os << (d ? "," : "") << "{\"peak\":" << dm.peak_activation_units << ",\"pool\":" << dm.chunk_pool_size
         << ",\"final\":" << dm.final_activation_units << ",\"peak_bytes\":" << q(dm.peak_activation_bytes)
         << ",\"units\":[";
      for (std::size_t x = 0; x < dm.steps.size(); ++x) os << (x ? "," : "") << dm.steps[x].activation_units;
      os << "],\"times\":[";
      for (std::size_t x = 0; x < dm.steps.size(); ++x) os << (x ? "," : "") << g17(dm.steps[x].time);
      os << "]}";
    }
    os << "],\"timeline\":[";
    for (int d = 0; d < p; ++d) {
      os << (d ? "," : "") << "[";
      const auto& tl = r.timeline.per_device[d];
      for (std::size_t x = 0; x < tl.size(); ++x)
        os << (x ? "," : "") << "[" << tl[x].pass << "," << g17(tl[x].start) << "," << g17(tl[x].end) << "]";
      os << "]";
    }
    os << "],\"transfers\":" << r.timeline.transfers.size() << "}";
    return os.str();
  });
}

// place_vocab (simulator.cpp:414-522) on gen_slimpipe(p, v, m, n) with the
// given base-simulation costs; the result's validity and per-device order
// ([kind, microbatch, slice, stage] per pass).
int sp_plan_vocab_json(int p, int v, int m, int n, int distribute, double alpha, double beta, int64_t seq_len,
                       char** out) {
  return guarded(out, [&] {
    Schedule s = gen_slimpipe(gen_cfg(p, v, m, n));
    SimInputs in;
    in.cost.alpha_linear = alpha;
    in.cost.beta_attn = beta;
    in.seq_len = seq_len;
    const Schedule out = place_vocab(s, distribute != 0, in);
    const Diagnostics d = validate_schedule(out);
    std::ostringstream os;
    os << "{\"valid\":" << (d.ok() ? "true" : "false") << ",\"violations\":" << d.violations.size()
       << ",\"order\":[";
    for (std::size_t dev = 0; dev < out.device_order.size(); ++dev) {
      os << (dev ? "," : "") << "[";
      for (std::size_t x = 0; x < out.device_order[dev].size(); ++x) {
        const Pass& q = out.passes[out.device_order[dev][x]];
        os << (x ? "," : "") << "[" << int(q.kind) << "," << q.microbatch << "," << q.slice << "," << q.stage << "]";
      }
      os << "]";
    }
    os << "]}";
    return os.str();
  });
}

// Scenario text -> the normalised scenario JSON (reference scenario.cpp
// scenario_from_json then scenario_to_json); malformed JSON, wrong types and
// unknown fields are SP_ERR_INVALID.
int sp_plan_scenario_json(const char* text, char** out) {
  return guarded(out, [&] { return scenario_to_json(scenario_from_json(text)); });
}

// Gantt (JSON, or SVG when svg != 0) of simulate(gen_slimpipe(p, v, m, n))
// with the inputs of sp_plan_simulate_json and the unit memory model.
int sp_plan_gantt_json(int p, int v, int m, int n, int mode, const double* cost, const double* comm,
                       int64_t seq_len, int svg, char** out) {
  return guarded(out, [&] {
    const Schedule s = gen_slimpipe(gen_cfg(p, v, m, n));
    SimInputs in;
    in.cost.alpha_linear = cost[0];
    in.cost.beta_attn = cost[1];
    in.cost.bwd_input_mult = cost[2];
    in.cost.bwd_weight_mult = cost[3];
    in.comm.bandwidth = comm[0];
    in.comm.latency = comm[1];
    in.seq_len = seq_len;
    in.exchange = ExchangeMode(mode);
    in.memory = unit_memory_model(p, v, n);
    const SimResult r = simulate(s, in);
    return svg ? gantt_svg(s, r.timeline) : gantt_json(s, r.timeline);
  });
}

namespace {
// executor schedule + a measured per-device timeline (see sp_plan_gantt_measured)
std::pair<Schedule, Timeline> measured(int p, int v, int m, int n, int vocab_parallel, int64_t seq_len,
                                       const int32_t* counts, const int32_t* pass_ids, const double* starts,
                                       const double* ends) {
  Schedule s = gen_slimpipe(gen_cfg(p, v, m, n));
  if (vocab_parallel) {
    SimInputs in;
    in.cost.alpha_linear = 1.0 / double(seq_len);
    in.cost.beta_attn = 1.0 / (double(seq_len) * double(seq_len));
    in.seq_len = seq_len;
    s = place_vocab(s, true, in);
  }
  Timeline tl;
  tl.per_device.resize(static_cast<size_t>(p));
  int64_t x = 0;
  for (int d = 0; d < p; ++d)
    for (int e = 0; e < counts[d]; ++e, ++x) {
      if (pass_ids[x] < 0 || size_t(pass_ids[x]) >= s.passes.size())
        throw std::invalid_argument("measured timeline: pass id out of range");
      tl.per_device[size_t(d)].push_back({PassId(pass_ids[x]), starts[x], ends[x]});
      tl.makespan = std::max(tl.makespan, ends[x]);
    }
  return {std::move(s), std::move(tl)};
}
}  // namespace

// The reference's metric definitions (simulator.cpp:348-409) on a measured
// timeline: makespan, bubble fraction, per-device busy / idle and phases.
int sp_plan_metrics_measured(int p, int v, int m, int n, int vocab_parallel, int64_t seq_len, const int32_t* counts,
                             const int32_t* pass_ids, const double* starts, const double* ends, char** out) {
  return guarded(out, [&] {
    auto [s, tl] = measured(p, v, m, n, vocab_parallel, seq_len, counts, pass_ids, starts, ends);
    const Metrics mt = metrics_from_timeline(s, tl, unit_memory_model(p, v, n), ExchangeAnnotation{});
    std::ostringstream os;
    os << "{\"makespan\":" << g17(mt.makespan) << ",\"bubble\":" << g17(mt.bubble_fraction) << ",\"busy\":[";
    for (int d = 0; d < p; ++d) os << (d ? "," : "") << g17(mt.device_busy[size_t(d)]);
    os << "],\"idle\":[";
    for (int d = 0; d < p; ++d) os << (d ? "," : "") << g17(mt.device_idle[size_t(d)]);
    os << "],\"phases\":[";
    for (int d = 0; d < p; ++d) {
      const DevicePhases& ph = mt.phases[size_t(d)];
      os << (d ? "," : "") << "[" << g17(ph.warmup_idle) << "," << g17(ph.midstream_idle) << ","
         << g17(ph.cooldown_idle) << "]";
    }
    os << "]}";
    return os.str();
  });
}

// Gantt of a MEASURED step: the executors' schedule (gen_slimpipe(p, v, m, n),
// plus place_vocab with the runtime's normalised costs when vocab_parallel)
// and each device's CUDA-event spans (counts[d] passes: pass id, start, end
// in ms, devices concatenated in order).
int sp_plan_gantt_measured(int p, int v, int m, int n, int vocab_parallel, int64_t seq_len, const int32_t* counts,
                           const int32_t* pass_ids, const double* starts, const double* ends, int svg, char** out) {
  return guarded(out, [&] {
    auto [s, tl] = measured(p, v, m, n, vocab_parallel, seq_len, counts, pass_ids, starts, ends);
    return svg ? gantt_svg(s, tl) : gantt_json(s, tl);
  });
}

}  // extern "C"
