// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" bridge over the *unmodified* reference sources
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libpipelab_ref.so).  Every function serialises a reference
// result into the same neutral JSON text the product's sp_plan_* entry points
// emit (paper_2504_14519_b200/csrc/host/capi_plan.cpp), so the parity tests can
// compare the two byte-for-byte.  Only tests/ and bench.py's cpu_baseline leg
// may load this library.
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <future>
#include <mutex>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "pipelab/attention.hpp"
#include "pipelab/analytics.hpp"
#include "pipelab/exchange.hpp"
#include "pipelab/gantt.hpp"
#include "pipelab/scenario.hpp"
#include "pipelab/schedule.hpp"
#include "pipelab/simulator.hpp"
#include "pipelab/workload.hpp"

using namespace pipelab;

namespace {

char* dup(const std::string& s) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.data(), s.size() + 1);
  return out;
}

char* error_json(const char* kind, const std::exception& e) {
  std::ostringstream os;
  os << "{\"error\":\"" << kind << "\",\"what\":\"" << e.what() << "\"}";
  return dup(os.str());
}

GenConfig make_cfg(int p, int v, int m, int n) {
  GenConfig c;
  c.p = p; c.v = v; c.m = m; c.n = n;
  c.cost.alpha_linear = 1.0;
  c.cost.beta_attn = 1.0;
  c.seq_len = n;
  return c;
}

void put_plan(std::ostringstream& os, const ExchangePlan& plan) {
  os << "{\"transfers\":[";
  for (size_t t = 0; t < plan.transfers.size(); ++t) {
    const Transfer& tr = plan.transfers[t];
    if (t) os << ",";
    os << "{\"src\":" << tr.src << ",\"dst\":" << tr.dst << ",\"chunks\":[";
    for (size_t c = 0; c < tr.kv_chunk_indices.size(); ++c)
      os << (c ? "," : "") << tr.kv_chunk_indices[c];
    os << "],\"q\":" << (tr.carries_query ? 1 : 0)
       << ",\"o\":" << (tr.carries_output ? 1 : 0) << "}";
  }
  os << "],\"loads\":[";
  for (size_t i = 0; i < plan.resulting_loads.size(); ++i)
    os << (i ? "," : "") << plan.resulting_loads[i];
  os << "]}";
}

std::string rat(const Rat& r) { return "\"" + r.str() + "\""; }

std::string dbl(double x) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", x);
  return buf;
}

Schedule mutate(Schedule s, int mutation) {
  if (mutation == 1) {  // swap BW(1,2) and BW(1,1) on device 1
    auto& order = s.device_order[0];
    int a = -1, b = -1;
    for (size_t i = 0; i < order.size(); ++i) {
      const Pass& ps = s.passes[order[i]];
      if (ps.kind == PassKind::BackwardFused && ps.microbatch == 1) {
        if (ps.slice == 2) a = static_cast<int>(i);
        if (ps.slice == 1) b = static_cast<int>(i);
      }
    }
    if (a >= 0 && b >= 0) std::swap(order[a], order[b]);
  } else if (mutation == 2) {  // drop the last pass of device 2
    if (s.device_order.size() > 1) s.device_order[1].pop_back();
  } else if (mutation == 3) {  // cycle-closing edge
    s.edges.push_back({s.device_order[0][1], s.device_order[0][0]});
  }
  return s;
}

}  // namespace

extern "C" {

void ref_free(char* p) { std::free(p); }

char* ref_schedule_json(int scheme, int p, int v, int m, int n) {
  try {
    return dup(schedule_to_json(generate(static_cast<Scheme>(scheme), make_cfg(p, v, m, n))));
  } catch (const std::invalid_argument& e) {
    return error_json("invalid_argument", e);
  } catch (const std::exception& e) {
    return error_json("runtime_error", e);
  }
}

char* ref_validate_json(int p, int v, int m, int n, int mutation) {
  try {
    Schedule s = mutate(gen_slimpipe(make_cfg(p, v, m, n)), mutation);
    Diagnostics d = validate_schedule(s);
    std::ostringstream os;
    os << "[";
    for (size_t i = 0; i < d.violations.size(); ++i) {
      const Violation& vi = d.violations[i];
      os << (i ? "," : "") << "{\"rule\":\"" << vi.rule << "\",\"message\":\""
         << vi.message << "\",\"pass\":" << (vi.pass ? *vi.pass : -2) << "}";
    }
    os << "]";
    return dup(os.str());
  } catch (const std::exception& e) {
    return error_json("invalid_argument", e);
  }
}

char* ref_balance_json(const int64_t* loads, const int32_t* devices, int count, int early) {
  try {
    std::vector<TickLoad> tl;
    for (int i = 0; i < count; ++i) tl.push_back({devices[i], loads[i]});
    ExchangePlan plan = balance_tick(tl);
    if (early) plan = to_early_exchange(tl, plan);
    std::ostringstream os;
    put_plan(os, plan);
    return dup(os.str());
  } catch (const std::exception& e) {
    return error_json("invalid_argument", e);
  }
}

char* ref_exchange_json(int p, int v, int m, int n, int mode, double beta) {
  try {
    GenConfig c = make_cfg(p, v, m, n);
    Schedule s = gen_slimpipe(c);
    CostModel cm = c.cost;
    cm.beta_attn = beta;
    ExchangeAnnotation ann = apply_exchange(s, cm, static_cast<ExchangeMode>(mode));
    std::ostringstream os;
    os << "{\"mode\":" << static_cast<int>(ann.mode) << ",\"ticks\":[";
    for (size_t t = 0; t < ann.ticks.size(); ++t) {
      const TickPlan& tp = ann.ticks[t];
      os << (t ? "," : "") << "{\"tick\":" << tp.tick << ",\"fwd\":" << (tp.forward ? 1 : 0)
         << ",\"junc\":" << (tp.juncture ? 1 : 0) << ",\"in\":[";
      for (size_t i = 0; i < tp.loads.size(); ++i)
        os << (i ? "," : "") << "[" << tp.loads[i].device << "," << tp.loads[i].kv_chunks << ","
           << tp.passes[i] << "]";
      os << "],\"plan\":";
      put_plan(os, tp.plan);
      os << "}";
    }
    os << "],\"balanced\":[";
    bool first = true;
    for (const auto& [pid, ch] : ann.balanced_chunks) {
      os << (first ? "" : ",") << "[" << pid << "," << ch << "]";
      first = false;
    }
    os << "]}";
    return dup(os.str());
  } catch (const std::invalid_argument& e) {
    return error_json("invalid_argument", e);
  } catch (const std::exception& e) {
    return error_json("runtime_error", e);
  }
}

// Model / run arrays: model = {L,h,H,a,g,V,bytes,loss_bytes}; par = {t,c,p,v};
// run = {S,m,n,ckpt(0 none,1 sel,2 full)}; offload as double.
char* ref_activation_json(const int64_t* model, const int64_t* par, const int64_t* run,
                          double offload) {
  try {
    ModelConfig mc{model[0], model[1], model[2], model[3], model[4], model[5], model[6], model[7]};
    ParallelismConfig pc;
    pc.tp = par[0]; pc.cp = par[1]; pc.pp = par[2]; pc.stages_per_device = par[3];
    RunConfig rc;
    rc.seq_len = run[0]; rc.microbatches = run[1]; rc.slices = run[2];
    rc.checkpointing = static_cast<Checkpointing>(run[3]);
    rc.offload_ratio = offload;
    MemoryModel mm = activation_bytes(mc, pc, rc);
    std::ostringstream os;
    os << "{\"ptl\":" << rat(mm.per_token_layer_bytes) << ",\"mh\":" << rat(mm.embedding_bytes)
       << ",\"ma\":" << rat(mm.microbatch_activation_bytes)
       << ",\"slice_stage\":" << rat(mm.slice_stage_bytes)
       << ",\"logits_slice\":" << rat(mm.logits_slice_bytes)
       << ",\"exchange_slice\":" << rat(mm.exchange_slice_bytes) << "}";
    return dup(os.str());
  } catch (const std::exception& e) {
    return error_json("invalid_argument", e);
  }
}

// The reference's closed forms (analytics.cpp:11-112), same JSON layout as
// sp_plan_analytics_json.
char* ref_analytics_json(int scheme, int64_t p, int64_t m, int64_t n, int64_t v, int64_t ma_num, int64_t ma_den) {
  try {
    const Scheme sc = Scheme(scheme);
    std::string j = "{\"accepts\":" + std::string(scheme_accepts(sc, p, m, n, v) ? "true" : "false");
    j += ",\"form_valid\":" + std::string(memory_form_valid(sc, p, m, n, v) ? "true" : "false");
    j += ",\"memory\":" + rat(memory_multiplier(sc, p, m, n, v));
    const BubbleBound b = bubble_bounds(sc, p, m, n, v);
    if (b.exact) j += ",\"bubble\":" + rat(*b.exact);
    if (b.interval) j += ",\"bubble_lo\":" + rat(b.interval->first) + ",\"bubble_hi\":" + rat(b.interval->second);
    j += ",\"upper_only\":" + std::string(b.upper_bound_only ? "true" : "false");
    if (sc == Scheme::SlimPipe) {
      j += ",\"attention_bubble\":" + rat(slim_attention_bubble(p, m, n, v));
      if (n >= p) j += ",\"acc_memory\":" + rat(slim_acc_memory(p, n, Rat(ma_num, ma_den)));
    }
    return dup(j + "}");
  } catch (const std::exception& e) {
    return error_json("invalid_argument", e);
  }
}

char* ref_exchange_volume(int64_t p, int64_t n, int64_t L, int64_t mh_num, int64_t mh_den) {
  try {
    Rat v = exchange_volume(p, n, L, Rat(mh_num, mh_den));
    Rat b = exchange_volume_bound(p, n, L, Rat(mh_num, mh_den));
    return dup("{\"theta\":" + rat(v) + ",\"bound\":" + rat(b) + "}");
  } catch (const std::exception& e) {
    return error_json("invalid_argument", e);
  }
}

// cost = {alpha, beta, bwd_in, bwd_w}; comm = {bandwidth, latency}; memory is
// the unit model (slice_stage = exchange_slice = 1, M_h = n) unless
// mem_rats (6 num/den pairs: ptl, mh, ma, slice_stage, logits, exchange) given.
char* ref_vocab_json(int p, int v, int m, int n, int distribute, double alpha, double beta, int64_t seq_len) {
  try {
    Schedule s = gen_slimpipe(make_cfg(p, v, m, n));
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
    return dup(os.str());
  } catch (const std::invalid_argument& e) {
    return error_json("invalid_argument", e);
  } catch (const std::exception& e) {
    return error_json("runtime_error", e);
  }
}

char* ref_scenario_json(const char* text) {
  try {
    return dup(scenario_to_json(scenario_from_json(text)));
  } catch (const std::invalid_argument& e) {
    return error_json("invalid_argument", e);
  } catch (const std::exception& e) {
    return error_json("runtime_error", e);
  }
}

char* ref_gantt_json(int p, int v, int m, int n, int mode, const double* cost, const double* comm, int64_t seq_len,
                     int svg) {
  try {
    Schedule s = gen_slimpipe(make_cfg(p, v, m, n));
    SimInputs in;
    in.cost.alpha_linear = cost[0];
    in.cost.beta_attn = cost[1];
    in.cost.bwd_input_mult = cost[2];
    in.cost.bwd_weight_mult = cost[3];
    in.comm.bandwidth = comm[0];
    in.comm.latency = comm[1];
    in.seq_len = seq_len;
    in.exchange = static_cast<ExchangeMode>(mode);
    in.memory = unit_memory_model(p, v, n);
    SimResult r = simulate(s, in);
    return dup(svg ? gantt_svg(s, r.timeline) : gantt_json(s, r.timeline));
  } catch (const std::exception& e) {
    return error_json("runtime_error", e);
  }
}

// a measured timeline given as arrays, through the reference's own exporter
char* ref_gantt_measured(int p, int v, int m, int n, const int32_t* counts, const int32_t* pass_ids,
                         const double* starts, const double* ends, int svg) {
  try {
    Schedule s = gen_slimpipe(make_cfg(p, v, m, n));
    Timeline tl;
    tl.per_device.resize(p);
    int64_t x = 0;
    for (int d = 0; d < p; ++d)
      for (int e = 0; e < counts[d]; ++e, ++x) {
        TimelineEntry te;
        te.pass = pass_ids[x];
        te.start = starts[x];
        te.end = ends[x];
        tl.per_device[d].push_back(te);
        if (ends[x] > tl.makespan) tl.makespan = ends[x];
      }
    return dup(svg ? gantt_svg(s, tl) : gantt_json(s, tl));
  } catch (const std::exception& e) {
    return error_json("runtime_error", e);
  }
}

char* ref_simulate_json(int p, int v, int m, int n, int mode, const double* cost,
                        const double* comm, int64_t seq_len, const int64_t* mem_rats) {
  try {
    GenConfig c = make_cfg(p, v, m, n);
    Schedule s = gen_slimpipe(c);
    SimInputs in;
    in.cost.alpha_linear = cost[0];
    in.cost.beta_attn = cost[1];
    in.cost.bwd_input_mult = cost[2];
    in.cost.bwd_weight_mult = cost[3];
    in.comm.bandwidth = comm[0];
    in.comm.latency = comm[1];
    in.seq_len = seq_len;
    in.exchange = static_cast<ExchangeMode>(mode);
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
    SimResult r = simulate(s, in);
    std::ostringstream os;
    os << "{\"makespan\":" << dbl(r.metrics.makespan)
       << ",\"bubble\":" << dbl(r.metrics.bubble_fraction) << ",\"busy\":[";
    for (int d = 0; d < p; ++d) os << (d ? "," : "") << dbl(r.metrics.device_busy[d]);
    os << "],\"phases\":[";
    for (int d = 0; d < p; ++d)
      os << (d ? "," : "") << "[" << dbl(r.metrics.phases[d].warmup_idle) << ","
         << dbl(r.metrics.phases[d].midstream_idle) << ","
         << dbl(r.metrics.phases[d].cooldown_idle) << "]";
    os << "],\"p2p\":[";
    for (int d = 0; d < p; ++d) os << (d ? "," : "") << rat(r.metrics.p2p_bytes_sent[d]);
    os << "],\"exchange\":[";
    for (int d = 0; d < p; ++d) os << (d ? "," : "") << rat(r.metrics.exchange_bytes[d]);
    os << "],\"exchange_per_mb\":" << rat(r.metrics.exchange_bytes_per_microbatch_device)
       << ",\"fticks\":" << r.metrics.forward_ticks << ",\"jticks\":" << r.metrics.juncture_ticks
       << ",\"memory\":[";
    for (int d = 0; d < p; ++d) {
      const DeviceMemory& dm = r.memory.per_device[d];
      os << (d ? "," : "") << "{\"peak\":" << dm.peak_activation_units
         << ",\"pool\":" << dm.chunk_pool_size << ",\"final\":" << dm.final_activation_units
         << ",\"peak_bytes\":" << rat(dm.peak_activation_bytes) << ",\"units\":[";
      for (size_t i = 0; i < dm.steps.size(); ++i)
        os << (i ? "," : "") << dm.steps[i].activation_units;
      os << "],\"times\":[";
      for (size_t i = 0; i < dm.steps.size(); ++i) os << (i ? "," : "") << dbl(dm.steps[i].time);
      os << "]}";
    }
    os << "],\"timeline\":[";
    for (int d = 0; d < p; ++d) {
      os << (d ? "," : "") << "[";
      const auto& tl = r.timeline.per_device[d];
      for (size_t i = 0; i < tl.size(); ++i)
        os << (i ? "," : "") << "[" << tl[i].pass << "," << dbl(tl[i].start) << ","
           << dbl(tl[i].end) << "]";
      os << "]";
    }
    os << "],\"transfers\":" << r.timeline.transfers.size() << "}";
    return dup(os.str());
  } catch (const std::invalid_argument& e) {
    return error_json("invalid_argument", e);
  } catch (const std::exception& e) {
    return error_json("runtime_error", e);
  }
}

// Reference chunk_attention on row-major fp64 data (one head). chunk_sizes
// partitions the rows of k/v. Writes finalised output and the streaming state.
int ref_chunk_attention(const double* q, int rows, int d, const double* k, const double* v,
                        const int* chunk_sizes, int nchunks, int causal, double* out,
                        double* partial, double* row_max, double* row_sumexp) {
  try {
    Mat qm(rows, d);
    std::memcpy(qm.a.data(), q, sizeof(double) * rows * d);
    std::vector<KvChunk> chunks;
    int pos = 0;
    for (int c = 0; c < nchunks; ++c) {
      int len = chunk_sizes[c];
      KvChunk ch{Mat(len, d), Mat(len, d)};
      std::memcpy(ch.keys.a.data(), k + static_cast<size_t>(pos) * d, sizeof(double) * len * d);
      std::memcpy(ch.values.a.data(), v + static_cast<size_t>(pos) * d, sizeof(double) * len * d);
      pos += len;
      chunks.push_back(std::move(ch));
    }
    auto [o, st] = chunk_attention(qm, chunks, causal != 0);
    std::memcpy(out, o.a.data(), sizeof(double) * rows * d);
    if (partial) std::memcpy(partial, st.partial_output.a.data(), sizeof(double) * rows * d);
    for (int r = 0; r < rows; ++r) {
      if (row_max) row_max[r] = st.row_max[r];
      if (row_sumexp) row_sumexp[r] = st.row_sumexp[r];
    }
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// merge_partials + finalize of two states (partial, max, sumexp each).
int ref_merge(int rows, int d, const double* pa, const double* ma, const double* la,
              const double* pb, const double* mb, const double* lb, double* out_partial,
              double* out_max, double* out_sum, double* out_final) {
  auto load = [&](const double* p, const double* m, const double* l) {
    AttnChunkState s = empty_state(rows, d);
    std::memcpy(s.partial_output.a.data(), p, sizeof(double) * rows * d);
    for (int r = 0; r < rows; ++r) { s.row_max[r] = m[r]; s.row_sumexp[r] = l[r]; }
    return s;
  };
  AttnChunkState o = merge_partials(load(pa, ma, la), load(pb, mb, lb));
  std::memcpy(out_partial, o.partial_output.a.data(), sizeof(double) * rows * d);
  for (int r = 0; r < rows; ++r) { out_max[r] = o.row_max[r]; out_sum[r] = o.row_sumexp[r]; }
  Mat f = finalize(o);
  std::memcpy(out_final, f.a.data(), sizeof(double) * rows * d);
  return 0;
}

// CPU baseline: `heads` independent chunk_attention calls (Ls queries against
// `nchunks` chunks of Ls keys, causal), one std::async task per head as the
// reference CLI sweep does (pipelab_main.cpp:228-239).  Inputs are drawn
// uniform(-1,1) from mt19937_64(seed) like verify.cpp:71-76.  Returns the
// wall seconds of the attention calls only.
double ref_time_chunk_attention(int heads, int ls, int nchunks, int d, int threads,
                                unsigned long long seed) {
  std::vector<Mat> qs;
  std::vector<std::vector<KvChunk>> kvs;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (int h = 0; h < heads; ++h) {
    Mat q(ls, d);
    for (double& x : q.a) x = dist(rng);
    std::vector<KvChunk> ch;
    for (int c = 0; c < nchunks; ++c) {
      KvChunk kc{Mat(ls, d), Mat(ls, d)};
      for (double& x : kc.keys.a) x = dist(rng);
      for (double& x : kc.values.a) x = dist(rng);
      ch.push_back(std::move(kc));
    }
    qs.push_back(std::move(q));
    kvs.push_back(std::move(ch));
  }
  auto t0 = std::chrono::steady_clock::now();
  int next = 0;
  std::mutex mu;
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&]() {
      for (;;) {
        int h;
        {
          std::lock_guard<std::mutex> g(mu);
          h = next++;
        }
        if (h >= heads) return;
        volatile double sink = chunk_attention(qs[h], kvs[h], true).first.a[0];
        (void)sink;
      }
    });
  for (auto& th : pool) th.join();
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"
