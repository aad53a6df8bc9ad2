// The executor's per-pass view of an exchange plan (host only): for one
// rank, which of its passes ship attention work out (Q + KV chunks to a
// peer, partial back) and which serve a peer's pass.  Shared by the runtime
// (runtime.cpp) and the planning C-ABI (sp_exchange_passes_json), so the
// wiring the executor runs is testable without a GPU.
//
// Source: the tick plans of the reference's apply_exchange
// (simulator.cpp:56-108; transfers per tick from balance_tick /
// to_early_exchange, exchange.cpp:10-96), minus the transfers the placement
// filter drops (slimpipe.h exchange_min_chunks / exchange_skip_last).
#pragma once

#include <map>
#include <vector>

#include "pipelab/exchange.hpp"
#include "pipelab/schedule.hpp"
#include "pipelab/simulator.hpp"

namespace sp {

struct XOut {  // this rank ships Q (+ KV chunks) of its pass to `peer`
  int peer;
  std::vector<int> chunks;  // sender-microbatch chunk ids, 1-based, ascending
  int base;                 // chunk offset in this rank's partial-receive pool
};
struct XIn {  // this rank computes a partial for `peer`'s pass
  int peer, i_src;
  std::vector<int> chunks;
  int base;  // chunk offset in the receive pool
};
struct PassX {
  int cls = 0;  // 0 forward tick, 1 backward tick
  std::vector<XOut> out;
  std::vector<XIn> in;
  int in_chunks = 0, out_chunks = 0;
};

// rank is 0-based; p devices.  Transfers are sorted by (src, dst) in every
// tick plan, so both ends post their NCCL calls in the same order.  The
// filter is a pure function of the plan, identical on every rank.
inline std::map<int, PassX> exchange_passes(const pipelab::Schedule& sched, const pipelab::ExchangeAnnotation& ann,
                                            int rank, int p, int min_chunks, bool skip_last) {
  std::map<int, PassX> xplan;
  const int me = rank + 1;
  for (const pipelab::TickPlan& tp : ann.ticks) {
    auto pass_of = [&](int dev) -> int {
      for (std::size_t x = 0; x < tp.loads.size(); ++x)
        if (tp.loads[x].device == dev) return tp.passes[x];
      return -1;
    };
    for (const pipelab::Transfer& tr : tp.plan.transfers) {
      const int sp = pass_of(tr.src), dp = pass_of(tr.dst);
      if (sp < 0 || dp < 0) continue;
      if (int(tr.kv_chunk_indices.size()) < min_chunks) continue;
      if (skip_last && tr.dst == p) continue;
      std::vector<int> ch(tr.kv_chunk_indices.begin(), tr.kv_chunk_indices.end());
      if (tr.src == me) {
        PassX& px = xplan[sp];
        px.cls = tp.forward ? 0 : 1;
        px.out.push_back({tr.dst - 1, ch, px.out_chunks});
        px.out_chunks += int(ch.size());
      }
      if (tr.dst == me) {
        PassX& px = xplan[dp];
        px.cls = tp.forward ? 0 : 1;
        px.in.push_back({tr.src - 1, sched.passes[sp].slice, ch, px.in_chunks});
        px.in_chunks += int(ch.size());
      }
    }
  }
  return xplan;
}

}  // namespace sp
