// Point-to-point transport of the step executor (runtime.cpp).
//
// A Link is one communicator: ranks 0..size-1, FIFO send/recv per ordered
// (sender, receiver) pair, stream-ordered on both ends, and group semantics
// like ncclGroupStart/End (the operations of a group may complete in any
// order, so a group holding both a send to and a receive from the same peer
// cannot deadlock against the peer's mirror group).  The executor's stage
// edges (reference schedule.cpp:102-130 cross-device edges) and the exchange
// transfers (simulator.cpp:56-108 tick plans) are written against it.
//
// Two implementations:
//   * NCCL (one process per GPU, NVLink/NVSwitch) — the production path;
//   * loopback (every rank a host thread of ONE process on ONE GPU): a
//     receive publishes its destination and raises a device flag; the
//     matching send waits for that flag, copies straight into the
//     destination and raises a "done" flag that the receive's stream waits
//     on.  Waits and signals are all small kernels (a spinning one-CTA wait,
//     a one-thread release store), like NCCL's, never stream memory
//     operations: a front-end wait or a write that must wait for its
//     stream's previous kernel holds the whole hardware channel, and a
//     channel shared with a peer's stream closes a cycle.  No host-side rendezvous, so the host enqueue
//     never blocks on a peer — the same progress semantics as NCCL.  It lets
//     a single-GPU box run (and test) the multi-stage protocol bit for bit.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <memory>
#include <vector>

namespace sp {

class Link {
 public:
  virtual ~Link() = default;
  virtual int send(const void* buf, int64_t count, ncclDataType_t dt, int peer, cudaStream_t st) = 0;
  virtual int recv(void* buf, int64_t count, ncclDataType_t dt, int peer, cudaStream_t st) = 0;
  virtual int group_start() = 0;
  virtual int group_end() = 0;
  // collectives (vocabulary parallelism); the loopback link does not offer them
  virtual int broadcast(void* buf, int64_t count, ncclDataType_t dt, int root, cudaStream_t st);
  virtual int all_reduce(float* buf, int64_t count, ncclRedOp_t op, cudaStream_t st);
  virtual int reduce(float* buf, int64_t count, int root, cudaStream_t st);
  // pre-size any scratch the collectives need for `count` floats (allocation
  // must not happen inside an enqueued step)
  virtual int reserve(int64_t count) { return 0; }
};

// Takes ownership of `comm` (destroyed with the link).
std::unique_ptr<Link> make_nccl_link(ncclComm_t comm);

// Loopback world of `ranks` threads on the current device.
struct LoopWorld;
LoopWorld* loop_world_create(int ranks);
void loop_world_destroy(LoopWorld* w);
int loop_world_size(const LoopWorld* w);
int loop_world_errors(const LoopWorld* w);  // size mismatches seen by the copy kernel
// Communicator `comm_id` (independent FIFO space per id) over the global
// ranks `members` (link rank x = members[x]); `me` is this link's own rank.
std::unique_ptr<Link> make_loop_link(LoopWorld* w, int comm_id, std::vector<int> members, int me);

}  // namespace sp
