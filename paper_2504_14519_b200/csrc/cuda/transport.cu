// Transports behind sp::Link (csrc/host/transport.hpp): NCCL for one process
// per GPU, and the single-GPU loopback that runs every rank as a host thread
// of one process (tests and single-GPU boxes).
#include <algorithm>
#include <atomic>
#include <memory>
#include <mutex>
#include <set>
#include <vector>

#include "kernels.hpp"
#include "transport.hpp"

namespace sp {

int Link::broadcast(void*, int64_t, ncclDataType_t, int, cudaStream_t) {
  return set_error(SP_ERR_UNSUPPORTED, "transport: collectives are not available on this link");
}
int Link::all_reduce(float*, int64_t, ncclRedOp_t, cudaStream_t) {
  return set_error(SP_ERR_UNSUPPORTED, "transport: collectives are not available on this link");
}
int Link::reduce(float*, int64_t, int, cudaStream_t) {
  return set_error(SP_ERR_UNSUPPORTED, "transport: collectives are not available on this link");
}

namespace {

int nccl_rc(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return SP_OK;
  return set_error(SP_ERR_NCCL, "%s: %s", what, ncclGetErrorString(r));
}

class NcclLink final : public Link {
 public:
  explicit NcclLink(ncclComm_t c) : c_(c) {}
  ~NcclLink() override {
    if (c_) ncclCommDestroy(c_);
  }
  int send(const void* buf, int64_t count, ncclDataType_t dt, int peer, cudaStream_t st) override {
    return nccl_rc(ncclSend(buf, size_t(count), dt, peer, c_, st), "ncclSend");
  }
  int recv(void* buf, int64_t count, ncclDataType_t dt, int peer, cudaStream_t st) override {
    return nccl_rc(ncclRecv(buf, size_t(count), dt, peer, c_, st), "ncclRecv");
  }
  int group_start() override { return nccl_rc(ncclGroupStart(), "ncclGroupStart"); }
  int group_end() override { return nccl_rc(ncclGroupEnd(), "ncclGroupEnd"); }
  int broadcast(void* buf, int64_t count, ncclDataType_t dt, int root, cudaStream_t st) override {
    return nccl_rc(ncclBroadcast(buf, buf, size_t(count), dt, root, c_, st), "ncclBroadcast");
  }
  int all_reduce(float* buf, int64_t count, ncclRedOp_t op, cudaStream_t st) override {
    return nccl_rc(ncclAllReduce(buf, buf, size_t(count), ncclFloat32, op, c_, st), "ncclAllReduce");
  }
  int reduce(float* buf, int64_t count, int root, cudaStream_t st) override {
    return nccl_rc(ncclReduce(buf, buf, size_t(count), ncclFloat32, ncclSum, root, c_, st), "ncclReduce");
  }

 private:
  ncclComm_t c_;
};

// ------------------------------------------------------------------ loopback
constexpr int kSlots = 4096;  // messages in flight per (communicator, sender, receiver)
constexpr int kComms = 8;

struct Mail {
  void* dst;
  int64_t bytes;
};

struct Channel {
  uint32_t* ready = nullptr;  // device [kSlots]: seq+1 once receive `seq` is posted
  uint32_t* done = nullptr;   // device [kSlots]: seq+1 once send `seq` landed
  Mail* mail = nullptr;       // pinned, device-mapped [kSlots]: receive destinations
  std::atomic<uint64_t> sseq{0}, rseq{0};
};

__device__ __forceinline__ void spin_until(const uint32_t* flag, uint32_t value) {
  uint32_t v;
  while (true) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (int32_t(v - value) >= 0) break;
    __nanosleep(256);
  }
}

// Raise a flag from the stream (everything before it on the stream is
// complete when this kernel runs): a kernel, not a stream memory operation —
// a memop that must wait for the stream's previous kernel holds the whole
// hardware channel, and a channel shared with a peer's spinning wait closes
// a cycle.
__global__ void loop_signal_kernel(uint32_t* flag, uint32_t value) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
  }
}

// A stream-ordered wait that occupies one small CTA (like an NCCL kernel)
// rather than a hardware channel: a front-end stream wait would also stall
// every other stream that shares its channel (CUDA_DEVICE_MAX_CONNECTIONS),
// which with a dozen streams per rank can close a cycle between ranks.
__global__ void loop_wait_kernel(const uint32_t* flag, uint32_t value) {
  if (threadIdx.x == 0) spin_until(flag, value);
}

// The sender's copy, launched behind a loop_wait_kernel on the receive's
// ready flag (one spinning CTA per waiting stream, never a grid of them: a
// grid of spinners could fill every SM and starve the kernel it waits for);
// destination and size come from the receiver's mailbox, published before
// that flag was raised.
__global__ void loop_copy_kernel(const Mail* mail, const uint8_t* __restrict__ src, int64_t bytes, int* err) {
  const volatile Mail* vm = mail;
  uint8_t* dst = static_cast<uint8_t*>(vm->dst);
  if (vm->bytes != bytes) {
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(err, 1);
    return;
  }
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x, nth = int64_t(gridDim.x) * blockDim.x;
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    const int64_t n16 = bytes >> 4;
    const int4* s = reinterpret_cast<const int4*>(src);
    int4* d = reinterpret_cast<int4*>(dst);
    for (int64_t x = tid; x < n16; x += nth) d[x] = s[x];
    for (int64_t x = (n16 << 4) + tid; x < bytes; x += nth) dst[x] = src[x];
  } else {
    for (int64_t x = tid; x < bytes; x += nth) dst[x] = src[x];
  }
}

// out[i] = op(out[i], in[i]) (op 0 sum, 1 max) — the combine step of the
// loopback collectives
__global__ void loop_combine_kernel(float* out, const float* in, int64_t n, int op) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = op ? fmaxf(out[i], in[i]) : out[i] + in[i];
}

}  // namespace

struct LoopWorld {
  int n = 0;
  std::vector<std::unique_ptr<Channel>> ch;  // [comm][src][dst]
  uint32_t* flags = nullptr;
  Mail* mail = nullptr;
  int* err = nullptr;
  Channel& at(int comm, int src, int dst) { return *ch[size_t((comm * n + src) * n + dst)]; }
};

LoopWorld* loop_world_create(int ranks) {
  if (ranks < 1 || preload_kernels() != SP_OK) return nullptr;
  auto w = std::make_unique<LoopWorld>();
  w->n = ranks;
  const size_t nch = size_t(kComms) * ranks * ranks;
  if (cudaMalloc(&w->flags, nch * 2 * kSlots * sizeof(uint32_t)) != cudaSuccess) return nullptr;
  if (cudaMemset(w->flags, 0, nch * 2 * kSlots * sizeof(uint32_t)) != cudaSuccess) return nullptr;
  if (cudaHostAlloc(reinterpret_cast<void**>(&w->mail), nch * kSlots * sizeof(Mail),
                    cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
    return nullptr;
  if (cudaMalloc(&w->err, sizeof(int)) != cudaSuccess || cudaMemset(w->err, 0, sizeof(int)) != cudaSuccess)
    return nullptr;
  for (size_t x = 0; x < nch; ++x) {
    auto c = std::make_unique<Channel>();
    c->ready = w->flags + x * 2 * kSlots;
    c->done = c->ready + kSlots;
    c->mail = w->mail + x * kSlots;
    w->ch.push_back(std::move(c));
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return nullptr;
  return w.release();
}

void loop_world_destroy(LoopWorld* w) {
  if (!w) return;
  cudaDeviceSynchronize();
  cudaFree(w->flags);
  cudaFree(w->err);
  cudaFreeHost(w->mail);
  delete w;
}

int loop_world_size(const LoopWorld* w) { return w ? w->n : 0; }

int loop_world_errors(const LoopWorld* w) {
  int e = 0;
  if (w) cudaMemcpy(&e, w->err, sizeof e, cudaMemcpyDeviceToHost);
  return e;
}

namespace {

int dt_bytes(ncclDataType_t dt) {
  switch (dt) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

#define SP_LOOP_TRY(x)        \
  do {                        \
    if (int rc_ = (x)) return rc_; \
  } while (0)

class LoopLink final : public Link {
 public:
  LoopLink(LoopWorld* w, int id, std::vector<int> members, int me) : w_(w), id_(id), mem_(std::move(members)), me_(me) {}

  int send(const void* buf, int64_t count, ncclDataType_t dt, int peer, cudaStream_t st) override {
    if (grouping_) {
      ops_.push_back({true, buf, nullptr, count * dt_bytes(dt), peer, st});
      return SP_OK;
    }
    return do_send(buf, count * dt_bytes(dt), peer, st);
  }
  int recv(void* buf, int64_t count, ncclDataType_t dt, int peer, cudaStream_t st) override {
    if (grouping_) {
      ops_.push_back({false, nullptr, buf, count * dt_bytes(dt), peer, st});
      return SP_OK;
    }
    uint64_t seq = 0;
    if (int rc = post(buf, count * dt_bytes(dt), peer, st, &seq)) return rc;
    return wait_done(peer, seq, st);
  }
  int group_start() override {
    grouping_ = true;
    return SP_OK;
  }
  // Receives are posted first, then the sends run, then the receives wait:
  // a group never waits on its own later members.
  int group_end() override {
    grouping_ = false;
    std::vector<uint64_t> seqs(ops_.size());
    for (size_t x = 0; x < ops_.size(); ++x)
      if (!ops_[x].is_send)
        if (int rc = post(ops_[x].rbuf, ops_[x].bytes, ops_[x].peer, ops_[x].st, &seqs[x])) return clear(rc);
    for (const Op& o : ops_)
      if (o.is_send)
        if (int rc = do_send(o.sbuf, o.bytes, o.peer, o.st)) return clear(rc);
    for (size_t x = 0; x < ops_.size(); ++x)
      if (!ops_[x].is_send)
        if (int rc = wait_done(ops_[x].peer, seqs[x], ops_[x].st)) return clear(rc);
    return clear(SP_OK);
  }

 private:
  struct Op {
    bool is_send;
    const void* sbuf;
    void* rbuf;
    int64_t bytes;
    int peer;
    cudaStream_t st;
  };
  int clear(int rc) {
    ops_.clear();
    return rc;
  }
  Channel& chan(int src_local, int dst_local) { return w_->at(id_, mem_[size_t(src_local)], mem_[size_t(dst_local)]); }

  int post(void* buf, int64_t bytes, int peer, cudaStream_t st, uint64_t* seq_out) {
    Channel& c = chan(peer, me_);
    const uint64_t seq = c.rseq++;
    const int slot = int(seq % kSlots);
    c.mail[slot].dst = buf;
    c.mail[slot].bytes = bytes;
    *seq_out = seq;
    loop_signal_kernel<<<1, 32, 0, st>>>(c.ready + slot, uint32_t(seq + 1));
    count_launch();
    return cuda_status(cudaGetLastError(), "loopback post");
  }
  int wait_done(int peer, uint64_t seq, cudaStream_t st) {
    Channel& c = chan(peer, me_);
    loop_wait_kernel<<<1, 32, 0, st>>>(c.done + seq % kSlots, uint32_t(seq + 1));
    count_launch();
    return cuda_status(cudaGetLastError(), "loopback wait");
  }
  int do_send(const void* buf, int64_t bytes, int peer, cudaStream_t st) {
    Channel& c = chan(me_, peer);
    const uint64_t seq = c.sseq++;
    const int slot = int(seq % kSlots);
    const int blocks = int(std::min<int64_t>(296, (bytes / 16 + 255) / 256 + 1));
    loop_wait_kernel<<<1, 32, 0, st>>>(c.ready + slot, uint32_t(seq + 1));
    loop_copy_kernel<<<blocks, 256, 0, st>>>(c.mail + slot, static_cast<const uint8_t*>(buf), bytes, w_->err);
    count_launch(2);
    if (int rc = cuda_status(cudaGetLastError(), "loopback copy")) return rc;
    loop_signal_kernel<<<1, 32, 0, st>>>(c.done + slot, uint32_t(seq + 1));
    count_launch();
    return cuda_status(cudaGetLastError(), "loopback done");
  }

  LoopWorld* w_;
  int id_;
  std::vector<int> mem_;
  int me_;
  bool grouping_ = false;
  std::vector<Op> ops_;
  float* scratch_ = nullptr;  // collectives: peers' contributions at the root
  int64_t scratch_n_ = 0;

 public:
  ~LoopLink() override {
    if (scratch_) cudaFree(scratch_);
  }
  // Collectives over point-to-point messages (vocabulary parallelism on one
  // GPU): the root gathers every peer's buffer, combines, and (all-reduce /
  // broadcast) sends the result back.  Same arithmetic as a reduction tree
  // up to the fp32 summation order.
  int broadcast(void* buf, int64_t count, ncclDataType_t dt, int root, cudaStream_t st) override {
    const int n = int(mem_.size());
    if (me_ == root) {
      SP_LOOP_TRY(group_start());
      for (int q = 0; q < n; ++q)
        if (q != root) SP_LOOP_TRY(send(buf, count, dt, q, st));
      return group_end();
    }
    return recv(buf, count, dt, root, st);
  }
  int reduce(float* buf, int64_t count, int root, cudaStream_t st) override {
    return gather_combine(buf, count, 0, root, st, false);
  }
  int reserve(int64_t count) override {
    const int64_t need = int64_t(mem_.size() - 1) * count;
    if (need <= scratch_n_) return SP_OK;
    if (scratch_) cudaFree(scratch_);
    scratch_ = nullptr;
    scratch_n_ = 0;
    if (cudaError_t e = cudaMalloc(&scratch_, size_t(std::max<int64_t>(need, 1)) * 4))
      return cuda_status(e, "loopback collective scratch");
    scratch_n_ = need;
    return SP_OK;
  }
  int all_reduce(float* buf, int64_t count, ncclRedOp_t op, cudaStream_t st) override {
    if (op != ncclSum && op != ncclMax) return set_error(SP_ERR_UNSUPPORTED, "loopback all_reduce: sum or max only");
    return gather_combine(buf, count, op == ncclMax ? 1 : 0, 0, st, true);
  }

 private:
  int gather_combine(float* buf, int64_t count, int op, int root, cudaStream_t st, bool back) {
    const int n = int(mem_.size());
    if (me_ != root) {
      SP_LOOP_TRY(send(buf, count, ncclFloat32, root, st));
      return back ? recv(buf, count, ncclFloat32, root, st) : SP_OK;
    }
    if (int64_t(n - 1) * count > scratch_n_)
      return set_error(SP_ERR_RUNTIME, "loopback collective: scratch not reserved for %lld floats", (long long)count);
    SP_LOOP_TRY(group_start());
    for (int q = 0, x = 0; q < n; ++q)
      if (q != root) SP_LOOP_TRY(recv(scratch_ + int64_t(x++) * count, count, ncclFloat32, q, st));
    SP_LOOP_TRY(group_end());
    const int blocks = int(std::min<int64_t>(592, (count + 255) / 256 + 1));
    for (int x = 0; x < n - 1; ++x) {
      loop_combine_kernel<<<blocks, 256, 0, st>>>(buf, scratch_ + int64_t(x) * count, count, op);
      count_launch();
    }
    SP_LOOP_TRY(cuda_status(cudaGetLastError(), "loopback combine"));
    if (!back) return SP_OK;
    SP_LOOP_TRY(group_start());
    for (int q = 0; q < n; ++q)
      if (q != root) SP_LOOP_TRY(send(buf, count, ncclFloat32, q, st));
    return group_end();
  }
};

}  // namespace

std::unique_ptr<Link> make_nccl_link(ncclComm_t comm) { return std::make_unique<NcclLink>(comm); }

std::unique_ptr<Link> make_loop_link(LoopWorld* w, int comm_id, std::vector<int> members, int me) {
  if (!w || comm_id < 0 || comm_id >= kComms) return nullptr;
  for (int m : members)
    if (m < 0 || m >= w->n) return nullptr;
  return std::make_unique<LoopLink>(w, comm_id, std::move(members), me);
}

// Force-load this file's kernels (cudaFuncGetAttributes) — see preload_kernels
int preload_transport() {
  cudaFuncAttributes a;
  for (const void* k : {reinterpret_cast<const void*>(loop_signal_kernel), reinterpret_cast<const void*>(loop_wait_kernel),
                        reinterpret_cast<const void*>(loop_copy_kernel), reinterpret_cast<const void*>(loop_combine_kernel)})
    if (cudaError_t e = cudaFuncGetAttributes(&a, k)) return cuda_status(e, "preload transport");
  return SP_OK;
}

// CUDA lazy loading (the default) loads a kernel at its first launch, and a
// load may wait for the context to go idle.  A spinning receive (an NCCL
// kernel, or a loopback wait) is then a deadlock: it waits for a peer whose
// next kernel cannot load until the spinner ends.  The round-1 vocab-parallel
// and interleaved stalls had exactly this shape (the host blocked inside step
// enqueue at the first launch of a kernel type while a receive was posted).
// Every kernel of the library is therefore loaded up front, before any
// communication; library GEMMs are warmed by the runtime (warm_gemms).
int preload_kernels() {
  static std::mutex mu;
  static std::set<int> done;
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return cuda_status(e, "preload");
  std::lock_guard<std::mutex> g(mu);
  if (done.count(dev)) return SP_OK;
  for (int (*f)() : {preload_layers, preload_attn_fwd, preload_attn_fwd_v4, preload_attn_bwd, preload_attn_bwd_v2,
                     preload_attn_merge, preload_transport})
    if (int rc = f()) return rc;
  done.insert(dev);
  return SP_OK;
}

}  // namespace sp

extern "C" {

int sp_loopback_create(int ranks, void** world) {
  sp::LoopWorld* w = sp::loop_world_create(ranks);
  if (!w)
    return sp::set_error(SP_ERR_CUDA, "loopback world: stream memory operations or allocation unavailable");
  *world = w;
  return SP_OK;
}

int sp_loopback_destroy(void* world) {
  sp::loop_world_destroy(static_cast<sp::LoopWorld*>(world));
  return SP_OK;
}

int sp_loopback_errors(void* world) { return sp::loop_world_errors(static_cast<sp::LoopWorld*>(world)); }

// Both ranks of the self-test enqueued from ONE host thread (rank 0's
// operations, then rank 1's — enqueue never blocks), then both streams
// synchronised: isolates the device protocol from host threading.
int sp_loopback_pingpong_1thread(void* world, void* buf0, void* buf1, void* rbuf0, void* rbuf1, int64_t bytes,
                                 int iters) {
  auto* w = static_cast<sp::LoopWorld*>(world);
  auto l0 = sp::make_loop_link(w, 6, {0, 1}, 0), l1 = sp::make_loop_link(w, 6, {0, 1}, 1);
  if (!l0 || !l1) return sp::set_error(SP_ERR_INVALID, "pingpong: bad world");
  cudaStream_t s0, s1;
  cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  int rc = SP_OK;
  for (int i = 0; i < iters && rc == SP_OK; ++i) {
    rc = l0->send(buf0, bytes, ncclUint8, 1, s0);
    if (!rc) rc = l0->recv(rbuf0, bytes, ncclUint8, 1, s0);
  }
  for (int i = 0; i < iters && rc == SP_OK; ++i) {
    rc = l1->recv(rbuf1, bytes, ncclUint8, 0, s1);
    if (!rc) rc = l1->send(buf1, bytes, ncclUint8, 0, s1);
  }
  if (!rc) rc = sp::cuda_status(cudaStreamSynchronize(s0), "pingpong sync 0");
  if (!rc) rc = sp::cuda_status(cudaStreamSynchronize(s1), "pingpong sync 1");
  cudaStreamDestroy(s0);
  cudaStreamDestroy(s1);
  return rc;
}

// Transport self-test (tests/test_loopback_gpu.py): rank `rank` of a 2-rank
// world exchanges `iters` messages of `bytes` with rank 1-rank on its own
// stream — rank 0 sends then receives, rank 1 receives then sends, plus one
// grouped send+recv per iteration — and returns when its stream is done.
int sp_loopback_pingpong(void* world, int rank, void* send_buf, void* recv_buf, int64_t bytes, int iters) {
  auto* w = static_cast<sp::LoopWorld*>(world);
  auto link = sp::make_loop_link(w, 7, {0, 1}, rank);
  if (!link) return sp::set_error(SP_ERR_INVALID, "pingpong: bad world/rank");
  cudaStream_t st;
  if (cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) return sp::cuda_status(e, "pingpong stream");
  const int peer = 1 - rank;
  int rc = SP_OK;
  for (int i = 0; i < iters && rc == SP_OK; ++i) {
    if (rank == 0) {
      rc = link->send(send_buf, bytes, ncclUint8, peer, st);
      if (!rc) rc = link->recv(recv_buf, bytes, ncclUint8, peer, st);
    } else {
      rc = link->recv(recv_buf, bytes, ncclUint8, peer, st);
      if (!rc) rc = link->send(send_buf, bytes, ncclUint8, peer, st);
    }
    if (!rc) rc = link->group_start();
    if (!rc) rc = link->send(send_buf, bytes, ncclUint8, peer, st);
    if (!rc) rc = link->recv(recv_buf, bytes, ncclUint8, peer, st);
    if (!rc) rc = link->group_end();
  }
  if (!rc) rc = sp::cuda_status(cudaStreamSynchronize(st), "pingpong sync");
  cudaStreamDestroy(st);
  return rc;
}

}  // extern "C"
