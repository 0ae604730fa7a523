// TEST INFRASTRUCTURE: an NCCL-compatible stand-in that runs N ranks as N threads of one process
// on ONE GPU, so the library's multi-rank device path (halo pack, grouped send/recv into the halo
// buffer, halo-aware SpMV, allreduces) can be exercised where only one GPU exists (NCCL itself
// refuses two ranks on one device).  Loaded by the library through TE_NCCL_LIB.
//
// Semantics (stream-ordered, like NCCL): every call is a rendezvous of all ranks of the
// communicator; each rank records a "ready" event on its stream before arriving; the last thread
// to arrive enqueues all copies / reductions on rank 0's stream after waiting for every ready
// event, records a "done" event, and makes every rank's stream wait on it.  Reductions sum in rank
// order 0..N-1.  Send/Recv (grouped or not) are matched pairwise: the k-th Recv at d from s with
// the k-th Send from s to d; a rank posts all operations of its group, the second party of each
// pair enqueues the copy on the receiver's stream (after the sender's ready event) and makes the
// sender's stream wait for it; a rank returns from ncclGroupEnd once all its operations matched.
// Supported: ncclGetUniqueId, ncclCommInitRank, ncclCommDestroy, ncclAllReduce (double; sum/max),
// ncclAllGather, ncclSend/ncclRecv inside ncclGroupStart/End, ncclGetErrorString.
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

struct P2P {
  bool send;
  const void* sbuf;
  void* rbuf;
  size_t bytes;
  int peer;
};

struct Arrival {
  int kind = 0;  // 1 allreduce, 2 allgather
  const void* send = nullptr;
  void* recv = nullptr;
  size_t count = 0;
  ncclDataType_t type = ncclDouble;
  ncclRedOp_t op = ncclSum;
  cudaStream_t stream = nullptr;
};

struct Shared {
  int nranks = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<Arrival> slots;
  std::vector<cudaEvent_t> ready;
  cudaEvent_t done = nullptr;
  double* tmp = nullptr;
  size_t tmp_cap = 0;
  std::string error;
};

struct ncclComm {
  int rank = 0;
  Shared* sh = nullptr;
};

static std::mutex g_mu;
static std::map<std::string, Shared*> g_comms;
static std::atomic<long> g_calls{0};
static thread_local int t_group_depth = 0;
static thread_local std::vector<P2P> t_group_ops;
static thread_local ncclComm* t_group_comm = nullptr;
static thread_local cudaStream_t t_group_stream = nullptr;

extern "C" long fake_nccl_calls() { return g_calls.load(); }
static bool dbg() {
  static int d = getenv("FAKE_NCCL_DEBUG") ? 1 : 0;
  return d != 0;
}

static size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

struct Ptrs {
  const double* p[8];
};
__global__ void k_reduce(Ptrs src, int nsrc, double* dst, size_t count, int is_max) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double a = src.p[0][i];
    for (int r = 1; r < nsrc; ++r) a = is_max ? fmax(a, src.p[r][i]) : a + src.p[r][i];
    dst[i] = a;
  }
}

// executed by the last arriving thread, with the lock held
static void execute(Shared* sh) {
  const int N = sh->nranks;
  cudaStream_t s0 = sh->slots[0].stream;
  for (int r = 0; r < N; ++r) cudaStreamWaitEvent(s0, sh->ready[r], 0);
  const Arrival& a0 = sh->slots[0];
  if (a0.kind == 1) {
    if (a0.type != ncclDouble || N > 8) {
      sh->error = "fake_nccl: allreduce supports double, <= 8 ranks";
    } else {
      if (sh->tmp_cap < a0.count) {
        cudaFree(sh->tmp);
        cudaMalloc(&sh->tmp, sizeof(double) * a0.count);
        sh->tmp_cap = a0.count;
      }
      Ptrs p{};
      for (int r = 0; r < N; ++r) p.p[r] = static_cast<const double*>(sh->slots[r].send);
      const int grid = (int)((a0.count + 255) / 256) + 1;
      k_reduce<<<grid, 256, 0, s0>>>(p, N, sh->tmp, a0.count, a0.op == ncclMax);
      for (int r = 0; r < N; ++r)
        cudaMemcpyAsync(sh->slots[r].recv, sh->tmp, sizeof(double) * a0.count, cudaMemcpyDeviceToDevice, s0);
    }
  } else if (a0.kind == 2) {
    const size_t b = a0.count * type_size(a0.type);
    for (int dst = 0; dst < N; ++dst)
      for (int src = 0; src < N; ++src)
        cudaMemcpyAsync(static_cast<char*>(sh->slots[dst].recv) + (size_t)src * b, sh->slots[src].send, b,
                        cudaMemcpyDeviceToDevice, s0);
  }
  cudaEventRecord(sh->done, s0);
  for (int r = 0; r < N; ++r) cudaStreamWaitEvent(sh->slots[r].stream, sh->done, 0);
}

static ncclResult_t arrive(ncclComm* c, Arrival&& a) {
  g_calls++;
  if (dbg()) fprintf(stderr, "[fake_nccl] rank %d collective kind %d count %zu\n", c->rank, a.kind, a.count);
  Shared* sh = c->sh;
  cudaEventRecord(sh->ready[c->rank], a.stream);
  std::unique_lock<std::mutex> lk(sh->mu);
  sh->slots[c->rank] = std::move(a);
  const uint64_t gen = sh->gen;
  if (++sh->arrived == sh->nranks) {
    for (int r = 1; r < sh->nranks; ++r)
      if (sh->slots[r].kind != sh->slots[0].kind) sh->error = "fake_nccl: ranks called different collectives";
    if (sh->error.empty()) execute(sh);
    sh->arrived = 0;
    sh->gen++;
    sh->cv.notify_all();
  } else {
    sh->cv.wait(lk, [&] { return sh->gen != gen; });
  }
  return sh->error.empty() ? ncclSuccess : ncclInternalError;
}

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  static std::atomic<unsigned> ctr{0};
  std::memset(id, 0, sizeof(*id));
  std::snprintf(id->internal, sizeof(id->internal), "fake-nccl-%u", ctr.fetch_add(1));
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  Shared* sh;
  {
    std::lock_guard<std::mutex> g(g_mu);
    std::string key(id.internal, strnlen(id.internal, sizeof(id.internal)));
    auto it = g_comms.find(key);
    if (it == g_comms.end()) {
      sh = new Shared;
      sh->nranks = nranks;
      sh->slots.resize(nranks);
      sh->ready.resize(nranks);
      for (auto& e : sh->ready) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&sh->done, cudaEventDisableTiming);
      g_comms[key] = sh;
    } else {
      sh = it->second;
    }
  }
  if (sh->nranks != nranks) return ncclInvalidArgument;
  auto* c = new ncclComm;
  c->rank = rank;
  c->sh = sh;
  *comm = c;
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  delete comm;  // the shared state is kept for the process lifetime (test helper)
  return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t type, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t stream) {
  Arrival a;
  a.kind = 1; a.send = send; a.recv = recv; a.count = count; a.type = type; a.op = op; a.stream = stream;
  return arrive(comm, std::move(a));
}

ncclResult_t ncclAllGather(const void* send, void* recv, size_t count, ncclDataType_t type, ncclComm_t comm,
                           cudaStream_t stream) {
  Arrival a;
  a.kind = 2; a.send = send; a.recv = recv; a.count = count; a.type = type; a.stream = stream;
  return arrive(comm, std::move(a));
}

ncclResult_t ncclGroupStart() {
  if (t_group_depth++ == 0) {
    t_group_ops.clear();
    t_group_comm = nullptr;
    t_group_stream = nullptr;
  }
  return ncclSuccess;
}

struct Posted {
  bool send;
  int src, dst;
  long seq;
  const void* sbuf;
  void* rbuf;
  size_t bytes;
  cudaStream_t stream;
  cudaEvent_t ready;
  bool* matched;
};
struct P2PState {
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::pair<int, int>, long> send_seq, recv_seq;
  std::vector<Posted> pending;
};
static std::map<Shared*, P2PState*> g_p2p;

static void do_copy(const Posted& snd, const Posted& rcv) {
  cudaStreamWaitEvent(rcv.stream, snd.ready, 0);
  if (rcv.bytes) cudaMemcpyAsync(rcv.rbuf, snd.sbuf, rcv.bytes, cudaMemcpyDeviceToDevice, rcv.stream);
  cudaEvent_t fin;
  cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
  cudaEventRecord(fin, rcv.stream);
  cudaStreamWaitEvent(snd.stream, fin, 0);
  cudaEventDestroy(fin);
  cudaEventDestroy(snd.ready);
}

static ncclResult_t p2p(bool send, const void* sb, void* rb, size_t count, ncclDataType_t type, int peer,
                        ncclComm_t comm, cudaStream_t stream) {
  const bool implicit = t_group_depth == 0;
  if (implicit) ncclGroupStart();
  t_group_ops.push_back(P2P{send, sb, rb, count * type_size(type), peer});
  t_group_comm = comm;
  t_group_stream = stream;
  return implicit ? ncclGroupEnd() : ncclSuccess;
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t type, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
  return p2p(true, buf, nullptr, count, type, peer, comm, stream);
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t type, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
  return p2p(false, nullptr, buf, count, type, peer, comm, stream);
}

ncclResult_t ncclGroupEnd() {
  if (--t_group_depth > 0) return ncclSuccess;
  if (!t_group_comm) return ncclSuccess;  // no operations posted by this rank
  g_calls++;
  ncclComm* c = t_group_comm;
  if (dbg()) fprintf(stderr, "[fake_nccl] rank %d group of %zu p2p ops\n", c->rank, t_group_ops.size());
  P2PState* ps;
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_p2p.find(c->sh);
    if (it == g_p2p.end()) it = g_p2p.emplace(c->sh, new P2PState).first;
    ps = it->second;
  }
  std::vector<char> flags(t_group_ops.size(), 0);
  std::unique_lock<std::mutex> lk(ps->mu);
  bool bad = false;
  for (size_t i = 0; i < t_group_ops.size(); ++i) {
    const P2P& op = t_group_ops[i];
    Posted me{};
    me.send = op.send;
    me.src = op.send ? c->rank : op.peer;
    me.dst = op.send ? op.peer : c->rank;
    me.seq = op.send ? ps->send_seq[{me.src, me.dst}]++ : ps->recv_seq[{me.src, me.dst}]++;
    me.sbuf = op.sbuf;
    me.rbuf = op.rbuf;
    me.bytes = op.bytes;
    me.stream = t_group_stream;
    me.matched = reinterpret_cast<bool*>(&flags[i]);
    if (me.send) {
      cudaEventCreateWithFlags(&me.ready, cudaEventDisableTiming);
      cudaEventRecord(me.ready, me.stream);
    }
    auto pit = ps->pending.begin();
    for (; pit != ps->pending.end(); ++pit)
      if (pit->send != me.send && pit->src == me.src && pit->dst == me.dst && pit->seq == me.seq) break;
    if (pit != ps->pending.end()) {
      const Posted& other = *pit;
      if (other.bytes != me.bytes) bad = true;
      if (me.send) do_copy(me, other); else do_copy(other, me);
      *other.matched = true;
      *me.matched = true;
      ps->pending.erase(pit);
      ps->cv.notify_all();
    } else {
      ps->pending.push_back(me);
    }
  }
  ps->cv.wait(lk, [&] {
    for (char f : flags)
      if (!f) return false;
    return true;
  });
  return bad ? ncclInternalError : ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) {
  return r == ncclSuccess ? "success (fake_nccl)" : "fake_nccl error";
}

}  // extern "C"
