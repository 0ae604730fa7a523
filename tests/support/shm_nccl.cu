// TEST INFRASTRUCTURE: an NCCL-compatible stand-in for several PROCESSES on one GPU (NCCL itself
// refuses two ranks on one device), so the library's cross-process paths run for real: the halo
// plan exchange, the allreduces and, above all, halo mode 1, where each process maps the other
// processes' Krylov bases through CUDA IPC (cudaIpcGetMemHandle / cudaIpcOpenMemHandle) and its
// SpMV reads their V columns directly.  Loaded by the library through TE_NCCL_LIB.
//
// Every call is host-staged and blocking: the caller's stream is synchronised, the payload goes
// through a POSIX shared-memory segment (named by TE_SHM_NAME, which ncclGetUniqueId returns),
// and a process-shared barrier orders the ranks; reductions sum in rank order 0..P-1
// (deterministic).  Send/Recv are executed at ncclGroupEnd, pairwise (a rank with no exchange
// does not take part, as with NCCL): each send waits for its (src, dst) mailbox to be empty,
// deposits the payload and raises the mailbox flag; then each receive waits for the flag, takes
// the payload and clears it.
// Supported: ncclGetUniqueId, ncclCommInitRank, ncclCommDestroy, ncclAllReduce (double; sum/max),
// ncclAllGather, ncclSend/ncclRecv inside ncclGroupStart/End, ncclGetErrorString.  The symbol
// fake_nccl_calls marks it as a stand-in (the library then does not capture NCCL into graphs).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace {
constexpr size_t kSlot = 1u << 20;  // per-rank collective slot and per-(src,dst) mailbox (20 MB segment)
constexpr int kMaxRanks = 4;

struct Header {
  std::atomic<int> count;
  std::atomic<int> gen;
  std::atomic<int> attached;
  std::atomic<int> full[kMaxRanks * kMaxRanks];  // mailbox (src, dst) holds an undelivered message
};

size_t seg_bytes() { return 4096 + (size_t)kMaxRanks * kSlot + (size_t)kMaxRanks * kMaxRanks * kSlot; }

struct P2P {
  bool send;
  const void* sbuf;
  void* rbuf;
  size_t bytes;
  int peer;
  cudaStream_t stream;
};

thread_local int t_depth = 0;
thread_local std::vector<P2P> t_ops;
thread_local ncclComm* t_comm = nullptr;
long g_calls = 0;

size_t tsize(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclFloat16: case ncclBfloat16: return 2;
    default: return 8;
  }
}
}  // namespace

struct ncclComm {
  int rank = 0, nranks = 1;
  unsigned char* base = nullptr;
  std::string name;
  Header* hdr() { return reinterpret_cast<Header*>(base); }
  unsigned char* slot(int r) { return base + 4096 + (size_t)r * kSlot; }
  unsigned char* box(int src, int dst) { return base + 4096 + (size_t)kMaxRanks * kSlot + ((size_t)src * kMaxRanks + dst) * kSlot; }
  void barrier() {
    Header* h = hdr();
    const int g = h->gen.load(std::memory_order_acquire);
    if (h->count.fetch_add(1, std::memory_order_acq_rel) == nranks - 1) {
      h->count.store(0, std::memory_order_relaxed);
      h->gen.store(g + 1, std::memory_order_release);
    } else {
      while (h->gen.load(std::memory_order_acquire) == g) usleep(20);
    }
  }
};

extern "C" {

long fake_nccl_calls() { return g_calls; }

const char* ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "success" : "shm_nccl error"; }

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  std::memset(id, 0, sizeof *id);
  const char* n = getenv("TE_SHM_NAME");
  if (!n) return ncclInvalidUsage;
  std::strncpy(reinterpret_cast<char*>(id->internal), n, sizeof(id->internal) - 1);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  if (nranks > kMaxRanks || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  auto* c = new ncclComm();
  c->rank = rank;
  c->nranks = nranks;
  c->name = std::string(reinterpret_cast<const char*>(id.internal));
  const int fd = shm_open(c->name.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0) return ncclSystemError;
  if (ftruncate(fd, (off_t)seg_bytes()) != 0) { close(fd); return ncclSystemError; }
  void* p = mmap(nullptr, seg_bytes(), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return ncclSystemError;
  c->base = static_cast<unsigned char*>(p);  // a fresh segment is zero-filled: counters start at 0
  c->hdr()->attached.fetch_add(1);
  while (c->hdr()->attached.load() < nranks) usleep(100);
  *comm = c;
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t c) {
  if (!c) return ncclSuccess;
  c->barrier();
  const bool last = c->hdr()->attached.fetch_sub(1) == 1;
  munmap(c->base, seg_bytes());
  if (last) shm_unlink(c->name.c_str());
  delete c;
  return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* s, void* r, size_t count, ncclDataType_t t, ncclRedOp_t op, ncclComm_t c,
                           cudaStream_t st) {
  ++g_calls;
  if (t != ncclDouble || (op != ncclSum && op != ncclMax)) return ncclInvalidArgument;
  const size_t bytes = count * 8;
  if (bytes > kSlot) return ncclInvalidArgument;
  if (cudaStreamSynchronize(st) != cudaSuccess) return ncclUnhandledCudaError;
  if (cudaMemcpy(c->slot(c->rank), s, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return ncclUnhandledCudaError;
  c->barrier();
  std::vector<double> acc(count);
  std::memcpy(acc.data(), c->slot(0), bytes);
  for (int q = 1; q < c->nranks; ++q) {
    const double* v = reinterpret_cast<const double*>(c->slot(q));
    for (size_t i = 0; i < count; ++i) acc[i] = op == ncclSum ? acc[i] + v[i] : (v[i] > acc[i] ? v[i] : acc[i]);
  }
  c->barrier();
  if (cudaMemcpyAsync(r, acc.data(), bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) return ncclUnhandledCudaError;
  if (cudaStreamSynchronize(st) != cudaSuccess) return ncclUnhandledCudaError;
  return ncclSuccess;
}

ncclResult_t ncclAllGather(const void* s, void* r, size_t count, ncclDataType_t t, ncclComm_t c, cudaStream_t st) {
  ++g_calls;
  const size_t bytes = count * tsize(t);
  if (bytes > kSlot) return ncclInvalidArgument;
  if (cudaStreamSynchronize(st) != cudaSuccess) return ncclUnhandledCudaError;
  if (cudaMemcpy(c->slot(c->rank), s, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return ncclUnhandledCudaError;
  c->barrier();
  std::vector<unsigned char> all(bytes * c->nranks);
  for (int q = 0; q < c->nranks; ++q) std::memcpy(all.data() + q * bytes, c->slot(q), bytes);
  c->barrier();
  if (cudaMemcpyAsync(r, all.data(), all.size(), cudaMemcpyHostToDevice, st) != cudaSuccess) return ncclUnhandledCudaError;
  if (cudaStreamSynchronize(st) != cudaSuccess) return ncclUnhandledCudaError;
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
  ++t_depth;
  return ncclSuccess;
}

ncclResult_t ncclSend(const void* s, size_t count, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t st) {
  ++g_calls;
  if (t_depth == 0) return ncclInvalidUsage;  // the library groups every send/recv
  t_comm = c;
  t_ops.push_back({true, s, nullptr, count * tsize(t), peer, st});
  return ncclSuccess;
}

ncclResult_t ncclRecv(void* r, size_t count, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t st) {
  ++g_calls;
  if (t_depth == 0) return ncclInvalidUsage;
  t_comm = c;
  t_ops.push_back({false, nullptr, r, count * tsize(t), peer, st});
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (--t_depth > 0) return ncclSuccess;
  ncclComm* c = t_comm;
  std::vector<P2P> ops;
  ops.swap(t_ops);
  t_comm = nullptr;
  if (!c) return ncclSuccess;  // nothing to exchange: no part in anyone else's transfers
  Header* h = c->hdr();
  for (const P2P& o : ops) {
    if (!o.send) continue;
    if (o.bytes > kSlot) return ncclInvalidArgument;
    std::atomic<int>& f = h->full[c->rank * kMaxRanks + o.peer];
    while (f.load(std::memory_order_acquire) != 0) usleep(20);
    if (cudaStreamSynchronize(o.stream) != cudaSuccess) return ncclUnhandledCudaError;
    if (cudaMemcpy(c->box(c->rank, o.peer), o.sbuf, o.bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
      return ncclUnhandledCudaError;
    f.store(1, std::memory_order_release);
  }
  for (const P2P& o : ops) {
    if (o.send) continue;
    std::atomic<int>& f = h->full[o.peer * kMaxRanks + c->rank];
    while (f.load(std::memory_order_acquire) == 0) usleep(20);
    if (cudaStreamSynchronize(o.stream) != cudaSuccess) return ncclUnhandledCudaError;
    if (cudaMemcpyAsync(o.rbuf, c->box(o.peer, c->rank), o.bytes, cudaMemcpyHostToDevice, o.stream) != cudaSuccess)
      return ncclUnhandledCudaError;
    if (cudaStreamSynchronize(o.stream) != cudaSuccess) return ncclUnhandledCudaError;
    f.store(0, std::memory_order_release);
  }
  return ncclSuccess;
}

}  // extern "C"
