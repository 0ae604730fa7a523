// C ABI (include/te.h) and the host restart loop of Algorithm 1.
// The large-space work of every step runs in the kernels of kernels.cu; the host only does
// the m x m problem (host_math.cpp) once per restart, as the paper prescribes.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <unistd.h>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/te.h"
#include "host_math.h"
#include "kernels.cuh"
#include "nccl_shim.h"

#include <chrono>
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a profiler is attached

namespace {
// NVTX range for the lifetime of a scope (te_evolve, each restart's Krylov decomposition, the
// host step search, V.omega): nsys/ncu timelines show the algorithm's phases
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};
}  // namespace

using te::KDev;
using te::Launch;

// ------------------------------------------------------------------------------------------
// status
// ------------------------------------------------------------------------------------------
static thread_local int g_status = TE_OK;
static thread_local std::string g_msg;

static int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_status = code;
  g_msg = buf;
  return code;
}
static void clear_err() {
  g_status = TE_OK;
  g_msg.clear();
  // the runtime's last-error slot is per thread and shared with every other CUDA user in it
  // (e.g. torch): drop anything left there so only this call's own failures are reported
  (void)cudaGetLastError();
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return set_err(e_ == cudaErrorMemoryAllocation ? TE_ERR_OOM : TE_ERR_CUDA, "%s: %s (%s:%d)", #call, \
                     cudaGetErrorString(e_), __FILE__, __LINE__);                             \
  } while (0)

#define CKN(call)                                                                             \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess)                                                                    \
      return set_err(TE_ERR_NCCL, "%s: %s", #call, te::nccl().GetErrorString(r_));            \
  } while (0)

// ------------------------------------------------------------------------------------------
// handle
// ------------------------------------------------------------------------------------------
struct te_dist {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
};

namespace {
constexpr int kProfKernels = 7;  // 0 spmv(_proj) 1 update_proj 2 update_norm 3 combine 4 halo 5 proj_dots 6 host
constexpr int kEvPool = 4 * te::kMaxCols + 16;
struct Sched {
  double tau;
  int32_t m_eff;
  double err;
};
}  // namespace

struct te_handle {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int64_t n = 0, n_global = 0, row_begin = 0;
  bool cplx = false;
  int64_t nnz = 0;
  int64_t* d_rowptr = nullptr;
  int32_t* d_col = nullptr;
  void* d_val = nullptr;
  double norm1 = 0.0;
  // workspace
  int m_cap = 0;
  int64_t ldv = 0;
  double2* d_V = nullptr;
  double2* d_W = nullptr;
  double* d_small = nullptr;  // alpha[64] beta[64] | flag (2 ints) | s[65] nrm2[64] scalar
  double2* d_g = nullptr;     // [0] reduction slot (||p''_{j-1}||^2) | g1[64] | g2[64] | coef[64]
  double2* d_G = nullptr;     // Gram matrix 64 x 64 (f2)
  double2* d_part = nullptr;
  double* d_partn = nullptr;
  unsigned* d_counter = nullptr;
  int max_grid = 0;
  double* h_small = nullptr;  // pinned: alpha beta flag + scalar
  double2* h_coef = nullptr;  // pinned: omega~
  // profiling / bookkeeping
  bool profile = false;
  int variant = 2;
  int ortho = 0;  // 0 CGS2 (default), 1 paper-literal 3-term Lanczos (f1)
  int integrator = 0;  // 0 adaptive tanh-sinh (default), 1 Gauss-Legendre
  int spmv_nf_wide = 0;
  int spmv_force_halo = 0;
  int spmv_tiled = 7;
  int64_t* d_tile_ring = nullptr;
  int64_t ntiles_ring = 0;
  int spmv_ring_tpr = 1;
  int ring_stages = 4;
  // staged-x ring SpMV (variant 8): tiles + plan, built at create (kept when it is the default)
  // or on first selection
  int64_t* d_tile_xs = nullptr;
  int64_t ntiles_xs = 0;
  int4* d_xs_meta = nullptr;
  int2* d_xs_rng = nullptr;
  uint16_t* d_lcol = nullptr;
  int spmv_xs_tpr = 1, xs_ecap = 0, xs_xcap = 0, xs_stages = 2, xs_xpol = 0, xs_nf = 8;
  double xs_global_frac = 1.0;  // entries the plan left to global gathers / nnz
  double xs_global_tiles = 1.0; // tiles with at least one such entry / tiles
  double xs_x_per_entry = 0.0;  // staged x slots / entries (bulk-copied x per product)
  // slot-window SELL-32 with a value dictionary (variant 9), built at create when applicable
  int64_t* d_sw_sptr = nullptr;
  int32_t* d_sw_base = nullptr;
  uint16_t* d_sw_ent = nullptr;
  void* d_sw_diag = nullptr;
  void* d_sw_dict = nullptr;
  int64_t sw_nslice = 0, sw_slots = 0;
  int sw_ndict = 0;
  int sw_bits = 16;
  // panel sweep (x larger than L2): the far windows live in a second set of arrays (pass 2)
  int64_t* d_swb_sptr = nullptr;
  int32_t* d_swb_base = nullptr;
  uint16_t* d_swb_ent = nullptr;
  int64_t swb_slots = 0;
  int sw_ka = 0, sw_sb = 0, sw_lo = 0, sw_ob = 0;  // panel slice bits (0: single pass), slice bits, outer range
  double sw_fill = 0.0;  // slot entries (32 per slot) / off-diagonal entries
  // column-blocked copy of H for the ring (variant 10): one CSR + ring tile table per cb_cols
  // columns of x, built at create for large x (single rank)
  struct ColBlk {
    int64_t* rowptr = nullptr;
    int32_t* col = nullptr;
    void* val = nullptr;
    int64_t* tiles = nullptr;
    int64_t ntiles = 0;
    int tpr = 1;
  };
  std::vector<ColBlk> cb;
  int64_t cb_cols = 0;
  int64_t ncol_limit = 0;
  // SELL-32-sigma copy of H (SpMV variant 6), built on first selection
  int32_t* d_scol = nullptr;
  void* d_sval = nullptr;
  int64_t* d_sptr = nullptr;
  int32_t* d_slen = nullptr;
  int32_t* d_sperm = nullptr;
  int64_t nslices = 0;
  std::vector<CUtensorMap> tmaps;
  int prefetch = 0;
  int norm_tma = 0;      // K3 above 8 columns on the TMA ring (default from 2^22 rows; TE_NORM_TMA read at create)
  int proj_const_r = 1;  // TE_PROJ_CONST_R=0 (read at create): the runtime-R build of the TMA projection kernels
  cudaEvent_t ev0[kEvPool], ev1[kEvPool];
  int ev_cls[kEvPool];
  double ev_bytes[kEvPool];
  int ev_used = 0;
  bool ev_ready = false;
  cudaEvent_t evk0 = nullptr, evk1 = nullptr;  // V.omega (outside the per-restart graph)
  bool evk_pending = false;
  double evk_bytes = 0.0;
  te_kernel_profile prof[kProfKernels];
  int64_t launches = 0;
  std::vector<Sched> sched;
  // CUDA graph of one restart's launches (replayed every restart)
  bool use_graph = true;
  bool capturing = false;
  cudaGraphExec_t gexec = nullptr;
  int g_m = -1, g_variant = -1, g_spmv = -1, g_ortho = -1, g_prefetch = -1, g_halo = -1;
  bool g_profile = false;
  double g_tol_rate = -1.0;
  const void* g_V = nullptr;
  int64_t g_launches = 0;
  int g_nev = 0;
  int g_ev_cls[kEvPool];
  double g_ev_bytes[kEvPool];
  // distributed
  te_dist* dist = nullptr;
  int64_t n_halo = 0;
  double2* d_halo = nullptr;
  // halo entries of the local rows (k_spmv_halo) and the side stream of the halo exchange
  int32_t* d_hrow = nullptr;
  int64_t* d_hrowptr = nullptr;
  int32_t* d_hcol = nullptr;
  void* d_hval = nullptr;
  int64_t nh = 0, nh_entries = 0;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int comm_sms = 8;  // SMs the SpMV leaves free for the concurrent NCCL exchange (TE_COMM_SMS)
  double2* d_sendbuf = nullptr;
  int32_t* d_send_idx = nullptr;
  // halo mode 1 (TE_OPT_HALO): halo columns read from peer memory inside the SpMV
  int halo_mode = 0;
  int32_t* d_halo_owner = nullptr;
  int32_t* d_halo_lidx = nullptr;
  const double2** d_peer_base = nullptr;
  int64_t* d_peer_ldv = nullptr;
  std::vector<void*> ipc_open;          // peer V mappings opened through CUDA IPC (closed on reset)
  const double2* peer_for_V = nullptr;  // the V allocation the peer table describes
  std::vector<int64_t> send_counts, recv_counts;
  int64_t n_send = 0;
};

extern "C" {
static int build_sell(te_handle* h);
}

namespace {

// device layout of d_small (doubles)
constexpr int kOffAlpha = 0, kOffBeta = 64, kOffFlag = 128, kOffS = 130, kOffNrm = 196, kOffScalar = 260,
              kSmallLen = 264;
// layout of d_g (double2): the reduction slot, g1, g2, the V.omega coefficients
constexpr int kOffG1 = 1, kOffG2 = 65, kOffCoef = 129, kGLen = 193;

KDev make_kdev(te_handle* h, double tol_rate, int m) {
  KDev d{};
  d.n = h->n;
  d.ldv = h->ldv;
  d.V = h->d_V;
  d.W = h->d_W;
  d.rowptr = h->d_rowptr;
  d.col = h->d_col;
  d.val = h->d_val;
  d.halo = h->d_halo;
  d.hrow = h->d_hrow;
  d.hrowptr = h->d_hrowptr;
  d.hcol = h->d_hcol;
  d.hval = h->d_hval;
  d.nh = h->nh;
  d.peer_base = h->d_peer_base;
  d.peer_ldv = h->d_peer_ldv;
  d.halo_owner = h->d_halo_owner;
  d.halo_lidx = h->d_halo_lidx;
  d.tile_ring = h->d_tile_ring;
  d.ntiles_ring = h->ntiles_ring;
  d.tile_xs = h->d_tile_xs;
  d.ntiles_xs = h->ntiles_xs;
  d.xs_meta = h->d_xs_meta;
  d.xs_rng = h->d_xs_rng;
  d.lcol = h->d_lcol;
  d.xs_ecap = h->xs_ecap;
  d.xs_xcap = h->xs_xcap;
  d.xs_rmax = te::kXsRmax;
  d.xs_xpol = h->xs_xpol;
  d.sw_sptr = h->d_sw_sptr;
  d.sw_base = h->d_sw_base;
  d.sw_ent = h->d_sw_ent;
  d.sw_diag = h->d_sw_diag;
  d.sw_dict = h->d_sw_dict;
  d.sw_nslice = h->sw_nslice;
  d.sw_ndict = h->sw_ndict;
  d.sw_bits = h->sw_bits;
  d.sw_pass = 0;
  d.sw_sb = h->sw_sb;
  d.sw_lo = h->sw_lo;
  d.sw_ob = h->sw_ob;
  d.scol = h->d_scol;
  d.sval = h->d_sval;
  d.sptr = h->d_sptr;
  d.slen = h->d_slen;
  d.sperm = h->d_sperm;
  d.nslices = h->nslices;
  d.alpha = h->d_small + kOffAlpha;
  d.beta = h->d_small + kOffBeta;
  d.flag = reinterpret_cast<int*>(h->d_small + kOffFlag);
  d.s = h->d_small + kOffS;
  d.nrm2 = h->d_small + kOffNrm;
  d.gsync = h->d_g;
  d.g1 = h->d_g + kOffG1;
  d.g2 = h->d_g + kOffG2;
  d.defer = h->ortho != 1;
  d.part = h->d_part;
  d.partn = h->d_partn;
  d.counter = h->d_counter;
  d.tol_rate = tol_rate;
  d.m = m;
  d.ortho = h->ortho;
  d.G = h->d_G;
  return d;
}

// halo mode 1: k_spmv_halo reads the halo entries from the owning ranks' V columns (any SpMV variant)
bool peer_active(const te_handle* h) { return h->dist && h->dist->nranks > 1 && h->halo_mode == 1; }
// the NCCL halo exchange runs on the side stream concurrently with the local-column SpMV
bool exchange_active(const te_handle* h) {
  return h->dist && h->dist->nranks > 1 && !peer_active(h) && (h->n_send > 0 || h->n_halo > 0);
}

Launch make_launch(te_handle* h) {
  Launch L;
  L.stream = h->stream;
  L.num_sms = h->num_sms;
  const int64_t t256 = (h->n + 255) / 256;
  L.grid_k3 = (int)std::max<int64_t>(1, std::min<int64_t>(8 * h->num_sms, t256));
  L.proj_tma = h->variant == 3 ? 1 : (h->variant == 5 ? 3 : 2);
  L.tmaps = h->tmaps.data();
  L.spmv_nf_wide = h->spmv_nf_wide;
  L.spmv_force_halo = h->spmv_force_halo;
  L.halo_peer = peer_active(h) ? 1 : 0;
  L.grid_spmv = exchange_active(h) ? std::max(1, h->num_sms - h->comm_sms) : h->num_sms;
  L.spmv_ring_tpr = h->spmv_ring_tpr;
  L.spmv_xs_tpr = h->spmv_xs_tpr;
  L.xs_stages = h->xs_stages;
  L.xs_nf = h->xs_nf;
  L.ring_stages = h->ring_stages;
  L.spmv_tiled = h->spmv_tiled;
  L.prefetch = h->prefetch;
  L.proj_const_r = h->proj_const_r;
  L.norm_tma = h->norm_tma;
  return L;
}

int free_workspace(te_handle* h) {
  cudaFree(h->d_V);
  cudaFree(h->d_W);
  h->d_V = nullptr;
  h->d_W = nullptr;
  h->m_cap = 0;
  // the peer table described the freed V: every rank reallocates V at the same call (same m_max,
  // collective evolve), so every rank re-runs the collective setup_peers before its next restart,
  // even when cudaMalloc hands back the same address
  h->peer_for_V = nullptr;
  return TE_OK;
}

// 2-D TMA descriptors of V (dim0 = 2n doubles, contiguous; dim1 = columns, stride ldv*16 B),
// one per column count: box = 64 R doubles (32 R complex rows, R = proj_rsub) x ncols columns.
int build_tensor_maps(te_handle* h) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return set_err(TE_ERR_CUDA, "cuTensorMapEncodeTiled not available");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const int nmaps = std::min(h->m_cap, te::kMaxCols);
  h->tmaps.assign(te::kMaxCols, CUtensorMap{});
  for (int c = 1; c <= nmaps; ++c) {
    cuuint64_t gdim[2] = {(cuuint64_t)(2 * h->n), (cuuint64_t)h->m_cap};
    cuuint64_t gstride[1] = {(cuuint64_t)(h->ldv * 16)};
    cuuint32_t box[2] = {(cuuint32_t)(64 * te::proj_rsub(c)), (cuuint32_t)c};
    cuuint32_t estr[2] = {1u, 1u};
    CUresult r = encode(&h->tmaps[c - 1], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, h->d_V, gdim, gstride, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(TE_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) for %d columns", (int)r, c);
  }
  return TE_OK;
}

// All initialisation is stream-ordered on the handle's current stream: the handle's own stream is
// non-blocking, so a plain cudaMemset (legacy default stream, asynchronous for device memory) could
// land after the v0 upload or the first kernels of that stream (an intermittent wrong first SpMV
// and corrupted reduction tickets, seen as rare parity failures in the GPU tests)
int ensure_workspace(te_handle* h, int m) {
  cudaStream_t s = h->stream ? h->stream : h->own_stream;
  if (h->d_small == nullptr) {
    CK(cudaMalloc(&h->d_small, sizeof(double) * kSmallLen));
    CK(cudaMemsetAsync(h->d_small, 0, sizeof(double) * kSmallLen, s));
    CK(cudaMalloc(&h->d_g, sizeof(double2) * kGLen));
    CK(cudaMemsetAsync(h->d_g, 0, sizeof(double2) * kGLen, s));
    CK(cudaMalloc(&h->d_G, sizeof(double2) * te::kMaxCols * te::kMaxCols));
    CK(cudaMemsetAsync(h->d_G, 0, sizeof(double2) * te::kMaxCols * te::kMaxCols, s));
    h->max_grid = 8 * h->num_sms;
    CK(cudaMalloc(&h->d_part, sizeof(double2) * te::kMaxCols * h->max_grid));
    CK(cudaMalloc(&h->d_partn, sizeof(double) * h->max_grid));
    CK(cudaMalloc(&h->d_counter, sizeof(unsigned) * 8));
    CK(cudaMemsetAsync(h->d_counter, 0, sizeof(unsigned) * 8, s));
    CK(cudaMallocHost(&h->h_small, sizeof(double) * kSmallLen));
    CK(cudaMallocHost(&h->h_coef, sizeof(double2) * 64));
  }
  if (m <= h->m_cap) return TE_OK;
  free_workspace(h);
  h->ldv = (h->n + 31) / 32 * 32;
  const size_t bytes = sizeof(double2) * (size_t)h->ldv * (size_t)m;
  cudaError_t e = cudaMalloc(&h->d_V, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    h->d_V = nullptr;
    return set_err(TE_ERR_OOM, "cannot allocate the Krylov basis (%zu bytes)", bytes);
  }
  CK(cudaMemsetAsync(h->d_V, 0, bytes, s));
  CK(cudaMalloc(&h->d_W, sizeof(double2) * (size_t)h->ldv));
  h->m_cap = m;
  return build_tensor_maps(h);
}

// ---------------------------------------------------------------- profiling around launches
void prof_begin(te_handle* h) {
  if (!h->profile) return;
  if (!h->ev_ready) {
    for (int i = 0; i < kEvPool; ++i) {
      cudaEventCreate(&h->ev0[i]);
      cudaEventCreate(&h->ev1[i]);
    }
    cudaEventCreate(&h->evk0);
    cudaEventCreate(&h->evk1);
    h->ev_ready = true;
  }
  // external record: inside stream capture this becomes a timing event-record node of the graph
  if (h->ev_used < kEvPool)
    cudaEventRecordWithFlags(h->ev0[h->ev_used], h->stream, h->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
}
void prof_end(te_handle* h, int cls, double bytes) {
  ++h->launches;
  static const bool dbg = getenv("TE_DEBUG_SYNC") != nullptr;
  if (dbg) {
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "[te] kernel class %d failed: %s\n", cls, cudaGetErrorString(e));
  }
  if (!h->profile || h->ev_used >= kEvPool) return;
  cudaEventRecordWithFlags(h->ev1[h->ev_used], h->stream, h->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
  h->ev_cls[h->ev_used] = cls;
  h->ev_bytes[h->ev_used] = bytes;
  ++h->ev_used;
}
void prof_collect(te_handle* h) {
  if (h->evk_pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->evk0, h->evk1);
    h->prof[3].launches += 1;
    h->prof[3].total_ms += ms;
    h->prof[3].alg_bytes += h->evk_bytes;
    h->evk_pending = false;
  }
  for (int i = 0; i < h->ev_used; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev0[i], h->ev1[i]);
    te_kernel_profile& p = h->prof[h->ev_cls[i]];
    p.launches += 1;
    p.total_ms += ms;
    p.alg_bytes += h->ev_bytes[i];
  }
  h->ev_used = 0;
}

// ---------------------------------------------------------------- distributed collectives
int allreduce_sum(te_handle* h, double* buf, size_t count) {
  if (!h->dist || h->dist->nranks == 1) return TE_OK;
  CKN(te::nccl().AllReduce(buf, buf, count, ncclDouble, ncclSum, h->dist->comm, h->stream));
  return TE_OK;
}

// Fork: the side stream waits for everything issued so far on the main stream (V_j complete), packs
// V_j[send_idx] and runs the grouped send/recv into the halo buffer while the main stream runs
// the local-column SpMV; halo_join makes the main stream wait before k_spmv_halo.  Both are
// plain event edges, so a captured restart graph contains them (and the NCCL calls) as well.
int halo_exchange(te_handle* h, int j) {
  if (!exchange_active(h)) return TE_OK;
  const double2* x = h->d_V + (int64_t)j * h->ldv;
  CK(cudaEventRecord(h->ev_fork, h->stream));
  CK(cudaStreamWaitEvent(h->comm_stream, h->ev_fork, 0));
  if (h->n_send > 0) {
    te::launch_pack(x, h->d_send_idx, h->n_send, h->d_sendbuf, h->comm_stream);
    ++h->launches;
  }
  auto& N = te::nccl();
  CKN(N.GroupStart());
  int64_t so = 0, ro = 0;
  for (int q = 0; q < h->dist->nranks; ++q) {
    if (q == h->dist->rank) continue;
    if (h->send_counts[q] > 0)
      CKN(N.Send(h->d_sendbuf + so, 2 * (size_t)h->send_counts[q], ncclDouble, q, h->dist->comm, h->comm_stream));
    if (h->recv_counts[q] > 0)
      CKN(N.Recv(h->d_halo + ro, 2 * (size_t)h->recv_counts[q], ncclDouble, q, h->dist->comm, h->comm_stream));
    so += h->send_counts[q];
    ro += h->recv_counts[q];
  }
  CKN(N.GroupEnd());
  CK(cudaEventRecord(h->ev_join, h->comm_stream));
  return TE_OK;
}
int halo_join(te_handle* h) {
  if (!exchange_active(h)) return TE_OK;
  CK(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
  return TE_OK;
}

// Halo mode 1: every rank learns every rank's V base and column stride (collective, once per V
// allocation).  A peer in the same address space (several ranks as threads of one process) is
// addressed directly; another process's V is mapped through CUDA IPC (NVLink peer access).
int setup_peers(te_handle* h) {
  struct Rec {
    cudaIpcMemHandle_t hdl;
    uint64_t ptr;
    int64_t ldv;
    int64_t pid;
  };
  const int P = h->dist->nranks, me = h->dist->rank;
  Rec mine{};
  if (cudaIpcGetMemHandle(&mine.hdl, h->d_V) != cudaSuccess) {
    cudaGetLastError();  // not exportable: peers in this process still work through the pointer
    std::memset(&mine.hdl, 0, sizeof(mine.hdl));
  }
  mine.ptr = reinterpret_cast<uint64_t>(h->d_V);
  mine.ldv = h->ldv;
  mine.pid = (int64_t)getpid();
  std::vector<Rec> all(P);
  char* dbuf = nullptr;
  CK(cudaMalloc(&dbuf, sizeof(Rec) * (P + 1)));
  CK(cudaMemcpyAsync(dbuf, &mine, sizeof(Rec), cudaMemcpyHostToDevice, h->stream));
  {
    const ncclResult_t r = te::nccl().AllGather(dbuf, dbuf + sizeof(Rec), sizeof(Rec), ncclChar, h->dist->comm, h->stream);
    if (r != ncclSuccess) {
      cudaFree(dbuf);
      return set_err(TE_ERR_NCCL, "peer table allgather: %s", te::nccl().GetErrorString(r));
    }
  }
  CK(cudaMemcpyAsync(all.data(), dbuf + sizeof(Rec), sizeof(Rec) * P, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  cudaFree(dbuf);
  for (void* p : h->ipc_open) cudaIpcCloseMemHandle(p);
  h->ipc_open.clear();
  std::vector<const double2*> base(P);
  std::vector<int64_t> ldv(P);
  for (int q = 0; q < P; ++q) {
    ldv[q] = all[q].ldv;
    if (q == me || all[q].pid == mine.pid) {
      base[q] = reinterpret_cast<const double2*>(all[q].ptr);
    } else {
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, all[q].hdl, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return set_err(TE_ERR_CUDA, "cannot map rank %d's Krylov basis (CUDA IPC / peer access)", q);
      }
      h->ipc_open.push_back(p);
      base[q] = static_cast<const double2*>(p);
    }
  }
  if (!h->d_peer_base) {
    CK(cudaMalloc(&h->d_peer_base, sizeof(double2*) * P));
    CK(cudaMalloc(&h->d_peer_ldv, sizeof(int64_t) * P));
  }
  CK(cudaMemcpy(h->d_peer_base, base.data(), sizeof(double2*) * P, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->d_peer_ldv, ldv.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice));
  h->peer_for_V = h->d_V;
  return TE_OK;
}

// ---------------------------------------------------------------- one Krylov decomposition
// Launch the whole restart (Alg. 1 step 1) without host synchronisation: the kernels gate
// themselves on the device breakdown flag.  Then one D2H of alpha/beta/flag.
#define LCHECK(name)                                                                        \
  do {                                                                                      \
    cudaError_t e_ = cudaGetLastError();                                                    \
    if (e_ != cudaSuccess) return set_err(TE_ERR_CUDA, "launch of %s (step j=%d): %s", name, \
                                          (int)lj, cudaGetErrorString(e_));                 \
  } while (0)

void free_colblk(te_handle* h);
// column-blocked ring: x larger than kColBlkMinX is split into nb equal column blocks of at most
// colblk_bytes() of x each (TE_SPMV_COLBLK_MB, default 48 MB: measured on config 4 (n = 2^24,
// 268 MB of x) 96 / 64 / 48 / 32 / 24 MB blocks: 4.56 / 4.41 / 3.66 / 4.01 / 4.73 ms per SpMV vs
// 5.81 ms for the ring over the whole CSR), rounded to 32 columns
constexpr double kColBlkMinX = 160.0 * 1024 * 1024;
double colblk_bytes() {
  const char* e = getenv("TE_SPMV_COLBLK_MB");
  const double v = e ? atof(e) : 48.0;
  return std::max(1e-3, v) * 1024.0 * 1024.0;
}
int64_t colblk_cols(int64_t n) {
  const int64_t nb = std::max<int64_t>(1, (int64_t)std::ceil(16.0 * (double)n / colblk_bytes()));
  return std::max<int64_t>(32, ((n + nb - 1) / nb + 31) / 32 * 32);
}

// nnz-balanced tiles of the warp-specialised ring: <= 480/tpr rows and <= the stage capacity in
// entries, {first row, end row, first entry, end entry}
std::vector<int64_t> ring_tiles(int64_t n, const int64_t* rowptr, bool cplx, int stages, int tpr) {
  const int64_t rcap = 480 / tpr;
  const int64_t ncap = stages == 3 ? (cplx ? te::kRingNnzC3 : te::kRingNnz3) : (cplx ? te::kRingNnzC4 : te::kRingNnz4);
  std::vector<int64_t> tg;
  int64_t st = 0;
  for (int64_t r = 0; r < n; ++r) {
    const bool over_rows = (r + 1 - st) > rcap;
    const bool over_nnz = (rowptr[r + 1] - rowptr[st]) > ncap && r > st;
    if (over_rows || over_nnz) {
      tg.insert(tg.end(), {st, r, rowptr[st], rowptr[r]});
      st = r;
    }
  }
  if (n > 0) tg.insert(tg.end(), {st, n, rowptr[st], rowptr[n]});
  return tg;
}

// Column-blocked copy of the (single-rank) CSR: block b = columns [b B, (b+1) B); each block is a
// CSR over all rows with its own ring tile table and lanes per row (from its mean row length).
// Counts on the device, prefix sums on the host, fill on the device.  Leaves h->cb empty when
// there is no room.
int build_colblk(te_handle* h, int64_t B) {
  free_colblk(h);
  const int64_t n = h->n;
  const int nb = (int)((n + B - 1) / B);
  if (nb < 2 || h->ncol_limit != n) return TE_OK;
  cudaStream_t s = h->stream ? h->stream : h->own_stream;
  int32_t* dcnt = nullptr;
  if (cudaMalloc(&dcnt, sizeof(int32_t) * (size_t)n * nb) != cudaSuccess) {
    cudaGetLastError();
    return TE_OK;
  }
  te::launch_colblk_count(n, h->d_rowptr, h->d_col, B, nb, dcnt, s);
  std::vector<int32_t> cnt((size_t)n * nb);
  CK(cudaMemcpyAsync(cnt.data(), dcnt, sizeof(int32_t) * (size_t)n * nb, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  cudaFree(dcnt);
  const size_t vb = h->cplx ? 16 : 8;
  std::vector<int64_t> rp((size_t)n + 1);
  h->cb.resize((size_t)nb);
  for (int b = 0; b < nb; ++b) {
    rp[0] = 0;
    for (int64_t r = 0; r < n; ++r) rp[(size_t)r + 1] = rp[(size_t)r] + cnt[(size_t)b * n + r];
    const int64_t nz = rp[(size_t)n];
    auto& Bk = h->cb[(size_t)b];
    // lanes per row of this block's pass: the handle's rule (<= 20 real / 8 complex entries per lane)
    const double avg = (double)nz / (double)n;
    int tpr = 1;
    while (tpr < 8 && avg > (h->cplx ? 8.0 : 20.0) * tpr) tpr <<= 1;
    Bk.tpr = tpr;
    const std::vector<int64_t> tg = ring_tiles(n, rp.data(), h->cplx, h->ring_stages, tpr);
    Bk.ntiles = (int64_t)tg.size() / 4;
    // (+8 padding entries: the ring's 16-byte-aligned bulk copies may read past the last entry)
    if (cudaMalloc(&Bk.rowptr, sizeof(int64_t) * (n + 2)) != cudaSuccess || cudaMalloc(&Bk.col, 4 * (size_t)(nz + 8)) != cudaSuccess ||
        cudaMalloc(&Bk.val, vb * (size_t)(nz + 8)) != cudaSuccess || cudaMalloc(&Bk.tiles, sizeof(int64_t) * std::max<size_t>(4, tg.size())) != cudaSuccess) {
      cudaGetLastError();
      free_colblk(h);
      return TE_OK;
    }
    CK(cudaMemcpyAsync(Bk.rowptr, rp.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(Bk.col, 0, 4 * (size_t)(nz + 8), s));
    CK(cudaMemsetAsync(Bk.val, 0, vb * (size_t)(nz + 8), s));
    if (!tg.empty()) CK(cudaMemcpyAsync(Bk.tiles, tg.data(), sizeof(int64_t) * tg.size(), cudaMemcpyHostToDevice, s));
    te::launch_colblk_fill(n, h->d_rowptr, h->d_col, h->d_val, h->cplx, B, b, Bk.rowptr, Bk.col, Bk.val, s);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));  // rp / tg are reused for the next block
  }
  h->cb_cols = B;
  return TE_OK;
}

void free_colblk(te_handle* h) {
  for (auto& b : h->cb) {
    cudaFree(b.rowptr);
    cudaFree(b.col);
    cudaFree(b.val);
    cudaFree(b.tiles);
  }
  h->cb.clear();
  h->cb_cols = 0;
}

// K1a: the SpMV of step j.  Column-blocked (variant 10): one ring pass per column block, passes > 0
// accumulate into W (stream-ordered launches; row sums block by block, deterministic)
void spmv_call(te_handle* h, const KDev& d, int j, const Launch& L) {
  if (h->spmv_tiled != 10 || h->cb.empty()) {
    te::launch_spmv(d, h->cplx, j, L);
    if (h->spmv_tiled == 9 && h->sw_nslice > 0 && h->d_swb_sptr) {  // panel sweep: the far windows
      KDev db = d;
      db.sw_sptr = h->d_swb_sptr;
      db.sw_base = h->d_swb_base;
      db.sw_ent = h->d_swb_ent;
      db.sw_pass = 2;
      te::launch_spmv(db, h->cplx, j, L);
      ++h->launches;
    }
    return;
  }
  Launch Lr = L;
  Lr.spmv_tiled = 7;
  for (size_t b = 0; b < h->cb.size(); ++b) {
    KDev db = d;
    db.rowptr = h->cb[b].rowptr;
    db.col = h->cb[b].col;
    db.val = h->cb[b].val;
    db.tile_ring = h->cb[b].tiles;
    db.ntiles_ring = h->cb[b].ntiles;
    db.accw = b > 0 ? 1 : 0;
    Lr.spmv_ring_tpr = h->cb[b].tpr;
    te::launch_spmv(db, h->cplx, j, Lr);
  }
  h->launches += (int64_t)h->cb.size() - 1;
}

int issue_arnoldi(te_handle* h, int m, double tol_rate) {
  int lj = -1;
  KDev d = make_kdev(h, tol_rate, m);
  Launch L = make_launch(h);
  const double n = (double)h->n;
  const double vbytes = h->cplx ? 16.0 : 8.0;
  // H bytes of the streamed format: CSR (value + int32 column), staged-x (value + 16-bit slot),
  // staged-x with the value dictionary (8-bit code + 16-bit slot, plus one diagonal value per row)
  double bh = (double)(h->nnz + h->nh_entries) * (vbytes + 4.0) + 8.0 * (n + 1.0);
  if (h->spmv_tiled == 8 && h->ntiles_xs > 0)
    bh = (double)h->nnz * (vbytes + 2.0) + 8.0 * (n + 1.0);
  if (h->spmv_tiled == 8 && h->ntiles_xs > 0) bh += (double)h->nh_entries * (vbytes + 4.0);
  // column-blocked ring: algorithmic bytes are those of the CSR it was cut from (the per-pass row
  // pointers and the W re-reads of passes > 0 are overhead of the method, not counted)
  // slot-window SELL-32: 2 bytes per slot entry (padding included), the slot bases, the slice
  // pointers and the dense diagonal
  if (h->spmv_tiled == 9 && h->sw_nslice > 0)
    bh = (double)(h->sw_slots + h->swb_slots) * ((h->sw_bits == 8 ? 32.0 : 64.0) + 4.0) +
         8.0 * (double)(h->sw_nslice + 1) * (h->d_swb_sptr ? 2.0 : 1.0) + n * vbytes +
         (double)h->nh_entries * (vbytes + 4.0);
  te::launch_restart_init(d, L); LCHECK("restart_init");
  ++h->launches;
  for (int j = 0; j < m; ++j) {
    lj = j;
    int rc = halo_exchange(h, j);
    if (rc) return rc;
    const double ncols = j + 1;
    if (h->ortho == 1) {  // paper-literal Lanczos (Eq. 8 as printed)
      prof_begin(h);
      spmv_call(h, d, j, L); LCHECK("spmv");
      if ((rc = halo_join(h))) return rc;
      te::launch_spmv_halo(d, h->cplx, j, L); LCHECK("spmv_halo");
      prof_end(h, 0, bh + 16.0 * n + 16.0 * n);
      const double nv = j > 0 ? 2.0 : 1.0;
      prof_begin(h);
      te::launch_lanczos_dot(d, j, L); LCHECK("lanczos_dot");
      prof_end(h, 5, 16.0 * n * nv + 16.0 * n);
      if ((rc = allreduce_sum(h, reinterpret_cast<double*>(d.g1 + j), 2))) return rc;
      const bool wr = j + 1 < m;
      prof_begin(h);
      te::launch_lanczos_update(d, j, wr, L); LCHECK("lanczos_update");
      prof_end(h, 2, 16.0 * n * nv + 16.0 * n + (wr ? 16.0 * n : 0.0));
      if ((rc = allreduce_sum(h, d.nrm2 + j, 1))) return rc;
      continue;
    }
    // CGS2 and f2 (defer mode): the SpMV writes H V_j unscaled; the update kernel applies s_j after
    // the step's first reduction, which carries ||p''_{j-1}||^2 next to g1 (and, for f2, the
    // previous update pass's Gram dots g2): 2 allreduces per step for CGS2, 1 for f2 (plus one
    // barrier per step in peer-load halo mode, where a rank's SpMV reads its peers' V_j)
    prof_begin(h);
    spmv_call(h, d, j, L); LCHECK("spmv");
    if ((rc = halo_join(h))) return rc;
    te::launch_spmv_halo(d, h->cplx, j, L); LCHECK("spmv_halo");
    prof_end(h, 0, bh + 16.0 * n + 16.0 * n);
    prof_begin(h);
    te::launch_proj_dots(d, j, L); LCHECK("proj_dots");
    prof_end(h, 5, 16.0 * n * ncols + 16.0 * n);
    const bool wr = j + 1 < m;
    if (h->ortho == 2) {  // f2: CGS2 with the Gram-matrix second sweep, two V passes per step
      if ((rc = allreduce_sum(h, reinterpret_cast<double*>(h->d_g), 2 * (size_t)(kOffG2 + j)))) return rc;
      prof_begin(h);
      te::launch_gram_update(d, j, wr, L); LCHECK("gram_update");
      prof_end(h, 1, 16.0 * n * ncols + 16.0 * n + (wr ? 16.0 * n : 0.0));
    } else {
      if ((rc = allreduce_sum(h, reinterpret_cast<double*>(h->d_g), 2 * (size_t)(kOffG1 + j + 1)))) return rc;
      prof_begin(h);
      te::launch_update_proj(d, j, L); LCHECK("update_proj");
      prof_end(h, 1, 16.0 * n * ncols + 32.0 * n);
      if ((rc = allreduce_sum(h, reinterpret_cast<double*>(d.g2), 2 * (size_t)(j + 1)))) return rc;
      prof_begin(h);
      te::launch_update_norm(d, j, wr, L); LCHECK("update_norm");
      prof_end(h, 2, 16.0 * n * ncols + 16.0 * n + (wr ? 16.0 * n : 0.0));
    }
    if (peer_active(h) && wr) {  // V_{j+1} complete on every rank before any rank's next SpMV reads it
      if ((rc = allreduce_sum(h, h->d_small + kOffScalar, 1))) return rc;
    }
  }
  if (h->ortho != 1) {  // the last step's ||p''_{m-1}||^2 (h_{m+1,m}) is reduced once per restart
    const int rc = allreduce_sum(h, h->d_small + kOffNrm + (m - 1), 1);
    if (rc) return rc;
  }
  te::launch_finalize(d, m - 1, L); LCHECK("finalize");
  ++h->launches;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(h->h_small, h->d_small, sizeof(double) * (kOffFlag + 2), cudaMemcpyDeviceToHost, h->stream));
  return TE_OK;
}

// One restart's Arnoldi decomposition.  With graphs on (default, single rank) the launch sequence
// is captured once per (m, tol_rate, kernel set, basis allocation, profiling) and replayed; the
// profiling events are captured as event-record nodes and read back after each replay.
// Wait for the restart on the host.  With several ranks the wait polls the communicator's
// asynchronous error state, so a failed or vanished peer ends te_evolve with TE_ERR_NCCL (the
// communicator is aborted) instead of blocking forever in a collective.
int wait_restart(te_handle* h) {
  if (!h->dist || h->dist->nranks == 1 || !te::nccl().CommGetAsyncError) {
    CK(cudaStreamSynchronize(h->stream));
    return TE_OK;
  }
  for (int spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(h->stream);
    if (q == cudaSuccess) return TE_OK;
    if (q != cudaErrorNotReady) CK(q);
    ncclResult_t ar = ncclSuccess;
    if (te::nccl().CommGetAsyncError(h->dist->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress) {
      if (te::nccl().CommAbort) te::nccl().CommAbort(h->dist->comm);
      h->dist->comm = nullptr;
      return set_err(TE_ERR_NCCL, "NCCL communicator failed during the restart: %s", te::nccl().GetErrorString(ar));
    }
    if (spin > 64) usleep(20);
  }
}

int run_arnoldi(te_handle* h, int m, double tol_rate) {
  Nvtx range("te: Krylov decomposition (Alg. 1 step 1)");
  if (h->dist && h->dist->nranks > 1 && !h->dist->comm) return set_err(TE_ERR_NCCL, "communicator was aborted");
  if (peer_active(h) && h->peer_for_V != h->d_V) {  // collective; never inside a graph capture
    const int rc = setup_peers(h);
    if (rc) return rc;
  }
  // profiling uses per-launch CUDA events, which graphs do not time: direct launches then.  With
  // several ranks the restart graph holds the NCCL calls too (NCCL supports stream capture); the
  // test stand-in for NCCL (tests/support/fake_nccl.cu) does not, so it runs direct launches
  const bool graph = h->use_graph && !h->profile && (!h->dist || h->dist->nranks == 1 || !te::nccl().is_fake);
  if (!graph) {
    int rc = issue_arnoldi(h, m, tol_rate);
    if (rc) return rc;
    if ((rc = wait_restart(h))) return rc;
    if (h->profile) prof_collect(h);
    return TE_OK;
  }
  const bool hit = h->gexec && h->g_m == m && h->g_tol_rate == tol_rate && h->g_variant == h->variant &&
                   h->g_ortho == h->ortho && h->g_prefetch == h->prefetch && h->g_halo == h->halo_mode &&
                   h->g_spmv == h->spmv_tiled && h->g_profile == h->profile && h->g_V == (const void*)h->d_V;
  if (!hit) {
    if (h->gexec) {
      cudaGraphExecDestroy(h->gexec);
      h->gexec = nullptr;
    }
    if (h->profile && !h->ev_ready) prof_begin(h);  // make sure the event pool exists
    cudaStream_t user = h->stream;
    h->stream = h->own_stream;
    const int64_t l0 = h->launches;
    const int ev0 = h->ev_used;
    CK(cudaStreamBeginCapture(h->own_stream, cudaStreamCaptureModeThreadLocal));
    h->capturing = true;
    int rc = issue_arnoldi(h, m, tol_rate);
    h->capturing = false;
    cudaGraph_t g = nullptr;
    cudaError_t ce = cudaStreamEndCapture(h->own_stream, &g);
    h->stream = user;
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ce != cudaSuccess) return set_err(TE_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ce));
    ce = cudaGraphInstantiate(&h->gexec, g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) {
      h->gexec = nullptr;
      return set_err(TE_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ce));
    }
    h->g_launches = h->launches - l0;
    h->launches = l0;
    h->g_nev = h->ev_used - ev0;
    for (int i = 0; i < h->g_nev; ++i) {
      h->g_ev_cls[i] = h->ev_cls[ev0 + i];
      h->g_ev_bytes[i] = h->ev_bytes[ev0 + i];
    }
    h->ev_used = ev0;
    h->g_m = m;
    h->g_tol_rate = tol_rate;
    h->g_variant = h->variant;
    h->g_spmv = h->spmv_tiled;
    h->g_ortho = h->ortho;
    h->g_prefetch = h->prefetch;
    h->g_halo = h->halo_mode;
    h->g_profile = h->profile;
    h->g_V = h->d_V;
  }
  CK(cudaGraphLaunch(h->gexec, h->stream));
  h->launches += h->g_launches;
  {
    const int rc = wait_restart(h);
    if (rc) return rc;
  }
  if (h->profile) {
    for (int i = 0; i < h->g_nev; ++i) {
      h->ev_cls[i] = h->g_ev_cls[i];
      h->ev_bytes[i] = h->g_ev_bytes[i];
    }
    h->ev_used = h->g_nev;
    prof_collect(h);
  }
  return TE_OK;
}

int read_flag(te_handle* h, int m, int* m_eff, bool* breakdown) {
  const int* fl = reinterpret_cast<const int*>(h->h_small + kOffFlag);
  if (fl[0] == 2) return set_err(TE_ERR_NUMERICAL, "non-finite value in the Arnoldi recurrence (step %d)", fl[1]);
  *breakdown = fl[0] == 1;
  *m_eff = fl[0] == 0 ? m : fl[1];
  if (*m_eff < 1 || *m_eff > m) return set_err(TE_ERR_CUDA, "inconsistent device state (m_eff=%d)", *m_eff);
  return TE_OK;
}

// ---------------------------------------------------------------- Algorithm 1
// V[:,0] holds v0 on entry; on success V[:,0] holds v(t).
struct Sampling {
  int64_t n = 0;
  const double* times = nullptr;  // ascending, in [0, t]
  te_c128* out = nullptr;         // n x n_local host, row-major (sample-major)
  double* bounds = nullptr;       // nullable
};

int evolve_core(te_handle* h, double t, double tol, int m_max, const double* forced, int64_t nforced,
                te_stats* st, const Sampling* smp = nullptr) {
  Nvtx range("te_evolve");
  te_stats S{};
  S.one_norm = h->norm1;
  S.roundoff_step = (double)h->n_global * h->norm1 * std::ldexp(1.0, -52);  // Eq. 17
  S.t_step_min = 0.0;
  S.t_step_max = 0.0;
  h->sched.clear();
  auto fill = [&]() {
    S.roundoff_total = S.roundoff_step * (double)S.n_restarts;
    if (st) *st = S;
  };
  // ||v0|| = 1 check
  {
    KDev d = make_kdev(h, 0.0, 1);
    Launch L = make_launch(h);
    te::launch_norm2(d, h->d_V, h->d_small + kOffScalar, L);
    ++h->launches;
    int rc = allreduce_sum(h, h->d_small + kOffScalar, 1);
    if (rc) return rc;
    CK(cudaMemcpyAsync(h->h_small + kOffScalar, h->d_small + kOffScalar, sizeof(double), cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    const double nv = std::sqrt(h->h_small[kOffScalar]);
    if (!(std::fabs(nv - 1.0) <= 1e-8)) {
      fill();
      return set_err(TE_ERR_NOT_NORMALIZED, "| ||v0|| - 1 | = %.3e > 1e-8", std::fabs(nv - 1.0));
    }
  }
  int64_t si = 0;
  const size_t vbytes = sizeof(double2) * (size_t)h->n;
  if (smp) {  // samples at t_s <= 0: the initial state
    for (; si < smp->n && smp->times[si] <= 0.0; ++si) {
      CK(cudaMemcpyAsync(smp->out + (size_t)si * h->n, h->d_V, vbytes, cudaMemcpyDeviceToHost, h->stream));
      if (smp->bounds) smp->bounds[si] = 0.0;
    }
  }
  if (t == 0.0) {
    CK(cudaStreamSynchronize(h->stream));
    fill();
    return TE_OK;
  }
  const int m = (int)std::min<int64_t>(m_max, h->n_global);
  const double tol_rate = tol / t;  // Eq. 18
  double t_now = 0.0, tau_prev = 0.0;
  std::vector<std::complex<double>> om(m);
  int64_t k = 0;
  while (t_now < t) {
    if (forced && k >= nforced) break;
    int rc = run_arnoldi(h, m, tol_rate);
    if (rc) { fill(); return rc; }
    int m_eff = 0;
    bool brk = false;
    if ((rc = read_flag(h, m, &m_eff, &brk))) { fill(); return rc; }
    const auto host_t0 = std::chrono::steady_clock::now();
    Nvtx range_host("te: eigensolve + error integral + step search (Alg. 1 step 2)");
    const double* alpha = h->h_small + kOffAlpha;
    const double* beta = h->h_small + kOffBeta;
    te::SmallEig E;
    if (!te::tridiag_eig(m_eff, alpha, beta, E)) {
      fill();
      return set_err(TE_ERR_NUMERICAL, "tridiagonal eigensolver did not converge");
    }
    E.h = beta[m_eff - 1];
    const double rem = t - t_now;
    double tau, err;
    bool qok = true;
    if (forced) {
      tau = std::min(forced[k], rem);
      te::QuadResult q = te::integrate(E, 0.0, tau, tol_rate, h->integrator);
      err = q.value;
      qok = q.converged;
    } else {
      te::StepResult r = te::find_step(E, brk, k == 0, tau_prev, rem, tol_rate, t, h->integrator);
      if (r.collapse) {
        fill();
        return set_err(TE_ERR_STEP_COLLAPSE, "step size collapsed below 1e-13 t (m=%d too small for tol=%g)", m, tol);
      }
      tau = r.tau;
      err = r.err;
      qok = r.quad_ok;
    }
    // states at intermediate times inside this step: w_s = V exp(-iT(t_s - t_now)) e_1
    const double t_end = (tau >= rem) ? t : t_now + tau;
    for (; smp && si < smp->n && smp->times[si] <= t_end; ++si) {
      const double ds = std::min(smp->times[si] - t_now, tau);
      te::omega(E, ds, om.data());
      for (int q = 0; q < m_eff; ++q) {
        const double s = q == 0 ? 1.0 : 1.0 / beta[q - 1];
        h->h_coef[q] = make_double2(om[q].real() * s, om[q].imag() * s);
      }
      CK(cudaMemcpyAsync(h->d_g + kOffCoef, h->h_coef, sizeof(double2) * m_eff, cudaMemcpyHostToDevice, h->stream));
      KDev d = make_kdev(h, tol_rate, m);
      Launch L = make_launch(h);
      te::launch_combine(d, h->d_g + kOffCoef, m_eff, h->d_W, L);
      ++h->launches;
      CK(cudaMemcpyAsync(smp->out + (size_t)si * h->n, h->d_W, vbytes, cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));  // h_coef is reused below
      if (smp->bounds) smp->bounds[si] = S.err_bound + te::integrate(E, 0.0, ds, tol_rate, h->integrator).value;
    }
    // omega~_k = s_k omega_k with s_0 = 1, s_k = 1/beta_{k-1} (columns stored unnormalised)
    te::omega(E, tau, om.data());
    for (int q = 0; q < m_eff; ++q) {
      const double s = q == 0 ? 1.0 : 1.0 / beta[q - 1];
      h->h_coef[q] = make_double2(om[q].real() * s, om[q].imag() * s);
    }
    if (h->profile) {
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
      h->prof[6].launches += 1;
      h->prof[6].total_ms += ms;
    }
    CK(cudaMemcpyAsync(h->d_g + kOffCoef, h->h_coef, sizeof(double2) * m_eff, cudaMemcpyHostToDevice, h->stream));
    {
      KDev d = make_kdev(h, tol_rate, m);
      Launch L = make_launch(h);
      if (h->profile) {
        prof_begin(h);  // creates the event pool on first use
        cudaEventRecord(h->evk0, h->stream);
      }
      te::launch_combine(d, h->d_g + kOffCoef, m_eff, h->d_V, L);
      ++h->launches;
      if (peer_active(h)) {  // peers read the new V_0 directly in the next SpMV: barrier
        const int rc = allreduce_sum(h, h->d_small + kOffScalar, 1);
        if (rc) return rc;
      }
      if (h->profile) {
        cudaEventRecord(h->evk1, h->stream);
        h->evk_pending = true;
        h->evk_bytes = 16.0 * (double)h->n * (m_eff + 1);
      }
    }
    t_now = (tau >= rem) ? t : t_now + tau;
    tau_prev = tau;
    S.err_bound += err;
    S.n_restarts += 1;
    S.n_krylov_steps += m_eff;
    S.n_breakdowns += brk ? 1 : 0;
    if (S.roundoff_step > err) S.warnings |= TE_WARN_ROUNDOFF;
    if (!qok) S.warnings |= TE_WARN_QUADRATURE;
    S.t_step_min = (S.n_restarts == 1) ? tau : std::min(S.t_step_min, tau);
    S.t_step_max = std::max(S.t_step_max, tau);
    h->sched.push_back({tau, m_eff, err});
    ++k;
  }
  CK(cudaGetLastError());
  if (h->profile) {
    CK(cudaStreamSynchronize(h->stream));
    prof_collect(h);
  }
  fill();
  return TE_OK;
}

int check_evolve_args(te_handle* h, double t, double tol, int m_max) {
  if (!h) return set_err(TE_ERR_ARG, "null handle");
  if (!(t >= 0.0) || !std::isfinite(t)) return set_err(TE_ERR_ARG, "t must be finite and >= 0");
  if (!(tol > 0.0) || !std::isfinite(tol)) return set_err(TE_ERR_ARG, "tol must be > 0");
  if (m_max < 1 || m_max > TE_M_MAX) return set_err(TE_ERR_ARG, "m_max must be in [1, %d]", TE_M_MAX);
  return TE_OK;
}

// ---------------------------------------------------------------- staged-x SpMV plan
void free_xs(te_handle* h) {
  cudaFree(h->d_tile_xs);
  cudaFree(h->d_xs_meta);
  cudaFree(h->d_xs_rng);
  cudaFree(h->d_lcol);
  h->d_tile_xs = nullptr;
  h->d_xs_meta = nullptr;
  h->d_xs_rng = nullptr;
  h->d_lcol = nullptr;
  h->ntiles_xs = 0;
}

// Tiles of <= 32*15/TPR rows and <= xs_ecap entries (TPR: <= 8 entries per lane of a mean-length
// row), then the device plan (spmv_xs.cu): per tile the x ranges to stage and each entry's slot.
// rowptr: host copy of the (local) row pointers.
// Value dictionary on the device: distinct off-diagonal values (bit patterns) into a 1024-slot hash
// table; if there are at most 255, sorted by bit pattern they become codes 0..254 (255: padding in
// the slot-window SELL).  Returns the number of values, or -1
// when there are more than 255 (keys: the sorted values, imaginary part 0 for real H).
int collect_dict(te_handle* h, std::vector<double2>& keys_out) {
  cudaStream_t s = h->stream ? h->stream : h->own_stream;
  constexpr int cap = 1024;
  const size_t tb = te::dict_slot_bytes() * cap;
  void* table = nullptr;
  if (cudaMalloc(&table, tb + 16) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  unsigned* count = reinterpret_cast<unsigned*>(static_cast<char*>(table) + tb);
  cudaMemsetAsync(table, 0, tb + 16, s);
  te::launch_dict_insert(h->n, h->d_rowptr, h->d_col, h->d_val, h->cplx, table, cap, count, s);
  std::vector<unsigned char> ht(tb + 16);
  cudaMemcpyAsync(ht.data(), table, tb + 16, cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  cudaFree(table);
  if (e != cudaSuccess) return -1;
  unsigned cnt = 0;
  std::memcpy(&cnt, ht.data() + tb, sizeof cnt);
  if (cnt > 255) return -1;
  struct Slot { unsigned state, pad; double re, im; };
  std::vector<std::pair<std::pair<uint64_t, uint64_t>, double2>> keys;
  for (int i = 0; i < cap; ++i) {
    Slot sl;
    std::memcpy(&sl, ht.data() + (size_t)i * sizeof(Slot), sizeof sl);
    if (sl.state != 2u) continue;
    uint64_t a, b;
    std::memcpy(&a, &sl.re, 8);
    std::memcpy(&b, &sl.im, 8);
    keys.push_back({{a, b}, make_double2(sl.re, sl.im)});
  }
  std::sort(keys.begin(), keys.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
  keys_out.clear();
  for (const auto& k : keys) keys_out.push_back(k.second);
  return (int)keys_out.size();
}

// ---------------------------------------------------------------- slot-window SELL-32 (variant 9)
void free_sw(te_handle* h) {
  cudaFree(h->d_sw_sptr);
  cudaFree(h->d_sw_base);
  cudaFree(h->d_sw_ent);
  cudaFree(h->d_sw_diag);
  cudaFree(h->d_sw_dict);
  cudaFree(h->d_swb_sptr);
  cudaFree(h->d_swb_base);
  cudaFree(h->d_swb_ent);
  h->d_swb_sptr = nullptr;
  h->d_swb_base = nullptr;
  h->d_swb_ent = nullptr;
  h->swb_slots = 0;
  h->sw_ka = h->sw_sb = h->sw_lo = h->sw_ob = 0;
  h->d_sw_sptr = nullptr;
  h->d_sw_base = nullptr;
  h->d_sw_ent = nullptr;
  h->d_sw_diag = nullptr;
  h->d_sw_dict = nullptr;
  h->sw_nslice = h->sw_slots = 0;
  h->sw_ndict = 0;
}

// Build the slot-window SELL-32 copy of the local CSR: applicable when the off-diagonal values take
// at most 255 distinct values and the slot entries (32 per slot, padding included) stay within
// kSwMaxFill times the off-diagonal entry count.  Not applicable: TE_OK with sw_nslice = 0
// (sw_fill reports the padding ratio when the dictionary exists).
constexpr double kSwMaxFill = 1.6;    // 16-bit entries
// staged-x is the default only from this many rows on (config 1, n = 4096: ring 31.1K vs staged-x
// 28.9K Krylov steps/s; the tiny x is L1/L2-resident either way and the staging is overhead)
constexpr int64_t kXsMinRows = 65536;
constexpr double kSwMaxFill8 = 2.0;   // 8-bit entries (half the bytes per slot entry)
int plan_sw(te_handle* h) {
  free_sw(h);
  h->sw_fill = 0.0;
  if (h->ncol_limit != h->n) return TE_OK;  // local columns only (halo entries are kept apart)
  cudaStream_t s = h->stream ? h->stream : h->own_stream;
  std::vector<double2> kd;
  const int nd = collect_dict(h, kd);
  if (nd < 0) return TE_OK;
  if (kd.empty()) kd.push_back(make_double2(0.0, 0.0));
  const int64_t n = h->n, nsl = (n + 31) / 32;
  double2* dkeys = nullptr;
  int32_t* nslot = nullptr;
  int* derr = nullptr;
  auto cleanup = [&]() {
    cudaFree(dkeys);
    cudaFree(nslot);
    cudaFree(derr);
  };
  if (cudaMalloc(&dkeys, sizeof(double2) * kd.size()) != cudaSuccess || cudaMalloc(&nslot, sizeof(int32_t) * nsl) != cudaSuccess ||
      cudaMalloc(&derr, sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    cleanup();
    return TE_OK;
  }
  // 8-bit entries when the dictionary has <= 7 values (spin chains), else 16-bit (TE_SPMV_SW_BITS)
  bool b8 = nd <= 7;
  if (const char* e = getenv("TE_SPMV_SW_BITS")) b8 = b8 && atoi(e) != 16;
  CK(cudaMemcpyAsync(dkeys, kd.data(), sizeof(double2) * kd.size(), cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(derr, 0, sizeof(int), s));
  te::launch_sw_build(false, h->cplx, b8, 0, 0, n, h->d_rowptr, h->d_col, h->d_val, dkeys, nd, nullptr, nslot, nullptr, nullptr,
                      nullptr, derr, s);
  CK(cudaGetLastError());
  std::vector<int32_t> cnt((size_t)nsl);
  CK(cudaMemcpyAsync(cnt.data(), nslot, sizeof(int32_t) * nsl, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<int64_t> sptr((size_t)nsl + 1, 0);
  for (int64_t i = 0; i < nsl; ++i) sptr[(size_t)i + 1] = sptr[(size_t)i] + cnt[(size_t)i];
  // off-diagonal entries: nnz - n (every row of the model Hamiltonians stores its diagonal)
  const double offd = std::max<double>(1.0, (double)h->nnz - (double)n);
  h->sw_fill = (double)sptr[(size_t)nsl] * 32.0 / offd;
  if (h->sw_fill > (b8 ? kSwMaxFill8 : kSwMaxFill) && !getenv("TE_SPMV_SW_FORCE")) {
    cleanup();
    return TE_OK;
  }
  const size_t vb = h->cplx ? 16 : 8;
  // Panel sweep (two passes; opt-in): TE_SPMV_SW_PANEL = log2 of the slices per panel (0 / unset: one
  // pass).  Measured on config 5 with panels of 2^15 slices (16 MB of x): DRAM traffic per SpMV
  // 14.0 -> 8.7 GB, time 2.96 -> 3.09 ms (the kernel is bound by load latency under L2 load, not by
  // DRAM bytes), whole bench unchanged (65.2 vs 65.3 Krylov steps/s) - hence not default.
  int sb = 0;
  while ((int64_t(1) << sb) < nsl) ++sb;
  int ka = 0;
  if (const char* e = getenv("TE_SPMV_SW_PANEL")) ka = std::max(0, atoi(e));
  if (ka >= sb) ka = 0;  // the whole x is one panel
  if (cudaMalloc(&h->d_sw_diag, vb * (n + 2)) != cudaSuccess || cudaMalloc(&h->d_sw_dict, vb * 256) != cudaSuccess) {
    cudaGetLastError();
    cleanup();
    free_sw(h);
    return TE_OK;  // no room: the CSR kernels stay
  }
  std::vector<double> vr(kd.size());
  for (size_t i = 0; i < kd.size(); ++i) vr[i] = kd[i].x;
  if (h->cplx) CK(cudaMemcpyAsync(h->d_sw_dict, kd.data(), sizeof(double2) * nd, cudaMemcpyHostToDevice, s));
  else CK(cudaMemcpyAsync(h->d_sw_dict, vr.data(), sizeof(double) * nd, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(h->d_sw_diag, 0, vb * (n + 2), s));
  // one pass of the build: slot counts -> slice pointers -> window bases and entries
  // (pass 0: every window; 1: windows inside the slice's panel, with the diagonal; 2: the others)
  auto build_pass = [&](int pass, int64_t** d_sptr, int32_t** d_base, uint16_t** d_ent, int64_t* nslots) -> int {
    if (pass != 0) {
      te::launch_sw_build(false, h->cplx, b8, pass, ka, n, h->d_rowptr, h->d_col, h->d_val, dkeys, nd, nullptr, nslot,
                          nullptr, nullptr, nullptr, derr, s);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(cnt.data(), nslot, sizeof(int32_t) * nsl, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int64_t i = 0; i < nsl; ++i) sptr[(size_t)i + 1] = sptr[(size_t)i] + cnt[(size_t)i];
    }
    const int64_t ns = sptr[(size_t)nsl];
    if (cudaMalloc(d_sptr, sizeof(int64_t) * (nsl + 1)) != cudaSuccess ||
        cudaMalloc(d_base, sizeof(int32_t) * (ns + 8)) != cudaSuccess ||
        cudaMalloc(d_ent, (b8 ? 1 : 2) * 32 * (size_t)(ns + 8)) != cudaSuccess) {
      cudaGetLastError();
      return -1;
    }
    CK(cudaMemcpyAsync(*d_sptr, sptr.data(), sizeof(int64_t) * (nsl + 1), cudaMemcpyHostToDevice, s));
    te::launch_sw_build(true, h->cplx, b8, pass, ka, n, h->d_rowptr, h->d_col, h->d_val, dkeys, nd, *d_sptr, nullptr, *d_base,
                        *d_ent, pass == 2 ? nullptr : h->d_sw_diag, derr, s);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));  // sptr (host) is reused by the next pass
    *nslots = ns;
    return TE_OK;
  };
  int64_t slots_a = 0, slots_b = 0;
  int rcb = build_pass(ka > 0 ? 1 : 0, &h->d_sw_sptr, &h->d_sw_base, &h->d_sw_ent, &slots_a);
  if (rcb == TE_OK && ka > 0) rcb = build_pass(2, &h->d_swb_sptr, &h->d_swb_base, &h->d_swb_ent, &slots_b);
  if (rcb > 0) { cleanup(); free_sw(h); return rcb; }
  if (rcb < 0) {
    cleanup();
    free_sw(h);
    return TE_OK;  // no room: the CSR kernels stay
  }
  int herr = 0;
  CK(cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  cleanup();
  if (herr) {
    free_sw(h);
    return set_err(TE_ERR_CUDA, "slot-window SELL build: value missing from the dictionary");
  }
  if (ka > 0) {  // pass 2 sweeps the slices with sw_ob slice bits from sw_lo upwards outermost
    h->sw_ka = ka;
    h->sw_sb = sb;
    h->sw_ob = sb - ka;
    h->sw_lo = std::max(0, ka - h->sw_ob - 2);
    if (const char* e = getenv("TE_SPMV_SW_PANEL_LO")) h->sw_lo = std::max(0, std::min(ka, atoi(e)));
    h->swb_slots = slots_b;
  }
  const int64_t slots = slots_a;
  h->sw_nslice = nsl;
  h->sw_slots = slots;
  h->sw_ndict = nd;
  h->sw_bits = b8 ? 8 : 16;
  return TE_OK;
}

int plan_xs(te_handle* h, const int64_t* rowptr) {
  free_xs(h);

  const int64_t n = h->n;
  const double avg = n > 0 ? (double)h->nnz / (double)n : 0.0;
  int tx = 1;  // measured (config 2): one lane per row beats 2 / 4 (larger tiles, longer x ranges)
  while (tx < 8 && 16.0 * tx < avg) tx <<= 1;
  if (const char* e = getenv("TE_SPMV_XS_TPR")) {
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8) tx = v;
  }
  h->spmv_xs_tpr = tx;
  h->xs_ecap = h->cplx ? 2048 : 4096;
  if (const char* e = getenv("TE_SPMV_XS_ECAP")) h->xs_ecap = std::max(64, std::min(8192, atoi(e)));
  h->xs_stages = 2;
  if (const char* e = getenv("TE_SPMV_XS_XPOL")) h->xs_xpol = atoi(e) != 0;
  if (const char* e = getenv("TE_SPMV_XS_NF")) h->xs_nf = atoi(e) == 16 ? 16 : 8;
  if (const char* e = getenv("TE_SPMV_XS_STAGES")) h->xs_stages = atoi(e) == 3 ? 3 : 2;
  h->xs_xcap = te::xs_xcap_for(h->cplx, tx, h->xs_ecap, te::kXsBudget, h->xs_stages);
  const int64_t rcap = 32 * te::kXsConsumers / tx;
  std::vector<int64_t> tg;
  int64_t st = 0;
  for (int64_t r = 0; r < n; ++r) {
    const bool over_rows = (r + 1 - st) > rcap;
    const bool over_nnz = (rowptr[r + 1] - rowptr[st]) > h->xs_ecap && r > st;
    if (over_rows || over_nnz) {
      tg.insert(tg.end(), {st, r, rowptr[st], rowptr[r]});
      st = r;
    }
  }
  if (n > 0) tg.insert(tg.end(), {st, n, rowptr[st], rowptr[n]});
  const int64_t nt = (int64_t)tg.size() / 4;
  if (nt == 0) return TE_OK;
  if (cudaMalloc(&h->d_tile_xs, sizeof(int64_t) * tg.size()) != cudaSuccess ||
      cudaMalloc(&h->d_xs_meta, sizeof(int4) * nt) != cudaSuccess ||
      cudaMalloc(&h->d_xs_rng, sizeof(int2) * nt * te::kXsRmax) != cudaSuccess ||
      cudaMalloc(&h->d_lcol, sizeof(uint16_t) * (h->nnz + 16)) != cudaSuccess) {
    cudaGetLastError();
    free_xs(h);
    return set_err(TE_ERR_OOM, "staged-x SpMV plan: out of device memory");
  }
  cudaStream_t s = h->stream ? h->stream : h->own_stream;
  CK(cudaMemcpyAsync(h->d_tile_xs, tg.data(), sizeof(int64_t) * tg.size(), cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(h->d_lcol, 0xFF, sizeof(uint16_t) * (h->nnz + 16), s));
  CK(cudaMemsetAsync(h->d_xs_rng, 0, sizeof(int2) * nt * te::kXsRmax, s));
  te::launch_xs_plan(h->d_tile_xs, nt, h->d_col, h->n, h->xs_xcap, te::kXsRmax, te::kXsGap, h->d_xs_meta, h->d_xs_rng,
                     h->d_lcol, s);
  CK(cudaGetLastError());
  std::vector<int4> meta((size_t)nt);
  CK(cudaMemcpyAsync(meta.data(), h->d_xs_meta, sizeof(int4) * nt, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  int64_t ng = 0, tg_glob = 0, nxs = 0;
  for (const int4& m : meta) {
    ng += m.z;
    tg_glob += m.z > 0;
    nxs += m.y;
  }
  h->ntiles_xs = nt;
  h->xs_global_frac = h->nnz > 0 ? (double)ng / (double)h->nnz : 0.0;
  h->xs_global_tiles = (double)tg_glob / (double)nt;
  h->xs_x_per_entry = h->nnz > 0 ? (double)nxs / (double)h->nnz : 0.0;
  return TE_OK;
}

// ---------------------------------------------------------------- creation
te_handle* create_common(int64_t n, const int64_t* rowptr, const int32_t* col, const void* val, bool cplx,
                         int64_t n_global, int64_t row_begin, te_dist* dist, bool herm_check, int64_t ncol_limit) {
  clear_err();
  if (n < 1 || !rowptr || (!col && rowptr[n] > 0) || (!val && rowptr[n] > 0)) {
    set_err(TE_ERR_ARG, "bad arguments (n=%lld)", (long long)n);
    return nullptr;
  }
  if (rowptr[0] != 0) {
    set_err(TE_ERR_CSR, "rowptr[0] != 0");
    return nullptr;
  }
  for (int64_t i = 0; i < n; ++i)
    if (rowptr[i + 1] < rowptr[i]) {
      set_err(TE_ERR_CSR, "rowptr decreases at row %lld", (long long)i);
      return nullptr;
    }
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
    cudaGetLastError();
    set_err(TE_ERR_CUDA, "no CUDA device available");
    return nullptr;
  }
  te_handle* h = new te_handle();
  h->dist = dist;
  h->n = n;
  h->n_global = n_global;
  h->row_begin = row_begin;
  h->cplx = cplx;
  h->nnz = rowptr[n];
  for (auto& p : h->prof) p = te_kernel_profile{0, 0.0, 0.0};
  auto fail = [&](int code, const char* what) -> te_handle* {
    if (g_status == TE_OK) set_err(code, "%s", what);
    te_destroy(h);
    return nullptr;
  };
  if (cudaGetDevice(&h->device) != cudaSuccess) return fail(TE_ERR_CUDA, "cudaGetDevice");
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
  // a blocking stream: work on it is ordered with the legacy default stream, so device vectors a
  // caller produced there (stream argument 0) are complete before the library reads them
  if (cudaStreamCreateWithFlags(&h->own_stream, cudaStreamDefault) != cudaSuccess)
    return fail(TE_ERR_CUDA, "cudaStreamCreate");
  h->stream = h->own_stream;
  if (te::configure_kernels() != cudaSuccess) return fail(TE_ERR_CUDA, "kernel shared-memory configuration failed");
  const size_t vb = cplx ? 16 : 8;
  // padded by a few entries: the TMA SpMV's bulk copies round ranges out to 16-byte boundaries
  if (cudaMalloc(&h->d_rowptr, sizeof(int64_t) * (n + 4)) != cudaSuccess) return fail(TE_ERR_OOM, "rowptr alloc");
  if (cudaMalloc(&h->d_col, sizeof(int32_t) * (h->nnz + 8)) != cudaSuccess) return fail(TE_ERR_OOM, "col alloc");
  if (cudaMalloc(&h->d_val, vb * (h->nnz + 4)) != cudaSuccess) return fail(TE_ERR_OOM, "val alloc");
  cudaMemsetAsync(h->d_rowptr, 0, sizeof(int64_t) * (n + 4), h->stream);
  cudaMemsetAsync(h->d_col, 0, sizeof(int32_t) * (h->nnz + 8), h->stream);
  cudaMemsetAsync(h->d_val, 0, vb * (h->nnz + 4), h->stream);
  cudaMemcpyAsync(h->d_rowptr, rowptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, h->stream);
  if (h->nnz > 0) {
    cudaMemcpyAsync(h->d_col, col, sizeof(int32_t) * h->nnz, cudaMemcpyHostToDevice, h->stream);
    cudaMemcpyAsync(h->d_val, val, vb * h->nnz, cudaMemcpyHostToDevice, h->stream);
  }
  if (ensure_workspace(h, 1) != TE_OK) return fail(TE_ERR_OOM, "workspace");
  {  // lanes per row of the pipelined SpMV: the smallest power of two (1..8) leaving <= 20 (real
     // values) / <= 8 (complex values, half-size tiles) entries per lane of a mean-length row;
     // gathers in flight per lane 16 when that share fits one round, else 12 (complex: 8).
     // Measured on configs 2-6.  TE_SPMV_TPR / TE_SPMV_NF_WIDE override.
    const double avg = n > 0 ? (double)h->nnz / (double)n : 0.0;
    const double per_lane = cplx ? 8.0 : 20.0;
    int t = 1;
    while (t < 8 && per_lane * t < avg) t <<= 1;
    if (const char* e = getenv("TE_SPMV_TPR")) {
      const int v = atoi(e);
      if (v == 1 || v == 2 || v == 4 || v == 8) t = v;
    }
    h->spmv_ring_tpr = t;
    h->spmv_nf_wide = !cplx && avg <= 16.0 * t;
    if (const char* e = getenv("TE_SPMV_NF_WIDE")) h->spmv_nf_wide = atoi(e) != 0;
    if (const char* e = getenv("TE_PROJ_CONST_R")) h->proj_const_r = atoi(e) != 0;
    // K3 on the TMA ring from 2^22 rows: config 5 (2^26) 6.10 -> 6.79 TB/s, config 4 (2^24) 6.19 -> 6.69;
    // below, the ring's fill and drain cost more than it gains (config 2, 2^20 rows: 6.16 -> 5.50)
    h->norm_tma = n >= (int64_t(1) << 22);
    if (const char* e = getenv("TE_NORM_TMA")) h->norm_tma = atoi(e) != 0;
    if (const char* e = getenv("TE_SPMV_FORCE_HALO")) h->spmv_force_halo = atoi(e) != 0;
  }
  {  // warp-specialised ring SpMV (variant 7, default) tiles: <= kSpmvTileNnz(C) entries and
     // <= 480/tpr rows, {first row, end row, first entry, end entry}; lanes per row by the same rule
     // as the pipelined SpMV (measured best on configs 2-6: 1 / 2 / 8 / 2 / 4)
    int tr = h->spmv_ring_tpr;
    if (const char* e = getenv("TE_SPMV_RING_TPR")) {
      const int v = atoi(e);
      if (v == 1 || v == 2 || v == 4 || v == 8) tr = v;
    }
    h->spmv_ring_tpr = tr;
    // ring depth: 4 stages of 4096 entries for short real rows (a deeper ring absorbs more
    // per-warp variance), else 3 stages of 5632 / 2816 (larger tiles); measured: config 2 +1 %
    // with 4 stages, configs 3 / 5 / 6 +2 / +2 / +5 % with 3
    const double avg = n > 0 ? (double)h->nnz / (double)n : 0.0;
    h->ring_stages = (!cplx && avg <= 16.0) ? 4 : 3;
    if (const char* e = getenv("TE_SPMV_RING_STAGES")) h->ring_stages = atoi(e) == 3 ? 3 : 4;
    const std::vector<int64_t> tg = ring_tiles(n, rowptr, cplx, h->ring_stages, h->spmv_ring_tpr);
    h->ntiles_ring = (int64_t)tg.size() / 4;
    if (!tg.empty()) {
      if (cudaMalloc(&h->d_tile_ring, sizeof(int64_t) * tg.size()) != cudaSuccess) return fail(TE_ERR_OOM, "tiles");
      cudaMemcpyAsync(h->d_tile_ring, tg.data(), sizeof(int64_t) * tg.size(), cudaMemcpyHostToDevice, h->stream);
      cudaStreamSynchronize(h->stream);
    }
  }
  // validation + ||H||_1 on the device
  int* d_err = reinterpret_cast<int*>(h->d_counter + 4);
  unsigned long long* d_norm = reinterpret_cast<unsigned long long*>(h->d_small + kOffScalar);
  cudaMemsetAsync(d_err, 0, sizeof(int), h->stream);
  cudaMemsetAsync(d_norm, 0, sizeof(unsigned long long), h->stream);
  // distributed handles: local columns >= n address the halo; the Hermiticity test needs the
  // global matrix and is skipped there (ranks validate structure only)
  te::CsrCheck cc{d_err, d_norm};
  te::launch_csr_check(n, ncol_limit, h->d_rowptr, h->d_col, h->d_val, cplx, herm_check, cc, h->stream);
  int herr = 0;
  unsigned long long nb = 0;
  cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, h->stream);
  cudaMemcpyAsync(&nb, d_norm, sizeof(nb), cudaMemcpyDeviceToHost, h->stream);
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) {
    set_err(TE_ERR_CUDA, "create: %s", cudaGetErrorString(e));
    return fail(TE_ERR_CUDA, "create");
  }
  cudaMemsetAsync(h->d_counter, 0, sizeof(unsigned) * 8, h->stream);
  if (herr & 1) return fail(TE_ERR_CSR, "column indices out of range or not strictly increasing within a row");
  if (herr & 2) return fail(TE_ERR_NOT_HERMITIAN, "matrix is not Hermitian (or has non-finite values)");
  double nrm;
  std::memcpy(&nrm, &nb, sizeof nrm);
  h->norm1 = nrm;
  h->ncol_limit = ncol_limit;
  {  // SpMV format chosen at create (measured per SpMV launch):
     // * slot-window SELL-32 (9) when the off-diagonal values fit the 8-bit dictionary and the
     //   slot padding stays below kSwMaxFill (spin chains: 2 bytes per entry, coalesced x windows);
     // * else the staged-x ring (8) when its plan stages >= 95 % of the entries and rows are short
     //   (mean <= 40 entries): staged-x vs ring, config 3 -5 %, config 6 (78 entries per row) +27 %,
     //   config 4 (half the columns uniform: 50 % global gathers) +190 %;
     // * else the warp-specialised ring (7).  TE_SPMV_DEFAULT overrides.
    const double avg = n > 0 ? (double)h->nnz / (double)n : 0.0;
    int def = 7;
    int want = 0;
    if (const char* e = getenv("TE_SPMV_DEFAULT")) {
      const int v = atoi(e);
      if (v == 6 || v == 7 || v == 8 || v == 9 || v == 10) want = v;
    }
    if (want == 0 || want == 9) {
      if (plan_sw(h) != TE_OK) return fail(TE_ERR_CUDA, "slot-window SELL build");
      if (h->sw_nslice > 0) def = 9;
    }
    if (def != 9 && (want == 0 || want == 8) && avg <= 40.0 && (n >= kXsMinRows || want == 8)) {
      if (plan_xs(h, rowptr) != TE_OK) return fail(TE_ERR_OOM, "staged-x plan");
      if (h->ntiles_xs > 0 && (h->xs_global_frac <= 0.05 || want == 8)) def = 8;
    }
    if (want == 6 || want == 7 || want == 10) def = want == 10 ? 7 : want;
    if (def != 8) free_xs(h);
    if (def != 9) free_sw(h);
    h->spmv_tiled = def == 6 ? 7 : def;
    if (def == 6 && build_sell(h) == TE_OK) h->spmv_tiled = 6;
    // * the ring over column blocks (10) when x outgrows L2 (16 n > kColBlkMinX) on a single rank:
    //   each pass gathers from one L2-resident 2^22-column block of x instead of DRAM
    const char* cbe = getenv("TE_SPMV_COLBLK");
    if ((h->spmv_tiled == 7 && want == 0 && 16.0 * (double)n > kColBlkMinX && !(cbe && atoi(cbe) == 0)) || want == 10) {
      if (build_colblk(h, colblk_cols(n)) != TE_OK) return fail(TE_ERR_CUDA, "column-blocked copy");
      if (!h->cb.empty()) h->spmv_tiled = 10;
    }
  }
  h->launches += 1;
  return h;
}

}  // namespace

// ==========================================================================================
// C ABI
// ==========================================================================================
extern "C" {

int te_kernel_attributes(int which, int* regs, int* max_threads, int* static_smem, int* max_dyn_smem) {
  clear_err();
  if (!regs || !max_threads || !static_smem || !max_dyn_smem) return set_err(TE_ERR_ARG, "null");
  te::configure_kernels();
  const int r = te::kernel_attributes(which, regs, max_threads, static_smem, max_dyn_smem);
  if (r == -1) return set_err(TE_ERR_ARG, "unknown kernel %d", which);
  if (r != 0) return set_err(TE_ERR_CUDA, "cudaFuncGetAttributes failed");
  return TE_OK;
}

int te_last_status(void) { return g_status; }
const char* te_last_error(void) { return g_msg.c_str(); }
const char* te_version(void) { return "timeevolver-b200 0.1 (sm_100a)"; }

te_handle* te_create_csr(int64_t n, const int64_t* rowptr, const int32_t* col, const te_c128* val) {
  return create_common(n, rowptr, col, val, true, n, 0, nullptr, true, n);
}

te_handle* te_create_csr_real(int64_t n, const int64_t* rowptr, const int32_t* col, const double* val) {
  return create_common(n, rowptr, col, val, false, n, 0, nullptr, true, n);
}

void te_destroy(te_handle* h) {
  if (!h) return;
  if (h->stream) cudaStreamSynchronize(h->stream);
  cudaFree(h->d_rowptr);
  cudaFree(h->d_col);
  cudaFree(h->d_val);
  free_workspace(h);
  cudaFree(h->d_small);
  cudaFree(h->d_g);
  cudaFree(h->d_G);
  cudaFree(h->d_part);
  cudaFree(h->d_partn);
  cudaFree(h->d_counter);
  cudaFree(h->d_halo);
  cudaFree(h->d_hrow);
  cudaFree(h->d_hrowptr);
  cudaFree(h->d_hcol);
  cudaFree(h->d_hval);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
  cudaFree(h->d_halo_owner);
  cudaFree(h->d_halo_lidx);
  cudaFree(h->d_peer_base);
  cudaFree(h->d_peer_ldv);
  for (void* p : h->ipc_open) cudaIpcCloseMemHandle(p);
  cudaFree(h->d_tile_ring);
  free_xs(h);
  free_sw(h);
  free_colblk(h);
  cudaFree(h->d_scol);
  cudaFree(h->d_sval);
  cudaFree(h->d_sptr);
  cudaFree(h->d_slen);
  cudaFree(h->d_sperm);
  cudaFree(h->d_sendbuf);
  cudaFree(h->d_send_idx);
  if (h->h_small) cudaFreeHost(h->h_small);
  if (h->h_coef) cudaFreeHost(h->h_coef);
  if (h->ev_ready) {
    for (int i = 0; i < kEvPool; ++i) {
      cudaEventDestroy(h->ev0[i]);
      cudaEventDestroy(h->ev1[i]);
    }
    cudaEventDestroy(h->evk0);
    cudaEventDestroy(h->evk1);
  }
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
}

static int evolve_entry(te_handle* h, const void* v0, bool v0_dev, double t, double tol, int m_max, void* vout,
                        bool vout_dev, te_stats* st, cudaStream_t stream, const double* forced, int64_t nforced,
                        const Sampling* smp = nullptr) {
  clear_err();
  int rc = check_evolve_args(h, t, tol, m_max);
  if (rc) return rc;
  if (!v0 || !vout) return set_err(TE_ERR_ARG, "null vector");
  if (cudaSetDevice(h->device) != cudaSuccess) return set_err(TE_ERR_CUDA, "cudaSetDevice");
  h->stream = stream ? stream : h->own_stream;
  const int m = (int)std::min<int64_t>(m_max, h->n_global);
  if ((rc = ensure_workspace(h, std::max(m, 1)))) return rc;
  const size_t vbytes = sizeof(double2) * (size_t)h->n;
  CK(cudaMemcpyAsync(h->d_V, v0, vbytes, v0_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
  rc = evolve_core(h, t, tol, m_max, forced, nforced, st, smp);
  if (rc) {
    cudaStreamSynchronize(h->stream);
    h->stream = h->own_stream;
    return rc;
  }
  CK(cudaMemcpyAsync(vout, h->d_V, vbytes, vout_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->stream = h->own_stream;
  return TE_OK;
}

int te_evolve(te_handle* h, const te_c128* v0, double t, double tol, int m_max, te_c128* v_out, te_stats* stats) {
  return evolve_entry(h, v0, false, t, tol, m_max, v_out, false, stats, nullptr, nullptr, 0);
}

int te_evolve_dev(te_handle* h, const void* d_v0, double t, double tol, int m_max, void* d_vout, te_stats* stats,
                  void* stream) {
  return evolve_entry(h, d_v0, true, t, tol, m_max, d_vout, true, stats, static_cast<cudaStream_t>(stream), nullptr,
                      0);
}

int te_evolve_schedule(te_handle* h, const te_c128* v0, int64_t k, const double* t_steps, double tol, int m_max,
                       te_c128* v_out, te_stats* stats) {
  if (k < 0 || (k > 0 && !t_steps)) return set_err(TE_ERR_ARG, "bad schedule");
  double t = 0.0;
  for (int64_t i = 0; i < k; ++i) {
    if (!(t_steps[i] > 0.0) || !std::isfinite(t_steps[i])) return set_err(TE_ERR_ARG, "schedule steps must be > 0");
    t += t_steps[i];
  }
  return evolve_entry(h, v0, false, t, tol, m_max, v_out, false, stats, nullptr, t_steps, k);
}

int te_evolve_sampled(te_handle* h, const te_c128* v0, double t, double tol, int m_max, int64_t n_samples,
                      const double* sample_times, te_c128* samples_out, double* sample_bounds, te_c128* v_out,
                      te_stats* stats) {
  clear_err();
  if (n_samples < 0 || (n_samples > 0 && (!sample_times || !samples_out)))
    return set_err(TE_ERR_ARG, "bad sampling arguments");
  for (int64_t i = 0; i < n_samples; ++i) {
    if (!(sample_times[i] >= 0.0) || sample_times[i] > t || (i > 0 && sample_times[i] < sample_times[i - 1]))
      return set_err(TE_ERR_ARG, "sample times must be ascending and within [0, t]");
  }
  Sampling s;
  s.n = n_samples;
  s.times = sample_times;
  s.out = samples_out;
  s.bounds = sample_bounds;
  return evolve_entry(h, v0, false, t, tol, m_max, v_out, false, stats, nullptr, nullptr, 0, &s);
}

int64_t te_get_schedule(const te_handle* h, int64_t cap, double* t_steps, int32_t* m_eff, double* err_steps) {
  if (!h) return -TE_ERR_ARG;
  const int64_t k = (int64_t)h->sched.size();
  for (int64_t i = 0; i < std::min(cap, k); ++i) {
    if (t_steps) t_steps[i] = h->sched[i].tau;
    if (m_eff) m_eff[i] = h->sched[i].m_eff;
    if (err_steps) err_steps[i] = h->sched[i].err;
  }
  return k;
}

int te_krylov_basis(te_handle* h, const te_c128* v1, int m, double tol_rate, double* alpha, double* beta,
                    int* m_eff, int* breakdown, te_c128* V_out) {
  clear_err();
  if (!h || !v1 || !alpha || !beta || !m_eff) return set_err(TE_ERR_ARG, "null argument");
  if (m < 1 || m > TE_M_MAX) return set_err(TE_ERR_ARG, "m must be in [1, %d]", TE_M_MAX);
  if (cudaSetDevice(h->device) != cudaSuccess) return set_err(TE_ERR_CUDA, "cudaSetDevice");
  h->stream = h->own_stream;
  m = (int)std::min<int64_t>(m, h->n_global);
  int rc = ensure_workspace(h, m);
  if (rc) return rc;
  CK(cudaMemcpyAsync(h->d_V, v1, sizeof(double2) * h->n, cudaMemcpyHostToDevice, h->stream));
  if ((rc = run_arnoldi(h, m, tol_rate))) return rc;
  bool brk = false;
  int me = 0;
  if ((rc = read_flag(h, m, &me, &brk))) return rc;
  *m_eff = me;
  if (breakdown) *breakdown = brk ? 1 : 0;
  for (int q = 0; q < m; ++q) {
    alpha[q] = q < me ? h->h_small[kOffAlpha + q] : 0.0;
    beta[q] = q < me ? h->h_small[kOffBeta + q] : 0.0;
  }
  if (V_out) {
    std::vector<double2> col(h->n);
    for (int q = 0; q < me; ++q) {
      CK(cudaMemcpy(col.data(), h->d_V + (int64_t)q * h->ldv, sizeof(double2) * h->n, cudaMemcpyDeviceToHost));
      const double s = q == 0 ? 1.0 : 1.0 / h->h_small[kOffBeta + q - 1];
      for (int64_t i = 0; i < h->n; ++i) {
        V_out[(size_t)q * h->n + i].re = col[i].x * s;
        V_out[(size_t)q * h->n + i].im = col[i].y * s;
      }
    }
  }
  return TE_OK;
}

// SELL-32-sigma copy of the (local) CSR for SpMV variant 6: rows sorted by length (descending,
// stable) inside windows of kSellSigma rows, slices of 32 rows padded to the slice width and
// stored column-major; built by a device scatter from the device CSR.  Refused (TE_ERR_ARG) when
// padding would exceed the CSR's entry count (a few very long rows).
static int build_sell(te_handle* h) {
  if (h->nslices > 0 || h->n == 0) return TE_OK;
  const int64_t n = h->n;
  std::vector<int64_t> rp((size_t)n + 1);
  if (cudaMemcpy(rp.data(), h->d_rowptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost) != cudaSuccess)
    return set_err(TE_ERR_CUDA, "SELL: rowptr copy");
  const int64_t nsl = (n + 31) / 32;
  std::vector<int32_t> perm((size_t)nsl * 32, -1);
  std::vector<int32_t> idx;
  for (int64_t w0 = 0; w0 < n; w0 += te::kSellSigma) {
    const int64_t w1 = std::min<int64_t>(n, w0 + te::kSellSigma);
    idx.resize((size_t)(w1 - w0));
    for (int64_t r = w0; r < w1; ++r) idx[(size_t)(r - w0)] = (int32_t)r;
    std::stable_sort(idx.begin(), idx.end(),
                     [&](int32_t x, int32_t y) { return rp[x + 1] - rp[x] > rp[y + 1] - rp[y]; });
    std::copy(idx.begin(), idx.end(), perm.begin() + w0);
  }
  std::vector<int64_t> sptr((size_t)nsl + 1, 0);
  std::vector<int32_t> slen((size_t)nsl, 0);
  for (int64_t s = 0; s < nsl; ++s) {
    int64_t w = 0;
    for (int l = 0; l < 32; ++l) {
      const int32_t r = perm[(size_t)(s * 32 + l)];
      if (r >= 0) w = std::max<int64_t>(w, rp[r + 1] - rp[r]);
    }
    if (w > INT32_MAX) return set_err(TE_ERR_ARG, "SELL: row too long");
    slen[(size_t)s] = (int32_t)w;
    sptr[(size_t)s + 1] = sptr[(size_t)s] + 32 * w;
  }
  const int64_t total = sptr[(size_t)nsl];
  if (total > 2 * h->nnz + 32 * 64)
    return set_err(TE_ERR_ARG, "SELL: padding %lld entries for %lld nonzeros (rows too uneven)", (long long)total,
                   (long long)h->nnz);
  const size_t vb = h->cplx ? 16 : 8;
  auto fail = [&](const char* what) {
    cudaFree(h->d_scol); cudaFree(h->d_sval); cudaFree(h->d_sptr); cudaFree(h->d_slen); cudaFree(h->d_sperm);
    h->d_scol = nullptr; h->d_sval = nullptr; h->d_sptr = nullptr; h->d_slen = nullptr; h->d_sperm = nullptr;
    return set_err(TE_ERR_OOM, "SELL: %s", what);
  };
  if (cudaMalloc(&h->d_scol, sizeof(int32_t) * std::max<int64_t>(1, total)) != cudaSuccess) return fail("col");
  if (cudaMalloc(&h->d_sval, vb * std::max<int64_t>(1, total)) != cudaSuccess) return fail("val");
  if (cudaMalloc(&h->d_sptr, sizeof(int64_t) * (nsl + 1)) != cudaSuccess) return fail("ptr");
  if (cudaMalloc(&h->d_slen, sizeof(int32_t) * nsl) != cudaSuccess) return fail("len");
  if (cudaMalloc(&h->d_sperm, sizeof(int32_t) * nsl * 32) != cudaSuccess) return fail("perm");
  cudaMemcpyAsync(h->d_sptr, sptr.data(), sizeof(int64_t) * (nsl + 1), cudaMemcpyHostToDevice, h->stream);
  cudaMemcpyAsync(h->d_slen, slen.data(), sizeof(int32_t) * nsl, cudaMemcpyHostToDevice, h->stream);
  cudaMemcpyAsync(h->d_sperm, perm.data(), sizeof(int32_t) * nsl * 32, cudaMemcpyHostToDevice, h->stream);
  te::launch_sell_build(h->cplx, nsl * 32, h->d_rowptr, h->d_col, h->d_val, h->d_sperm, h->d_sptr, h->d_slen,
                        h->d_scol, h->d_sval, h->stream);
  const cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return fail(cudaGetErrorString(e));
  h->nslices = nsl;
  return TE_OK;
}

int te_set_option(te_handle* h, int option, double value) {
  clear_err();
  if (!h) return set_err(TE_ERR_ARG, "null handle");
  switch (option) {
    case TE_OPT_PROFILE:
      h->profile = value != 0.0;
      for (auto& p : h->prof) p = te_kernel_profile{0, 0.0, 0.0};
      h->ev_used = 0;
      return TE_OK;
    case TE_OPT_GRAPH:
      h->use_graph = value != 0.0;
      return TE_OK;
    case TE_OPT_KERNELS:
      if (value != 2.0 && value != 3.0 && value != 5.0)
        return set_err(TE_ERR_ARG, "TE_OPT_KERNELS must be 2 (hybrid), 3 (TMA ring) or 5 (register accumulators)");
      h->variant = (int)value;
      return TE_OK;
    case TE_OPT_ORTHO:
      if (value != 0.0 && value != 1.0 && value != 2.0)
        return set_err(TE_ERR_ARG, "TE_OPT_ORTHO must be 0 (CGS2), 1 (Lanczos) or 2 (CGS2, Gram second sweep)");
      h->ortho = (int)value;
      return TE_OK;
    case TE_OPT_HALO:
      if (value != 0.0 && value != 1.0) return set_err(TE_ERR_ARG, "TE_OPT_HALO must be 0 (NCCL exchange) or 1 (peer loads)");
      h->halo_mode = (int)value;
      return TE_OK;
    case TE_OPT_INTEGRATOR:
      if (value != 0.0 && value != 1.0) return set_err(TE_ERR_ARG, "TE_OPT_INTEGRATOR must be 0 or 1");
      h->integrator = (int)value;
      return TE_OK;
    case TE_OPT_SPMV:
      if (value != 6.0 && value != 7.0 && value != 8.0 && value != 9.0 && value != 10.0)
        return set_err(TE_ERR_ARG, "TE_OPT_SPMV must be 10 (column-blocked ring), 9 (slot-window SELL-32), 8 (staged-x ring), "
                                   "7 (ring) or 6 (SELL-32-sigma)");
      if (value == 10.0 && h->cb.empty()) {
        const int rc = build_colblk(h, colblk_cols(h->n));
        if (rc != TE_OK) return rc;
        if (h->cb.empty())
          return set_err(TE_ERR_ARG, "TE_OPT_SPMV 10: not applicable (x fits one column block, halo columns, or no memory)");
      }
      if (value == 6.0) {
        const int rc = build_sell(h);
        if (rc != TE_OK) return rc;
      }
      if (value == 9.0 && h->sw_nslice == 0) {
        const int rc = plan_sw(h);
        if (rc != TE_OK) return rc;
        if (h->sw_nslice == 0)
          return set_err(TE_ERR_ARG, "TE_OPT_SPMV 9: not applicable to this matrix (more than 255 distinct off-diagonal values, "
                                     "halo columns, or slot padding %.2f above the limit 1.6 (16-bit) / 2.0 (8-bit))", h->sw_fill);
      }
      if (value == 8.0 && h->ntiles_xs == 0) {
        std::vector<int64_t> rp((size_t)h->n + 1);
        if (cudaMemcpy(rp.data(), h->d_rowptr, sizeof(int64_t) * (h->n + 1), cudaMemcpyDeviceToHost) != cudaSuccess)
          return set_err(TE_ERR_CUDA, "staged-x plan: rowptr copy");
        const int rc = plan_xs(h, rp.data());
        if (rc != TE_OK) return rc;
      }
      h->spmv_tiled = (int)value;
      return TE_OK;
    case TE_OPT_PREFETCH:
      if (value < 0 || value > 16) return set_err(TE_ERR_ARG, "TE_OPT_PREFETCH must be in [0, 16]");
      h->prefetch = (int)value;
      return TE_OK;
    default:
      return set_err(TE_ERR_ARG, "unknown option %d", option);
  }
}

int te_get_option(const te_handle* h, int option, double* value) {
  clear_err();
  if (!h || !value) return set_err(TE_ERR_ARG, "null argument");
  switch (option) {
    case TE_OPT_PROFILE: *value = h->profile ? 1.0 : 0.0; return TE_OK;
    case TE_OPT_GRAPH: *value = h->use_graph ? 1.0 : 0.0; return TE_OK;
    case TE_OPT_KERNELS: *value = h->variant; return TE_OK;
    case TE_OPT_PREFETCH: *value = h->prefetch; return TE_OK;
    case TE_OPT_SPMV: *value = h->spmv_tiled; return TE_OK;
    case TE_OPT_ORTHO: *value = h->ortho; return TE_OK;
    case TE_OPT_INTEGRATOR: *value = h->integrator; return TE_OK;
    case TE_OPT_HALO: *value = h->halo_mode; return TE_OK;
    case TE_INFO_XS_GLOBAL: *value = h->ntiles_xs > 0 ? h->xs_global_frac : -1.0; return TE_OK;
    case TE_INFO_XS_GLOBAL_TILES: *value = h->ntiles_xs > 0 ? h->xs_global_tiles : -1.0; return TE_OK;
    case TE_INFO_XS_X_PER_ENTRY: *value = h->ntiles_xs > 0 ? h->xs_x_per_entry : -1.0; return TE_OK;
    case TE_INFO_SW_FILL: *value = h->sw_fill > 0.0 ? h->sw_fill : -1.0; return TE_OK;
    case TE_INFO_SW_PANEL: *value = h->sw_nslice > 0 ? (double)h->sw_ka : -1.0; return TE_OK;
    case TE_INFO_SW_FAR:
      *value = h->sw_nslice > 0 ? (double)h->swb_slots / (double)std::max<int64_t>(1, h->sw_slots + h->swb_slots) : -1.0;
      return TE_OK;
    default: return set_err(TE_ERR_ARG, "unknown option %d", option);
  }
}

int te_get_profile(const te_handle* h, int kernel, te_kernel_profile* out) {
  if (!h || !out || kernel < 0 || kernel >= kProfKernels) return set_err(TE_ERR_ARG, "bad arguments");
  *out = h->prof[kernel];
  return TE_OK;
}

int64_t te_launch_count(const te_handle* h) { return h ? h->launches : -1; }

int te_small_eig(int m, const double* alpha, const double* beta, double* lam, double* U) {
  clear_err();
  if (m < 1 || m > TE_M_MAX || !alpha || (m > 1 && !beta) || !lam || !U) return set_err(TE_ERR_ARG, "bad arguments");
  te::SmallEig E;
  if (!te::tridiag_eig(m, alpha, beta, E)) return set_err(TE_ERR_NUMERICAL, "tridiagonal eigensolver did not converge");
  for (int k = 0; k < m; ++k) lam[k] = E.lam[(size_t)k];
  for (size_t i = 0; i < (size_t)m * m; ++i) U[i] = E.U[i];
  return TE_OK;
}

int te_step_search(int m, const double* alpha, const double* beta, double h, int breakdown, int first,
                   double tau_prev, double rem, double tol_rate, double t_total, int integrator, double* tau,
                   double* err, int* quad_ok) {
  clear_err();
  if (m < 1 || m > TE_M_MAX || !alpha || (m > 1 && !beta) || !tau || !err) return set_err(TE_ERR_ARG, "bad arguments");
  te::SmallEig E;
  if (!te::tridiag_eig(m, alpha, beta, E)) return set_err(TE_ERR_NUMERICAL, "tridiagonal eigensolver did not converge");
  E.h = h;
  const te::StepResult r = te::find_step(E, breakdown != 0, first != 0, tau_prev, rem, tol_rate, t_total, integrator);
  if (r.collapse) return set_err(TE_ERR_STEP_COLLAPSE, "step size collapsed below 1e-13 t");
  *tau = r.tau;
  *err = r.err;
  if (quad_ok) *quad_ok = r.quad_ok ? 1 : 0;
  return TE_OK;
}
double te_one_norm(const te_handle* h) { return h ? h->norm1 : -1.0; }

// ------------------------------------------------------------------------------------------
// distributed
// ------------------------------------------------------------------------------------------
int te_nccl_unique_id(void* out128) {
  clear_err();
  if (!out128) return set_err(TE_ERR_ARG, "null");
  if (!te::nccl().ok) return set_err(TE_ERR_NCCL, "NCCL library not available: %s", te::nccl().err.c_str());
  ncclUniqueId id;
  CKN(te::nccl().GetUniqueId(&id));
  std::memcpy(out128, &id, sizeof id);
  return TE_OK;
}

te_dist* te_dist_init(int nranks, int rank, const void* id128) {
  clear_err();
  if (nranks < 1 || rank < 0 || rank >= nranks || !id128) {
    set_err(TE_ERR_ARG, "bad arguments");
    return nullptr;
  }
  te_dist* d = new te_dist();
  d->nranks = nranks;
  d->rank = rank;
  if (nranks > 1) {
    if (!te::nccl().ok) {
      set_err(TE_ERR_NCCL, "NCCL library not available: %s", te::nccl().err.c_str());
      delete d;
      return nullptr;
    }
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    ncclResult_t r = te::nccl().CommInitRank(&d->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      set_err(TE_ERR_NCCL, "ncclCommInitRank: %s", te::nccl().GetErrorString(r));
      delete d;
      return nullptr;
    }
  }
  return d;
}

void te_dist_destroy(te_dist* d) {
  if (!d) return;
  if (d->comm) te::nccl().CommDestroy(d->comm);
  delete d;
}

}  // extern "C"

// halo plan + distributed create live in dist.cpp
te_handle* te_internal_create_local(int64_t n_loc, int64_t n_global, int64_t row_begin, const int64_t* rowptr,
                                    const int32_t* col_local, const void* val, bool cplx, te_dist* dist,
                                    int64_t ncol_limit) {
  return create_common(n_loc, rowptr, col_local, val, cplx, n_global, row_begin, dist, false, ncol_limit);
}
ncclComm_t te_internal_comm(te_dist* d) { return d->comm; }
int te_internal_nranks(te_dist* d) { return d->nranks; }
int te_internal_rank(te_dist* d) { return d->rank; }

struct HaloCsr {
  std::vector<int32_t> rows;
  std::vector<int64_t> rowptr;
  std::vector<int32_t> col;
  std::vector<unsigned char> val;
};
int te_internal_setup_halo(te_handle* h, int64_t n_halo, const std::vector<int64_t>& recv_counts,
                           const std::vector<int64_t>& send_counts, const std::vector<int32_t>& send_idx,
                           double norm1_global, const std::vector<int64_t>& halo_global,
                           const std::vector<int64_t>& row_starts, const HaloCsr& hc) {
  h->n_halo = n_halo;
  h->nh = (int64_t)hc.rows.size();
  h->nh_entries = (int64_t)hc.col.size();
  if (h->nh > 0) {
    CK(cudaMalloc(&h->d_hrow, sizeof(int32_t) * h->nh));
    CK(cudaMalloc(&h->d_hrowptr, sizeof(int64_t) * (h->nh + 1)));
    CK(cudaMalloc(&h->d_hcol, sizeof(int32_t) * std::max<int64_t>(1, h->nh_entries)));
    CK(cudaMalloc(&h->d_hval, std::max<size_t>(16, hc.val.size())));
    CK(cudaMemcpy(h->d_hrow, hc.rows.data(), sizeof(int32_t) * h->nh, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->d_hrowptr, hc.rowptr.data(), sizeof(int64_t) * (h->nh + 1), cudaMemcpyHostToDevice));
    if (h->nh_entries > 0) {
      CK(cudaMemcpy(h->d_hcol, hc.col.data(), sizeof(int32_t) * h->nh_entries, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(h->d_hval, hc.val.data(), hc.val.size(), cudaMemcpyHostToDevice));
    }
  }
  if (h->dist && h->dist->nranks > 1) {
    CK(cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    if (const char* e = getenv("TE_COMM_SMS")) h->comm_sms = std::max(0, std::min(h->num_sms - 1, atoi(e)));
  }
  if (n_halo > 0) {  // owner rank and owner-local row of every halo entry (halo mode 1)
    std::vector<int32_t> own((size_t)n_halo), lidx((size_t)n_halo);
    int64_t k = 0;
    for (int q = 0; q < (int)recv_counts.size(); ++q)
      for (int64_t i = 0; i < recv_counts[q]; ++i, ++k) {
        own[(size_t)k] = q;
        lidx[(size_t)k] = (int32_t)(halo_global[(size_t)k] - row_starts[(size_t)q]);
      }
    CK(cudaMalloc(&h->d_halo_owner, sizeof(int32_t) * n_halo));
    CK(cudaMalloc(&h->d_halo_lidx, sizeof(int32_t) * n_halo));
    CK(cudaMemcpy(h->d_halo_owner, own.data(), sizeof(int32_t) * n_halo, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->d_halo_lidx, lidx.data(), sizeof(int32_t) * n_halo, cudaMemcpyHostToDevice));
  }
  h->recv_counts = recv_counts;
  h->send_counts = send_counts;
  h->n_send = (int64_t)send_idx.size();
  h->norm1 = norm1_global;
  if (n_halo > 0) CK(cudaMalloc(&h->d_halo, sizeof(double2) * n_halo));
  if (h->n_send > 0) {
    CK(cudaMalloc(&h->d_sendbuf, sizeof(double2) * h->n_send));
    CK(cudaMalloc(&h->d_send_idx, sizeof(int32_t) * h->n_send));
    CK(cudaMemcpy(h->d_send_idx, send_idx.data(), sizeof(int32_t) * h->n_send, cudaMemcpyHostToDevice));
  }
  return TE_OK;
}

int te_internal_set_error(int code, const char* msg) { return set_err(code, "%s", msg); }
cudaStream_t te_internal_stream(te_handle* h) { return h->own_stream; }
double te_internal_local_norm1(te_handle* h) { return h->norm1; }
void te_internal_set_norm1(te_handle* h, double v) { h->norm1 = v; }
