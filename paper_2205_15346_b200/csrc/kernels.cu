// Hot-path CUDA kernels for sm_100a: one Arnoldi/CGS2 step (Eq. 8, with the
// classical Gram-Schmidt + one re-orthogonalisation reading C1 of DESIGN.md) in three
// HBM-streaming launches, plus the restart assembly V.omega (Eq. 11).
//
//   K1 k_spmv_proj   p = s_j H V_j (CSR, entries staged through shared memory), then the
//                    sweep-1 projections g1_k = sum_i conj(V_ik) p_i, k <= j, in the epilogue
//   K2 k_update_proj p' = p - sum_k V_k e1_k  and  g2_k = sum_i conj(V_ik) p'_i : each V tile is
//                    staged ONCE in shared memory by cp.async.bulk (TMA bulk engine) through a
//                    4-stage mbarrier pipeline and used by both phases -> one HBM pass over V
//   K3 k_update_norm p'' = p' - sum_k V_k e2_k written as column j+1, and ||p''||^2
//   K4 k_combine     w = sum_k V_k (s_k omega_k), in place into column 0
// with e_k = s_k^2 g_k (s_k = 1/||V_k||: columns are stored unnormalised and scaled on the
// fly).  Reductions are deterministic: per-CTA partials in registers/shared memory, then the
// last CTA to finish (atomic ticket, integer only) sums the partials in a fixed order.
// No floating-point atomics anywhere.
#include "kernels.cuh"

#include <cuda.h>
#include <cstdio>
#include <utility>
#include <vector>

namespace te {

// --------------------------------------------------------------------------------------
// small helpers
// --------------------------------------------------------------------------------------
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
// a*b
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// conj(a)*b + c
__device__ __forceinline__ double2 cfma_conj(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.x, b.y, fma(-a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_cg(const double2* p) { return __ldcg(p); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "TE_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra TE_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// bulk (non-tensor) TMA copy global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// bulk L2 prefetch of a contiguous global range (no registers, no shared memory)
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// prefetch an arbitrary byte range, widened to 16-byte alignment
__device__ __forceinline__ void prefetch_range(const void* base, size_t begin, size_t end) {
  if (end <= begin) return;
  const uintptr_t a = ((uintptr_t)base + begin) & ~(uintptr_t)15;
  const uintptr_t b = ((uintptr_t)base + end + 15) & ~(uintptr_t)15;
  prefetch_l2((const void*)a, (unsigned)(b - a));
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Warp butterfly sum (all lanes end with the same, deterministic value).
__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
  }
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Step-j prologue shared by K1 (and the finalize kernel): decides from ||p''_{j-1}||^2 whether the
// recurrence continues (Alg. 1, breakdown threshold tol_rate, reading C6/C7).
// Returns the column scale s_j (0 => stop).  Only block 0 writes device state.
__device__ __forceinline__ double step_gate(const KDev& d, int j, bool writer) {
  if (d.flag[0] != 0) return 0.0;
  if (j == 0) {
    if (writer && d.ortho == 2) d.G[0] = make_double2(1.0, 0.0);
    return 1.0;
  }
  const double b = sqrt(d.nrm2[j - 1]);
  if (!isfinite(b)) {
    if (writer) { d.beta[j - 1] = b; d.flag[1] = j; d.flag[0] = 2; }
    return 0.0;
  }
  if (b < d.tol_rate) {                  // lucky breakdown: m_eff = j, h = beta_{j-1}
    if (writer) { d.beta[j - 1] = b; d.flag[1] = j; d.flag[0] = 1; }
    return 0.0;
  }
  const double sj = 1.0 / b;
  if (writer) {
    d.beta[j - 1] = b;
    d.s[j] = sj;
    if (d.ortho == 2) {  // f2: Gram row j from the dots of the pass that produced V_j
      for (int k = 0; k < j; ++k) {
        const double sk = d.s[k] * sj;
        const double2 g = d.g2[k];
        d.G[k * kMaxCols + j] = make_double2(sk * g.x, sk * g.y);
        d.G[j * kMaxCols + k] = make_double2(sk * g.x, -sk * g.y);
      }
      d.G[j * kMaxCols + j] = make_double2(1.0, 0.0);
    }
  }
  return sj;
}

// Per-CTA column partials -> global; the last CTA sums them in fixed block order.
// acc[q] holds column k = warp + kWarps*q summed over this thread's rows.
template <int NCW>
__device__ __forceinline__ void finish_columns(const KDev& d, double2 (&acc)[NCW], int ncols, int ctr,
                                               double2* out) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int q = 0; q < NCW; ++q) {
    const int k = warp + kWarps * q;
    double2 v = warp_sum(acc[q]);
    if (lane == 0 && k < ncols) d.part[(size_t)blockIdx.x * kMaxCols + k] = v;
  }
  __threadfence();
  __syncthreads();
  __shared__ int last;
  if (tid == 0) last = (atomicAdd(&d.counter[ctr], 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // 4 segments per column (tid/64), each summed sequentially, then combined in order
  __shared__ double2 seg[4][kMaxCols];
  const int c = tid & (kMaxCols - 1), sgi = tid >> 6;
  const int G = gridDim.x;
  const int per = (G + 3) / 4;
  double2 s = make_double2(0.0, 0.0);
  if (c < ncols) {
    const int b0 = sgi * per, b1 = min(G, b0 + per);
    for (int b = b0; b < b1; ++b) s = cadd(s, ld_cg(d.part + (size_t)b * kMaxCols + c));
  }
  seg[sgi][c] = s;
  __syncthreads();
  if (tid < ncols) {
    double2 t = seg[0][tid];
    t = cadd(t, seg[1][tid]);
    t = cadd(t, seg[2][tid]);
    t = cadd(t, seg[3][tid]);
    out[tid] = t;
  }
  if (tid == 0) d.counter[ctr] = 0u;
}

__device__ __forceinline__ void finish_scalar(const KDev& d, double v, int ctr, double* out) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __shared__ double ws[kWarps];
  v = warp_sum(v);
  if (lane == 0) ws[warp] = v;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kWarps; ++w) t += ws[w];
    d.partn[blockIdx.x] = t;
  }
  __threadfence();
  __syncthreads();
  __shared__ int last;
  if (tid == 0) last = (atomicAdd(&d.counter[ctr], 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double seg[kThreads];
  const int G = gridDim.x;
  const int per = (G + kThreads - 1) / kThreads;
  double s = 0.0;
  const int b0 = tid * per, b1 = min(G, b0 + per);
  for (int b = b0; b < b1; ++b) s += __ldcg(d.partn + b);
  seg[tid] = s;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int i = 0; i < kThreads; ++i) t += seg[i];
    *out = t;
    d.counter[ctr] = 0u;
  }
}

// --------------------------------------------------------------------------------------
// K1: SpMV + sweep-1 projections
// --------------------------------------------------------------------------------------
template <bool CPLX>
struct ValT;
template <>
struct ValT<false> {
  using T = double;
  static __device__ __forceinline__ double2 mul(double v, double2 x) { return make_double2(v * x.x, v * x.y); }
  static __device__ __forceinline__ double ldcs(const double* p) { return __ldcs(p); }
};
template <>
struct ValT<true> {
  using T = double2;
  static __device__ __forceinline__ double2 mul(double2 v, double2 x) {
    return make_double2(v.x * x.x - v.y * x.y, v.x * x.y + v.y * x.x);
  }
  static __device__ __forceinline__ double2 ldcs(const double2* p) { return __ldcs(p); }
};

constexpr size_t kK1Smem = sizeof(double2) * (kSpmvChunk + kSpmvRows) + sizeof(int64_t) * (kSpmvRows + 1);

template <bool CPLX, int NCW>
__global__ void __launch_bounds__(kThreads, 2) k_spmv_proj(KDev d, int j) {
  static_assert(kThreads == kSpmvRows, "one thread per tile row");
  using VT = typename ValT<CPLX>::T;
  extern __shared__ __align__(128) unsigned char smem[];
  double2* prod = reinterpret_cast<double2*>(smem);
  double2* ps = prod + kSpmvChunk;
  int64_t* rps = reinterpret_cast<int64_t*>(ps + kSpmvRows);
  __shared__ double sj_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) sj_s = step_gate(d, j, blockIdx.x == 0);
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;

  const VT* __restrict__ val = static_cast<const VT*>(d.val);
  const int32_t* __restrict__ col = d.col;
  const double2* __restrict__ x = d.V + (int64_t)j * d.ldv;
  const double2* __restrict__ halo = d.halo;
  const int64_t n = d.n;
  const int ncols = j + 1;
  double2 acc[NCW];
#pragma unroll
  for (int q = 0; q < NCW; ++q) acc[q] = make_double2(0.0, 0.0);

  const int64_t ntiles = (n + kSpmvRows - 1) / kSpmvRows;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * kSpmvRows;
    const int rows = (int)min((int64_t)kSpmvRows, n - r0);
    for (int i = tid; i <= rows; i += kThreads) rps[i] = __ldg(d.rowptr + r0 + i);
    __syncthreads();
    const int64_t b = rps[0], e = rps[rows];
    int64_t mylo = 0, myhi = 0;
    if (tid < rows) { mylo = rps[tid]; myhi = rps[tid + 1]; }
    double2 sum = make_double2(0.0, 0.0);
    for (int64_t cb = b; cb < e; cb += kSpmvChunk) {
      const int cnt = (int)min((int64_t)kSpmvChunk, e - cb);
      // gather-multiply over the chunk's entries: coalesced col/val streams, 4 gathers in flight
      for (int k0 = tid; k0 < cnt; k0 += 4 * kThreads) {
        int cc[4];
        VT vv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u * kThreads;
          if (k < cnt) {
            cc[u] = __ldg(col + cb + k);
            vv[u] = __ldg(val + cb + k);
          }
        }
        double2 xx[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u * kThreads;
          if (k < cnt) xx[u] = (cc[u] < n) ? __ldg(x + cc[u]) : __ldg(halo + (cc[u] - n));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u * kThreads;
          if (k < cnt) prod[k] = ValT<CPLX>::mul(vv[u], xx[u]);
        }
      }
      __syncthreads();
      const int64_t lo = max(mylo, cb), hi = min(myhi, cb + cnt);
      for (int64_t q = lo; q < hi; ++q) sum = cadd(sum, prod[q - cb]);  // row order, left to right
      __syncthreads();
    }
    const double2 p = make_double2(sum.x * sj, sum.y * sj);
    if (tid < rows) d.W[r0 + tid] = p;
    ps[tid] = p;
    __syncthreads();
    // sweep-1 projections on the fresh tile: warp w owns columns w, w+8, ...
#pragma unroll
    for (int q = 0; q < NCW; ++q) {
      const int k = warp + kWarps * q;
      if (k < ncols) {
        const double2* Vk = d.V + (int64_t)k * d.ldv + r0;
        if (rows == kSpmvRows) {
          double2 v[kSpmvRows / 32];
#pragma unroll
          for (int s = 0; s < kSpmvRows / 32; ++s) v[s] = ld_stream(Vk + lane + 32 * s);
#pragma unroll
          for (int s = 0; s < kSpmvRows / 32; ++s) acc[q] = cfma_conj(v[s], ps[lane + 32 * s], acc[q]);
        } else {
          for (int i = lane; i < rows; i += 32) acc[q] = cfma_conj(ld_stream(Vk + i), ps[i], acc[q]);
        }
      }
    }
    __syncthreads();
  }
  finish_columns<NCW>(d, acc, ncols, 0, d.g1);
}

// --------------------------------------------------------------------------------------
// K2: sweep-1 update + sweep-2 projections, V tile staged once (cp.async.bulk + mbarrier)
// --------------------------------------------------------------------------------------
constexpr int kStages = 4;
constexpr int kStageBudget = 48 * 1024;   // bytes of V+W per stage

size_t k2_smem_bytes(int ncols, int* tile_rows) {
  int tr = 1024;
  while (tr > 32 && (size_t)tr * (ncols + 1) * 16 > (size_t)kStageBudget) tr >>= 1;
  if (tile_rows) *tile_rows = tr;
  return (size_t)kStages * tr * (ncols + 1) * 16 + sizeof(double2) * kThreads + 128;
}

template <int NCW>
__global__ void __launch_bounds__(kThreads, 1) k_update_proj(KDev d, int j, int TR) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[kStages];
  __shared__ double2 coef[kMaxCols];
  __shared__ int go_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncols = j + 1;
  if (tid == 0) go_s = (d.flag[0] == 0);
  if (tid < ncols) {
    const double sk = d.s[tid];
    const double2 g = d.g1[tid];
    coef[tid] = make_double2(sk * sk * g.x, sk * sk * g.y);   // e1_k = s_k c1_k, c1_k = s_k g1_k
  }
  __syncthreads();
  if (!go_s) return;

  const int64_t n = d.n;
  const int64_t ntiles = (n + TR - 1) / TR;
  const size_t stage_elems = (size_t)TR * (ncols + 1);
  double2* stage0 = reinterpret_cast<double2*>(smem);
  double2* red = stage0 + kStages * stage_elems;   // kThreads double2 for the grouped update
  const uint64_t pol = policy_evict_first();

  auto issue = [&](int64_t tile, int st) {
    const int64_t r0 = tile * TR;
    const int rows = (int)min((int64_t)TR, n - r0);
    const unsigned bytes = (unsigned)rows * 16u;
    double2* Vs = stage0 + st * stage_elems;
    mbar_expect_tx(&bars[st], bytes * (unsigned)(ncols + 1));
    for (int k = 0; k < ncols; ++k) bulk_g2s(Vs + (size_t)k * TR, d.V + (int64_t)k * d.ldv + r0, bytes, &bars[st], pol);
    bulk_g2s(Vs + (size_t)ncols * TR, d.W + r0, bytes, &bars[st], pol);
  };

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      const int64_t tile = blockIdx.x + (int64_t)s * gridDim.x;
      if (tile < ntiles) issue(tile, s);
    }
  }
  double2 acc[NCW];
#pragma unroll
  for (int q = 0; q < NCW; ++q) acc[q] = make_double2(0.0, 0.0);

  const int G = TR >= kThreads ? 1 : kThreads / TR;  // threads sharing one row in the update
  for (int64_t it = 0;; ++it) {
    const int64_t tile = blockIdx.x + it * gridDim.x;
    if (tile >= ntiles) break;
    const int st = (int)(it % kStages);
    mbar_wait(&bars[st], (unsigned)((it / kStages) & 1));
    double2* Vs = stage0 + st * stage_elems;
    double2* Ws = Vs + (size_t)ncols * TR;
    const int64_t r0 = tile * TR;
    const int rows = (int)min((int64_t)TR, n - r0);
    // ---- phase U: p' = p - V e1 (rows of the tile), written to HBM and back into the stage
    if (G == 1) {
      for (int i = tid; i < rows; i += kThreads) {
        double2 a = make_double2(0.0, 0.0);
        for (int k = 0; k < ncols; ++k) a = cfma(Vs[(size_t)k * TR + i], coef[k], a);
        const double2 p = make_double2(Ws[i].x - a.x, Ws[i].y - a.y);
        Ws[i] = p;
        d.W[r0 + i] = p;
      }
    } else {
      const int g = tid / TR, i = tid - g * TR;
      double2 a = make_double2(0.0, 0.0);
      if (i < rows)
        for (int k = g; k < ncols; k += G) a = cfma(Vs[(size_t)k * TR + i], coef[k], a);
      red[tid] = a;
      __syncthreads();
      if (g == 0 && i < rows) {
        double2 t = red[i];
        for (int gg = 1; gg < G; ++gg) t = cadd(t, red[gg * TR + i]);
        const double2 p = make_double2(Ws[i].x - t.x, Ws[i].y - t.y);
        Ws[i] = p;
        d.W[r0 + i] = p;
      }
    }
    __syncthreads();
    // ---- phase D: g2_k += conj(V_ik) p'_i from the same staged tile
#pragma unroll
    for (int q = 0; q < NCW; ++q) {
      const int k = warp + kWarps * q;
      if (k < ncols) {
        const double2* Vk = Vs + (size_t)k * TR;
        for (int i = lane; i < rows; i += 32) acc[q] = cfma_conj(Vk[i], Ws[i], acc[q]);
      }
    }
    __syncthreads();
    if (tid == 0) {
      // generic-proxy writes to this stage (p') must be ordered before the async-proxy refill
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int64_t nt = blockIdx.x + (it + kStages) * gridDim.x;
      if (nt < ntiles) issue(nt, st);
    }
  }
  finish_columns<NCW>(d, acc, ncols, 1, d.g2);
}

// --------------------------------------------------------------------------------------
// Register-streaming variants (default): a group of TPR lanes owns one row; lane q of the group
// holds the row's V entries of columns k = q + TPR*c (c < kCPT) in registers, so each V element
// is read from HBM exactly once per kernel and reused from registers by both the update and the
// projection phase.  No shared-memory staging and no block-wide barriers inside the row loop.
// --------------------------------------------------------------------------------------
constexpr int kCPT = 8;  // columns per lane

// Cross-lane/cross-warp column sums of acc (lanes with equal q = lane % TPR share columns), in
// a fixed order, then the same last-CTA reduction as finish_columns.
template <int TPR>
__device__ __forceinline__ void finish_grouped(const KDev& d, double2 (&acc)[kCPT], int ncols, int ctr,
                                               double2* out) {
  __shared__ double2 red[kWarps][kMaxCols];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = lane % TPR;
#pragma unroll
  for (int c = 0; c < kCPT; ++c) {
#pragma unroll
    for (int off = TPR; off < 32; off <<= 1) {
      acc[c].x += __shfl_xor_sync(0xffffffffu, acc[c].x, off);
      acc[c].y += __shfl_xor_sync(0xffffffffu, acc[c].y, off);
    }
    const int k = q + TPR * c;
    if (lane < TPR && k < ncols) red[warp][k] = acc[c];
  }
  __syncthreads();
  if (tid < ncols) {
    double2 s = red[0][tid];
    for (int w = 1; w < kWarps; ++w) s = cadd(s, red[w][tid]);
    d.part[(size_t)blockIdx.x * kMaxCols + tid] = s;
  }
  __threadfence();
  __syncthreads();
  __shared__ int last;
  if (tid == 0) last = (atomicAdd(&d.counter[ctr], 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double2 seg[4][kMaxCols];
  const int c = tid & (kMaxCols - 1), sgi = tid >> 6;
  const int G = gridDim.x;
  const int per = (G + 3) / 4;
  double2 s = make_double2(0.0, 0.0);
  if (c < ncols) {
    const int b0 = sgi * per, b1 = min(G, b0 + per);
    for (int b = b0; b < b1; ++b) s = cadd(s, ld_cg(d.part + (size_t)b * kMaxCols + c));
  }
  seg[sgi][c] = s;
  __syncthreads();
  if (tid < ncols) {
    double2 t = seg[0][tid];
    t = cadd(t, seg[1][tid]);
    t = cadd(t, seg[2][tid]);
    t = cadd(t, seg[3][tid]);
    out[tid] = t;
  }
  if (tid == 0) d.counter[ctr] = 0u;
}

template <int TPR>
__device__ __forceinline__ double2 group_sum(double2 v) {
#pragma unroll
  for (int off = 1; off < TPR; off <<= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
  }
  return v;
}

// K1 (register variant): CSR-vector SpMV with TPR lanes per row + in-register projections.
// Rows of the block iteration pf ahead are pulled into L2 with bulk prefetches (V column
// segments, rowptr, col and val ranges) so the register loads of the current iteration hit L2.
template <bool CPLX, int TPR>
__global__ void __launch_bounds__(kThreads, 2) k_spmv_proj_r(KDev d, int j, int pf) {
  using VT = typename ValT<CPLX>::T;
  __shared__ double sj_s;
  const int tid = threadIdx.x, q = tid % TPR, grp = tid / TPR, warp = tid >> 5, lane = tid & 31;
  constexpr int RPB = kThreads / TPR;
  if (tid == 0) sj_s = step_gate(d, j, blockIdx.x == 0);
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;
  const VT* __restrict__ val = static_cast<const VT*>(d.val);
  const int32_t* __restrict__ col = d.col;
  const double2* __restrict__ x = d.V + (int64_t)j * d.ldv;
  const double2* __restrict__ halo = d.halo;
  const int64_t n = d.n, ldv = d.ldv;
  const int ncols = j + 1;
  const int64_t stride = (int64_t)gridDim.x * RPB;
  // warp 0 prefetches V column segments; warp 1 lane 0 the CSR ranges (rowptr values of the
  // block iteration pf ahead are loaded one iteration earlier to keep the issue non-blocking)
  auto pf_v = [&](int64_t rbp) {
    if (rbp >= n) return;
    const unsigned bytes = (unsigned)min((int64_t)RPB, n - rbp) * 16u;
    for (int k = lane; k < ncols; k += 32) prefetch_l2(d.V + rbp + (int64_t)k * ldv, bytes);
  };
  auto pf_csr = [&](int64_t rbp, int64_t lo, int64_t hi) {
    if (rbp >= n) return;
    const int64_t rows = min((int64_t)RPB, n - rbp);
    prefetch_range(d.rowptr, (size_t)rbp * 8, (size_t)(rbp + rows + 1) * 8);
    prefetch_range(col, (size_t)lo * 4, (size_t)hi * 4);
    prefetch_range(val, (size_t)lo * sizeof(VT), (size_t)hi * sizeof(VT));
  };
  int64_t nlo = 0, nhi = 0;  // rowptr bounds of block iteration (it + pf), loaded at it - 1
  if (pf > 0) {
    for (int i = 0; i < pf; ++i) {
      const int64_t rbp = (int64_t)blockIdx.x * RPB + i * stride;
      if (warp == 0) pf_v(rbp);
      if (warp == 1 && lane == 0 && rbp < n) {
        const int64_t lo = __ldg(d.rowptr + rbp), hi = __ldg(d.rowptr + min(rbp + RPB, n));
        pf_csr(rbp, lo, hi);
      }
    }
    const int64_t rbp = (int64_t)blockIdx.x * RPB + pf * stride;
    if (warp == 1 && lane == 0 && rbp < n) {
      nlo = __ldg(d.rowptr + rbp);
      nhi = __ldg(d.rowptr + min(rbp + RPB, n));
    }
  }
  double2 acc[kCPT];
#pragma unroll
  for (int c = 0; c < kCPT; ++c) acc[c] = make_double2(0.0, 0.0);
  for (int64_t rb = (int64_t)blockIdx.x * RPB; rb < n; rb += stride) {
    if (pf > 0) {
      const int64_t rbp = rb + pf * stride;
      if (warp == 0) pf_v(rbp);
      if (warp == 1 && lane == 0 && rbp < n) {
        pf_csr(rbp, nlo, nhi);
        const int64_t rbn = rbp + stride;
        if (rbn < n) {
          nlo = __ldg(d.rowptr + rbn);
          nhi = __ldg(d.rowptr + min(rbn + RPB, n));
        }
      }
    }
    const int64_t r = rb + grp;
    const bool act = r < n;
    double2 v[kCPT];
#pragma unroll
    for (int c = 0; c < kCPT; ++c) {
      const int k = q + TPR * c;
      v[c] = (act && k < ncols) ? ld_stream(d.V + r + (int64_t)k * ldv) : make_double2(0.0, 0.0);
    }
    double2 sum = make_double2(0.0, 0.0);
    if (act) {
      const int64_t lo = __ldg(d.rowptr + r), hi = __ldg(d.rowptr + r + 1);
      for (int64_t e = lo + q; e < hi; e += TPR) {
        const int c = __ldg(col + e);
        const VT w = __ldg(val + e);
        const double2 xv = (c < n) ? __ldg(x + c) : __ldg(halo + (c - n));
        sum = cadd(sum, ValT<CPLX>::mul(w, xv));
      }
    }
    sum = group_sum<TPR>(sum);
    const double2 p = make_double2(sum.x * sj, sum.y * sj);
    if (act && q == 0) d.W[r] = p;
#pragma unroll
    for (int c = 0; c < kCPT; ++c) acc[c] = cfma_conj(v[c], p, acc[c]);
  }
  finish_grouped<TPR>(d, acc, ncols, 0, d.g1);
}

// K2 (register variant): p' = p - V e1 and g2 = V^H p' with the row's V entries in registers
template <int TPR>
__global__ void __launch_bounds__(kThreads, 2) k_update_proj_r(KDev d, int j, int pf) {
  __shared__ double2 coef[kMaxCols];
  __shared__ int go_s;
  const int tid = threadIdx.x, q = tid % TPR, grp = tid / TPR, warp = tid >> 5, lane = tid & 31;
  constexpr int RPB = kThreads / TPR;
  const int ncols = j + 1;
  if (tid == 0) go_s = (d.flag[0] == 0);
  if (tid < ncols) {
    const double sk = d.s[tid];
    const double2 g = d.g1[tid];
    coef[tid] = make_double2(sk * sk * g.x, sk * sk * g.y);
  }
  __syncthreads();
  if (!go_s) return;
  const int64_t n = d.n, ldv = d.ldv;
  const int64_t stride = (int64_t)gridDim.x * RPB;
  auto pf_rows = [&](int64_t rbp) {
    if (rbp >= n) return;
    const unsigned bytes = (unsigned)min((int64_t)RPB, n - rbp) * 16u;
    for (int k = lane; k <= ncols; k += 32)
      prefetch_l2(k < ncols ? (const void*)(d.V + rbp + (int64_t)k * ldv) : (const void*)(d.W + rbp), bytes);
  };
  if (warp == 0)
    for (int i = 0; i < pf; ++i) pf_rows((int64_t)blockIdx.x * RPB + i * stride);
  double2 acc[kCPT];
#pragma unroll
  for (int c = 0; c < kCPT; ++c) acc[c] = make_double2(0.0, 0.0);
  for (int64_t rb = (int64_t)blockIdx.x * RPB; rb < n; rb += stride) {
    if (pf > 0 && warp == 0) pf_rows(rb + pf * stride);
    const int64_t r = rb + grp;
    const bool act = r < n;
    double2 v[kCPT];
#pragma unroll
    for (int c = 0; c < kCPT; ++c) {
      const int k = q + TPR * c;
      v[c] = (act && k < ncols) ? ld_stream(d.V + r + (int64_t)k * ldv) : make_double2(0.0, 0.0);
    }
    const double2 w = act ? __ldcs(d.W + r) : make_double2(0.0, 0.0);
    double2 a = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < kCPT; ++c) {
      const int k = q + TPR * c;
      if (k < ncols) a = cfma(v[c], coef[k], a);
    }
    a = group_sum<TPR>(a);
    const double2 p = make_double2(w.x - a.x, w.y - a.y);
    if (act && q == 0) d.W[r] = p;
#pragma unroll
    for (int c = 0; c < kCPT; ++c) acc[c] = cfma_conj(v[c], p, acc[c]);
  }
  finish_grouped<TPR>(d, acc, ncols, 1, d.g2);
}

// --------------------------------------------------------------------------------------
// TMA-tiled projection kernel (default path), warp-specialised:
//   warp S (producer, one elected lane) streams 32-row x ncols tiles of V with ONE 2-D TMA
//   tensor load per tile (cp.async.bulk.tensor.2d; box = 64 doubles x ncols columns) plus the
//   32-row slice of W (cp.async.bulk), into S shared-memory slots guarded by full/empty
//   mbarriers;  consumer warp w owns slot w and every S-th tile of its CTA, with no CTA-wide
//   barrier inside the loop.
//   MODE 0 (sweep-1):  g1 = V^H p            (dots only)
//   MODE 1 (sweep-2):  p' = p - V e1 -> W,  g2 = V^H p'   (update + dots on the same tile)
// Lane = row for the update; the 32x32 column sums of a tile are formed by a butterfly
// transpose-reduction (31 shuffles per 32 columns instead of 32 x 5), after which lane k owns
// column k and accumulates it across tiles in one register pair.
// --------------------------------------------------------------------------------------
constexpr int kTileR = 32;          // rows per consumer sub-tile (lane = row)
constexpr int kConsumers = 7;       // consumer warps (+1 producer warp = 256 threads)
constexpr int kMaxSlots = 32;
constexpr int kProjThreads = (kConsumers + 1) * 32;
constexpr size_t kProjSmemBudget = 200 * 1024;

// sub-tiles per TMA tile: at least kProjMinTile bytes per tile (fewer, larger TMA operations;
// a 128-row box is the largest single load).  Measured: tools/micro/mb_proj.cu.
size_t g_proj_min_tile = 16384;
int proj_rsub(int ncols) {
  int r = 1;
  while (r < 4 && (size_t)(ncols + 1) * kTileR * 16 * r < g_proj_min_tile) r <<= 1;
  return r;
}
static size_t proj_slot_bytes(int ncols) {
  const int R = proj_rsub(ncols);
  return (size_t)(ncols + 1) * kTileR * R * 16;
}
// Tile i -> slot i % S; slot s is owned by consumer warp s % C for its whole life, so each slot
// is consumed by one warp in round order and no warp can poll a slot's full barrier one phase
// early (mbarrier parity aliasing).
int proj_slots(int ncols) {
  int s = (int)(kProjSmemBudget / proj_slot_bytes(ncols));
  return s > kMaxSlots ? kMaxSlots : (s < 1 ? 1 : s);
}
int proj_consumers(int ncols) {
  const int s = proj_slots(ncols);
  return s < kConsumers ? s : kConsumers;
}
size_t proj_smem_bytes(int ncols) { return (size_t)proj_slots(ncols) * proj_slot_bytes(ncols) + 1024; }

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// re[c], im[c] (c < 32) per lane -> returns the sum over the 32 lanes of column c = lane
__device__ __forceinline__ double2 butterfly_colsum(double (&re)[32], double (&im)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double sr = up ? re[i] : re[i + s];
      const double si = up ? im[i] : im[i + s];
      const double kr = up ? re[i + s] : re[i];
      const double ki = up ? im[i + s] : im[i];
      re[i] = kr + __shfl_xor_sync(0xffffffffu, sr, s);
      im[i] = ki + __shfl_xor_sync(0xffffffffu, si, s);
    }
  }
  return make_double2(re[0], im[0]);
}

// TMA-tiled projection kernel (default path), warp-specialised.  The producer warp streams
// tiles of 32*R rows x ncols columns of V (ONE 2-D tensor load per tile, box 64R doubles x
// ncols) plus the matching rows of W (bulk copy) into S ring slots (full/empty mbarriers);
// tile i of the CTA uses slot i % S and is consumed by warp i % kConsumers, so the number of
// tiles in flight is set by shared memory (~200 KB), not by the number of warps.
//   MODE 0 (sweep-1):  g1 = V^H p                           (dots only)
//   MODE 1 (sweep-2):  p' = p - V e1 -> W,  g2 = V^H p'      (update + dots on the same tile)
// Lane = row for the update; the 32 x 32 column sums of a sub-tile come from a butterfly
// transpose-reduction (31 shuffles per 32 columns), after which lane k owns column k.
// 16-column variant: re[c], im[c] (c < 16) per lane -> sum over the 32 lanes of column
// c = lane & 15 (lanes l and l+16 hold the same value)
__device__ __forceinline__ double2 butterfly_colsum16(double (&re)[16], double (&im)[16]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    re[i] += __shfl_xor_sync(0xffffffffu, re[i], 16);
    im[i] += __shfl_xor_sync(0xffffffffu, im[i], 16);
  }
#pragma unroll
  for (int s = 8; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double sr = up ? re[i] : re[i + s];
      const double si = up ? im[i] : im[i + s];
      const double kr = up ? re[i + s] : re[i];
      const double ki = up ? im[i + s] : im[i];
      re[i] = kr + __shfl_xor_sync(0xffffffffu, sr, s);
      im[i] = ki + __shfl_xor_sync(0xffffffffu, si, s);
    }
  }
  return make_double2(re[0], im[0]);
}

// colsum for NREG register-accumulated columns: NREG = 32 -> lane k owns column k; NREG = 16 ->
// lanes k and k + 16 own column k
// 8-column variant: lanes l, l+8, l+16, l+24 end with the sum of column l & 7
__device__ __forceinline__ double2 butterfly_colsum8(double (&re)[8], double (&im)[8]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    re[i] += __shfl_xor_sync(0xffffffffu, re[i], 16);
    im[i] += __shfl_xor_sync(0xffffffffu, im[i], 16);
    re[i] += __shfl_xor_sync(0xffffffffu, re[i], 8);
    im[i] += __shfl_xor_sync(0xffffffffu, im[i], 8);
  }
#pragma unroll
  for (int s = 4; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double sr = up ? re[i] : re[i + s];
      const double si = up ? im[i] : im[i + s];
      const double kr = up ? re[i + s] : re[i];
      const double ki = up ? im[i + s] : im[i];
      re[i] = kr + __shfl_xor_sync(0xffffffffu, sr, s);
      im[i] = ki + __shfl_xor_sync(0xffffffffu, si, s);
    }
  }
  return make_double2(re[0], im[0]);
}
template <int NREG>
__device__ __forceinline__ double2 colsum_reg(double (&re)[NREG], double (&im)[NREG]) {
  if constexpr (NREG == 32) return butterfly_colsum(re, im);
  else if constexpr (NREG == 16) return butterfly_colsum16(re, im);
  else return butterfly_colsum8(re, im);
}

// NREG: columns whose per-lane partial sums persist in registers across tiles (32 or 16; the
// rest go through 16-wide butterflies per sub-tile).  MINB: resident CTAs per SM (the slot ring
// shares the shared-memory budget between them).
template <int MODE, int NREG = 32, int MINB = 1>
__global__ void __launch_bounds__(kProjThreads, MINB)
    k_proj_tma(const __grid_constant__ CUtensorMap tmV, KDev d, int j, int S, int R, int C, int write) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxSlots], empty[kMaxSlots];
  __shared__ double2 coef[kMaxCols];
  __shared__ double2 red[kConsumers][kMaxCols];
  __shared__ int go_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncols = j + 1;
  __shared__ double2 c1s[kMaxCols];
  __shared__ double nrm_s[kConsumers];
  if (tid == 0) go_s = (d.flag[0] == 0);
  if (MODE == 1 && tid < ncols) {
    const double sk = d.s[tid];
    const double2 g = d.g1[tid];
    coef[tid] = make_double2(sk * sk * g.x, sk * sk * g.y);   // e1_k = s_k c1_k
  }
  if (MODE == 3) {  // f2: c1 = s g1, c2 = c1 - G c1, coefficient on raw V_k: s_k (c1_k + c2_k)
    if (tid < ncols) {
      const double sk = d.s[tid];
      const double2 g = d.g1[tid];
      c1s[tid] = make_double2(sk * g.x, sk * g.y);
    }
    __syncthreads();
    if (tid < ncols) {
      double2 gc = make_double2(0.0, 0.0);
      for (int l = 0; l < ncols; ++l) gc = cfma(d.G[tid * kMaxCols + l], c1s[l], gc);
      const double2 c1 = c1s[tid];
      const double2 c = make_double2(c1.x + (c1.x - gc.x), c1.y + (c1.y - gc.y));
      const double sk = d.s[tid];
      coef[tid] = make_double2(sk * c.x, sk * c.y);
      if (tid == j && blockIdx.x == 0 && d.flag[0] == 0) d.alpha[j] = c.x;  // Re(c1_j + c2_j)
    }
  }
  // 1024-B alignment through an integer cast: the consumers then read the tiles with generic
  // LD.E.128 instead of LDS.128 — measured faster here (tools/micro/mb_proj.cu: dots at 23
  // columns 6.0 vs 4.2 TB/s with the LDS build, which also spills), so kept deliberately
  unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int TR = kTileR * R;
  const size_t vbytes = (size_t)ncols * TR * 16;
  const size_t slot_bytes = vbytes + (size_t)TR * 16;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (!go_s) return;
  const int64_t n = d.n;
  const int64_t ntiles = (n + TR - 1) / TR;

  if (warp == kConsumers) {  // ---------------- producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
      const uint64_t pol = policy_evict_first();
      for (int64_t i = 0;; ++i) {
        const int64_t tile = blockIdx.x + i * gridDim.x;
        if (tile >= ntiles) break;
        const int s = (int)(i % S);
        const int64_t round = i / S;
        if (round > 0) mbar_wait(&empty[s], (unsigned)((round - 1) & 1));
        const int rows = (int)min((int64_t)TR, n - tile * TR);
        unsigned char* base = smem + (size_t)s * slot_bytes;
        mbar_expect_tx(&full[s], (unsigned)vbytes + (unsigned)rows * 16u);
        tma_load_2d(base, &tmV, (int)(tile * TR * 2), 0, &full[s]);
        bulk_g2s(base + vbytes, d.W + tile * TR, (unsigned)rows * 16u, &full[s], pol);
      }
    }
  } else if (warp < C) {  // ------- consumers: warp owns slots warp, warp + C, ... (< S)
    // columns 0..31: per-lane partial sums over all of this warp's rows, kept in registers and
    // reduced across lanes once at the end; columns 32..: butterfly per 32-row sub-tile
    double aR[NREG], aI[NREG];
#pragma unroll
    for (int c = 0; c < NREG; ++c) aR[c] = aI[c] = 0.0;
    // 16-wide butterfly groups above NREG (<= 4): lane l & 15 owns column NREG + 16 g + (l & 15)
    double2 accb0 = make_double2(0.0, 0.0), accb1 = accb0, accb2 = accb0, accb3 = accb0;
    double nrm = 0.0;
    double2* outV = (MODE == 3 && write) ? d.V + (int64_t)(j + 1) * d.ldv : nullptr;
    bool more = true;
    for (int64_t base = 0; more; base += S) {
      for (int s = warp; s < S; s += C) {
        const int64_t i = base + s;
        const int64_t tile = blockIdx.x + i * gridDim.x;
        if (tile >= ntiles) { more = false; break; }
        mbar_wait(&full[s], (unsigned)((i / S) & 1));
        const double2* Vs = reinterpret_cast<const double2*>(smem + (size_t)s * slot_bytes);
        const double2* Ws = reinterpret_cast<const double2*>(smem + (size_t)s * slot_bytes + vbytes);
        const int64_t r0 = tile * TR;
        const int rows = (int)min((int64_t)TR, n - r0);
        for (int sub = 0; sub < R && MODE != 2; ++sub) {  // MODE 2: streaming only (microbenchmark)
          const int row = sub * kTileR + lane;
          if (sub * kTileR >= rows) break;  // warp-uniform
          double2 p = row < rows ? Ws[row] : make_double2(0.0, 0.0);
          if (MODE == 1 || MODE == 3) {
            // eight independent FMA chains over the columns, 8 tile loads in flight
            double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0, a4 = a0, a5 = a0, a6 = a0, a7 = a0;
            int k = 0;
            for (; k + 8 <= ncols; k += 8) {
              const double2 v0 = Vs[(k + 0) * TR + row], v1 = Vs[(k + 1) * TR + row];
              const double2 v2 = Vs[(k + 2) * TR + row], v3 = Vs[(k + 3) * TR + row];
              const double2 v4 = Vs[(k + 4) * TR + row], v5 = Vs[(k + 5) * TR + row];
              const double2 v6 = Vs[(k + 6) * TR + row], v7 = Vs[(k + 7) * TR + row];
              a0 = cfma(v0, coef[k + 0], a0);
              a1 = cfma(v1, coef[k + 1], a1);
              a2 = cfma(v2, coef[k + 2], a2);
              a3 = cfma(v3, coef[k + 3], a3);
              a4 = cfma(v4, coef[k + 4], a4);
              a5 = cfma(v5, coef[k + 5], a5);
              a6 = cfma(v6, coef[k + 6], a6);
              a7 = cfma(v7, coef[k + 7], a7);
            }
            // remainder (< 8 columns) on independent chains as well
            if (k + 0 < ncols) a0 = cfma(Vs[(k + 0) * TR + row], coef[k + 0], a0);
            if (k + 1 < ncols) a1 = cfma(Vs[(k + 1) * TR + row], coef[k + 1], a1);
            if (k + 2 < ncols) a2 = cfma(Vs[(k + 2) * TR + row], coef[k + 2], a2);
            if (k + 3 < ncols) a3 = cfma(Vs[(k + 3) * TR + row], coef[k + 3], a3);
            if (k + 4 < ncols) a4 = cfma(Vs[(k + 4) * TR + row], coef[k + 4], a4);
            if (k + 5 < ncols) a5 = cfma(Vs[(k + 5) * TR + row], coef[k + 5], a5);
            if (k + 6 < ncols) a6 = cfma(Vs[(k + 6) * TR + row], coef[k + 6], a6);
            const double2 a = cadd(cadd(cadd(a0, a1), cadd(a2, a3)), cadd(cadd(a4, a5), cadd(a6, a7)));
            p = make_double2(p.x - a.x, p.y - a.y);
            if (row >= rows) p = make_double2(0.0, 0.0);
            else if (MODE == 1) d.W[r0 + row] = p;
            else {
              if (outV) outV[r0 + row] = p;
              nrm = fma(p.x, p.x, fma(p.y, p.y, nrm));
            }
          }
#pragma unroll
          for (int c = 0; c < NREG; ++c) {
            if (c < ncols) {
              const double2 v = Vs[c * TR + row];
              aR[c] = fma(v.x, p.x, fma(v.y, p.y, aR[c]));   // conj(v) * p
              aI[c] = fma(v.x, p.y, fma(-v.y, p.x, aI[c]));
            }
          }
#pragma unroll 1
          for (int cb = NREG; cb < ncols; cb += 16) {  // columns NREG.. in 16-wide butterflies
            double re[16], im[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              const int k = cb + c;
              const double2 v = k < ncols ? Vs[k * TR + row] : make_double2(0.0, 0.0);
              re[c] = v.x * p.x + v.y * p.y;
              im[c] = v.x * p.y - v.y * p.x;
            }
            const double2 cs = butterfly_colsum16(re, im);
            const int g = (cb - NREG) >> 4;
            if (g == 0) accb0 = cadd(accb0, cs);
            else if (g == 1) accb1 = cadd(accb1, cs);
            else if (g == 2) accb2 = cadd(accb2, cs);
            else accb3 = cadd(accb3, cs);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
    const double2 acc0 = colsum_reg<NREG>(aR, aI);
    if (lane < NREG) red[warp][lane] = acc0;
    if (lane < 16) {
      const double2 ab[4] = {accb0, accb1, accb2, accb3};
#pragma unroll
      for (int g = 0; g < 4; ++g)
        if (NREG + 16 * g + lane < kMaxCols) red[warp][NREG + 16 * g + lane] = ab[g];
    }
    if (MODE == 3) {
      nrm = warp_sum(nrm);
      if (lane == 0) nrm_s[warp] = nrm;
    }
  }
  __syncthreads();
  // block partial in fixed warp order, then the last-CTA reduction
  double2* out = MODE == 0 ? d.g1 : d.g2;
  const int ctr = MODE == 0 ? 0 : 1;
  if (tid < ncols) {
    double2 t = red[0][tid];
    for (int w = 1; w < C; ++w) t = cadd(t, red[w][tid]);
    d.part[(size_t)blockIdx.x * kMaxCols + tid] = t;
  }
  if (MODE == 3 && tid == 0) {
    double t = 0.0;
    for (int w = 0; w < C; ++w) t += nrm_s[w];
    d.partn[blockIdx.x] = t;
  }
  __threadfence();
  __syncthreads();
  __shared__ int last;
  if (tid == 0) last = (atomicAdd(&d.counter[ctr], 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double2 seg[4][kMaxCols];
  const int G = gridDim.x;
  const int per = (G + 3) / 4;
  {
    const int c = tid & (kMaxCols - 1), sgi = tid >> 6;
    double2 sm = make_double2(0.0, 0.0);
    if (c < ncols) {
      const int b0 = sgi * per, b1 = min(G, b0 + per);
      for (int b = b0; b < b1; ++b) sm = cadd(sm, ld_cg(d.part + (size_t)b * kMaxCols + c));
    }
    seg[sgi][c] = sm;
  }
  __syncthreads();
  if (tid < ncols) {
    double2 t = seg[0][tid];
    t = cadd(t, seg[1][tid]);
    t = cadd(t, seg[2][tid]);
    t = cadd(t, seg[3][tid]);
    out[tid] = t;
  }
  if (MODE == 3 && tid == 0) {  // ||p''||^2 in fixed block order
    double t = 0.0;
    for (int b = 0; b < G; ++b) t += __ldcg(d.partn + b);
    d.nrm2[j] = t;
  }
  if (tid == 0) d.counter[ctr] = 0u;
}

// Register-streaming projection kernel with shuffle row-reduction (default): TPR lanes per row,
// lane q holds the row's V entries of columns q + TPR*c (c < 8) in registers.  Column sums over
// the warp's rows are formed by xor-shuffles over the row bits of the lane index and added to a
// per-warp shared-memory accumulator, so no per-column accumulator registers persist across rows
// (~60 registers -> 4 CTAs of 256 threads per SM, 8 loads of 16 B in flight per thread).
//   MODE 0:  g1 = V^H p                          MODE 1:  p' = p - V e1 -> W, g2 = V^H p'
template <int MODE, int TPR>
__global__ void __launch_bounds__(kThreads, 4) k_proj_s(KDev d, int j) {
  __shared__ double2 coef[kMaxCols];
  __shared__ double2 red[kWarps][kMaxCols];
  __shared__ int go_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = tid % TPR, grp = tid / TPR;
  constexpr int RPB = kThreads / TPR;
  const int ncols = j + 1;
  if (tid == 0) go_s = (d.flag[0] == 0);
  if (MODE == 1 && tid < ncols) {
    const double sk = d.s[tid];
    const double2 g = d.g1[tid];
    coef[tid] = make_double2(sk * sk * g.x, sk * sk * g.y);
  }
  for (int i = tid; i < kWarps * kMaxCols; i += kThreads) (&red[0][0])[i] = make_double2(0.0, 0.0);
  __syncthreads();
  if (!go_s) return;
  const int64_t n = d.n, ldv = d.ldv;
  const int cmax = (ncols + TPR - 1) / TPR;  // live column slots per lane
  for (int64_t rb = (int64_t)blockIdx.x * RPB; rb < n; rb += (int64_t)gridDim.x * RPB) {
    const int64_t r = rb + grp;
    const bool act = r < n;
    double2 v[kCPT];
#pragma unroll
    for (int c = 0; c < kCPT; ++c) {
      const int k = q + TPR * c;
      v[c] = (act && k < ncols) ? ld_stream(d.V + r + (int64_t)k * ldv) : make_double2(0.0, 0.0);
    }
    double2 p = act ? (MODE == 1 ? __ldcs(d.W + r) : __ldg(d.W + r)) : make_double2(0.0, 0.0);
    if (MODE == 1) {
      double2 a = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < kCPT; ++c) {
        const int k = q + TPR * c;
        if (k < ncols) a = cfma(v[c], coef[k], a);
      }
      a = group_sum<TPR>(a);
      p = make_double2(p.x - a.x, p.y - a.y);
      if (act && q == 0) d.W[r] = p;
    }
#pragma unroll
    for (int c = 0; c < kCPT; ++c) {
      if (c >= cmax) break;  // warp-uniform: only the live column slots are reduced
      double2 pr = make_double2(v[c].x * p.x + v[c].y * p.y, v[c].x * p.y - v[c].y * p.x);  // conj(v) p
#pragma unroll
      for (int off = TPR; off < 32; off <<= 1) {
        pr.x += __shfl_xor_sync(0xffffffffu, pr.x, off);
        pr.y += __shfl_xor_sync(0xffffffffu, pr.y, off);
      }
      const int k = q + TPR * c;
      if (lane < TPR && k < ncols) red[warp][k] = cadd(red[warp][k], pr);
    }
  }
  __syncthreads();
  double2* out = MODE == 0 ? d.g1 : d.g2;
  const int ctr = MODE;
  if (tid < ncols) {
    double2 t = red[0][tid];
    for (int w = 1; w < kWarps; ++w) t = cadd(t, red[w][tid]);
    d.part[(size_t)blockIdx.x * kMaxCols + tid] = t;
  }
  __threadfence();
  __syncthreads();
  __shared__ int last;
  if (tid == 0) last = (atomicAdd(&d.counter[ctr], 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double2 seg[4][kMaxCols];
  const int G = gridDim.x;
  const int per = (G + 3) / 4;
  {
    const int c = tid & (kMaxCols - 1), sgi = tid >> 6;
    double2 sm = make_double2(0.0, 0.0);
    if (c < ncols) {
      const int b0 = sgi * per, b1 = min(G, b0 + per);
      for (int b = b0; b < b1; ++b) sm = cadd(sm, ld_cg(d.part + (size_t)b * kMaxCols + c));
    }
    seg[sgi][c] = sm;
  }
  __syncthreads();
  if (tid < ncols) {
    double2 t = seg[0][tid];
    t = cadd(t, seg[1][tid]);
    t = cadd(t, seg[2][tid]);
    t = cadd(t, seg[3][tid]);
    out[tid] = t;
  }
  if (tid == 0) d.counter[ctr] = 0u;
}

// --------------------------------------------------------------------------------------
// TMA-fed SpMV (default): p = s_j H V_j -> W.  Tiles of <= kSpmvTmaNnz entries / kSpmvTmaRows
// rows (descriptors {first row, first entry} built at create).  The producer warp bulk-copies
// (cp.async.bulk) each tile's rowptr, col and val ranges into a ring of shared-memory slots;
// consumer warp (slot owner) gathers x (L2-resident) for 32 entries per instruction, 8 gathers
// in flight per lane, stages the products in its scratch and sums each row left to right.
// A single row longer than a tile is handled by its consumer straight from global memory.
// --------------------------------------------------------------------------------------
constexpr int kSpmvTmaNnz = kSpmvTmaNnzCap;
constexpr int kSpmvTmaRows = kSpmvTmaRowCap;
constexpr int kSmRp = ((kSpmvTmaRows + 4) * 8 + 15) / 16 * 16;
constexpr int kSmCol = ((kSpmvTmaNnz + 4) * 4 + 15) / 16 * 16;
size_t spmv_slot_bytes(bool cplx) { return kSmRp + kSmCol + (size_t)(kSpmvTmaNnz + 2) * (cplx ? 16 : 8) + 16; }
constexpr size_t kSpmvScratch = 0;  // (no per-warp product scratch: lane-per-row sums)
int spmv_slots(bool cplx) {
  const size_t avail = kProjSmemBudget - kConsumers * kSpmvScratch;
  int s = (int)(avail / spmv_slot_bytes(cplx));
  return s > kMaxSlots ? kMaxSlots : (s < kConsumers ? kConsumers : s);
}
size_t spmv_smem_bytes(bool cplx) { return kConsumers * kSpmvScratch + spmv_slots(cplx) * spmv_slot_bytes(cplx) + 1024; }

template <bool CPLX>
__global__ void __launch_bounds__(kProjThreads, 1) k_spmv_tma(KDev d, int j, int S) {
  using VT = typename ValT<CPLX>::T;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxSlots], empty[kMaxSlots];
  __shared__ double sj_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int C = kConsumers;
  // 1024-B alignment through an integer cast: the consumers then read the tiles with generic
  // LD.E.128 instead of LDS.128 — measured faster here (tools/micro/mb_proj.cu: dots at 23
  // columns 6.0 vs 4.2 TB/s with the LDS build, which also spills), so kept deliberately
  unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const size_t slot_bytes = kSmRp + kSmCol + (size_t)(kSpmvTmaNnz + 2) * sizeof(VT) + 16;
  unsigned char* slots = smem + C * kSpmvScratch;
  if (tid == 0) {
    sj_s = step_gate(d, j, blockIdx.x == 0);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;
  const int64_t n = d.n;
  const int64_t ntiles = d.ntiles_desc;
  const VT* __restrict__ val = static_cast<const VT*>(d.val);
  const int32_t* __restrict__ col = d.col;
  const double2* __restrict__ x = d.V + (int64_t)j * d.ldv;
  const double2* __restrict__ halo = d.halo;
  const int64_t* __restrict__ tdesc = d.tile_desc;  // pairs {first row, first entry}, ntiles+1

  if (warp == C) {  // ---------------- producer (whole warp loads descriptors, lane 0 issues)
    const uint64_t pol = policy_evict_first();
    for (int64_t base = 0;; base += 32) {
      const int64_t ti = blockIdx.x + (base + lane) * gridDim.x;
      int64_t ra = 0, ea = 0, rb = 0, eb = 0;
      if (ti < ntiles) {
        ra = __ldg(tdesc + 2 * ti);
        ea = __ldg(tdesc + 2 * ti + 1);
        rb = __ldg(tdesc + 2 * ti + 2);
        eb = __ldg(tdesc + 2 * ti + 3);
      }
      bool done = false;
      for (int l = 0; l < 32; ++l) {
        const int64_t i = base + l;
        const int64_t t = blockIdx.x + i * gridDim.x;
        if (t >= ntiles) { done = true; break; }
        const int64_t Ra = __shfl_sync(0xffffffffu, ra, l), Ea = __shfl_sync(0xffffffffu, ea, l);
        const int64_t Rb = __shfl_sync(0xffffffffu, rb, l), Eb = __shfl_sync(0xffffffffu, eb, l);
        if (lane == 0) {
          const int s = (int)(i % S);
          const int64_t round = i / S;
          if (round > 0) mbar_wait(&empty[s], (unsigned)((round - 1) & 1));
          unsigned char* sl = slots + (size_t)s * slot_bytes;
          if (Eb - Ea > kSpmvTmaNnz) {  // long row: consumer reads global memory
            mbar_expect_tx(&full[s], 0u);
          } else {
            const int64_t r0 = Ra & ~1LL, r1 = (Rb + 2) & ~1LL;          // rowptr[Ra..Rb], 16 B aligned
            const int64_t c0 = Ea & ~3LL, c1 = (Eb + 3) & ~3LL;          // col[Ea..Eb)
            constexpr int64_t VA = 16 / (int64_t)sizeof(VT);
            const int64_t v0 = Ea & ~(VA - 1), v1 = (Eb + VA - 1) & ~(VA - 1);
            const unsigned br = (unsigned)((r1 - r0) * 8), bc = (unsigned)((c1 - c0) * 4),
                           bv = (unsigned)((v1 - v0) * sizeof(VT));
            mbar_expect_tx(&full[s], br + (bc ? bc : 0u) + (bv ? bv : 0u));
            bulk_g2s(sl, d.rowptr + r0, br, &full[s], pol);
            if (bc) bulk_g2s(sl + kSmRp, col + c0, bc, &full[s], pol);
            if (bv) bulk_g2s(sl + kSmRp + kSmCol, val + v0, bv, &full[s], pol);
          }
        }
        __syncwarp();
      }
      if (done) break;
    }
  } else if (warp < C) {  // ---------------- consumers: warp owns slots warp, warp + C, ...
    bool more = true;
    for (int64_t base = 0; more; base += S) {
      for (int s = warp; s < S; s += C) {
        const int64_t i = base + s;
        const int64_t t = blockIdx.x + i * gridDim.x;
        if (t >= ntiles) { more = false; break; }
        const int64_t Ra = __ldg(tdesc + 2 * t), Ea = __ldg(tdesc + 2 * t + 1);
        const int64_t Rb = __ldg(tdesc + 2 * t + 2), Eb = __ldg(tdesc + 2 * t + 3);
        const int rows = (int)(Rb - Ra);
        const int cnt = (int)(Eb - Ea);
        mbar_wait(&full[s], (unsigned)((i / S) & 1));
        if (cnt > kSpmvTmaNnz) {  // one long row (rows == 1), straight from global memory
          double2 sum = make_double2(0.0, 0.0);
          for (int64_t e = Ea + lane; e < Eb; e += 32) {
            const int c = __ldg(col + e);
            const double2 xv = (c < n) ? __ldg(x + c) : __ldg(halo + (c - n));
            sum = cadd(sum, ValT<CPLX>::mul(__ldg(val + e), xv));
          }
          sum = warp_sum(sum);
          if (lane == 0) __stcs(d.W + Ra, make_double2(sum.x * sj, sum.y * sj));
        } else {
          const unsigned char* sl = slots + (size_t)s * slot_bytes;
          const int64_t* rp = reinterpret_cast<const int64_t*>(sl) + (Ra & 1);
          const int32_t* cs = reinterpret_cast<const int32_t*>(sl + kSmRp) + (Ea & 3);
          constexpr int64_t VA = 16 / (int64_t)sizeof(VT);
          const VT* vs = reinterpret_cast<const VT*>(sl + kSmRp + kSmCol) + (Ea & (VA - 1));
          // lane = row: the k-th entries of 32 consecutive rows are gathered together (neighbouring
          // rows have neighbouring columns in structured matrices -> few sectors per request);
          // each lane sums its own row left to right, kG gathers in flight
          constexpr int kG = 8;
          for (int rr0 = 0; rr0 < rows; rr0 += 32) {
            const int rr = rr0 + lane;
            int lo = 0, len = 0;
            if (rr < rows) {
              lo = (int)(rp[rr] - Ea);
              len = (int)(rp[rr + 1] - Ea) - lo;
            }
            int mlen = len;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) mlen = max(mlen, __shfl_xor_sync(0xffffffffu, mlen, off));
            double2 sum = make_double2(0.0, 0.0);
            for (int q0 = 0; q0 < mlen; q0 += kG) {
              int cc[kG];
              VT vv[kG];
#pragma unroll
              for (int u = 0; u < kG; ++u)
                if (q0 + u < len) { cc[u] = cs[lo + q0 + u]; vv[u] = vs[lo + q0 + u]; }
              double2 xx[kG];
#pragma unroll
              for (int u = 0; u < kG; ++u)
                if (q0 + u < len) xx[u] = (cc[u] < n) ? __ldg(x + cc[u]) : __ldg(halo + (cc[u] - n));
#pragma unroll
              for (int u = 0; u < kG; ++u)
                if (q0 + u < len) sum = cadd(sum, ValT<CPLX>::mul(vv[u], xx[u]));
            }
            if (rr < rows) __stcs(d.W + Ra + rr, make_double2(sum.x * sj, sum.y * sj));
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
  }
}

// Standalone SpMV, nnz-balanced tiles (default): tile t covers rows [tile_row[t], tile_row[t+1])
// holding ~kSpmvTileNnz entries (built at create time).  Each thread issues all kSpmvE col/val
// loads of a chunk at once, then all x gathers, products go to shared memory, and one thread
// per row sums its entries left to right (deterministic).  3 dependent latencies per chunk.
constexpr int kSpmvE = 4;
constexpr int kChunk = kThreads * kSpmvE;  // 1024 entries per chunk
template <bool CPLX>
__global__ void __launch_bounds__(kThreads, 4) k_spmv_tile(KDev d, int j) {
  using VT = typename ValT<CPLX>::T;
  __shared__ double2 prod[kChunk];
  __shared__ int64_t rps[kSpmvMaxTileRows + 1];
  __shared__ double sj_s;
  const int tid = threadIdx.x;
  if (tid == 0) sj_s = step_gate(d, j, blockIdx.x == 0);
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;
  const VT* __restrict__ val = static_cast<const VT*>(d.val);
  const int32_t* __restrict__ col = d.col;
  const double2* __restrict__ x = d.V + (int64_t)j * d.ldv;
  const double2* __restrict__ halo = d.halo;
  const int64_t n = d.n;
  constexpr int RPT = kSpmvMaxTileRows / kThreads;  // rows per thread (max)
  for (int64_t t = blockIdx.x; t < d.ntiles; t += gridDim.x) {
    const int64_t ra = __ldg(d.tile_row + t), rb = __ldg(d.tile_row + t + 1);
    const int rows = (int)(rb - ra);
    for (int i = tid; i <= rows; i += kThreads) rps[i] = __ldg(d.rowptr + ra + i);
    __syncthreads();
    const int64_t b = rps[0], e = rps[rows];
    double2 acc[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) acc[u] = make_double2(0.0, 0.0);
    for (int64_t cb = b; cb < e; cb += kChunk) {
      const int cnt = (int)min((int64_t)kChunk, e - cb);
      int cc[kSpmvE];
      VT vv[kSpmvE];
#pragma unroll
      for (int u = 0; u < kSpmvE; ++u) {
        const int q = tid + u * kThreads;
        if (q < cnt) {
          cc[u] = __ldg(col + cb + q);
          vv[u] = __ldg(val + cb + q);
        }
      }
      double2 xx[kSpmvE];
#pragma unroll
      for (int u = 0; u < kSpmvE; ++u) {
        const int q = tid + u * kThreads;
        if (q < cnt) xx[u] = (cc[u] < n) ? __ldg(x + cc[u]) : __ldg(halo + (cc[u] - n));
      }
#pragma unroll
      for (int u = 0; u < kSpmvE; ++u) {
        const int q = tid + u * kThreads;
        if (q < cnt) prod[q] = ValT<CPLX>::mul(vv[u], xx[u]);
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int i = tid + u * kThreads;
        if (i < rows) {
          const int64_t lo = max(rps[i], cb), hi = min(rps[i + 1], cb + cnt);
          for (int64_t q = lo; q < hi; ++q) acc[u] = cadd(acc[u], prod[q - cb]);
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int i = tid + u * kThreads;
      if (i < rows) __stcs(d.W + ra + i, make_double2(acc[u].x * sj, acc[u].y * sj));
    }
    __syncthreads();
  }
}

// SpMV variant 3: nnz-balanced tiles, col/val staged coalesced into shared memory, then one
// thread per row gathers x for its own entries (the k-th entries of neighbouring rows sit at
// neighbouring columns in structured matrices) and sums them left to right.
template <bool CPLX>
__global__ void __launch_bounds__(kThreads, 4) k_spmv_rowtile(KDev d, int j) {
  using VT = typename ValT<CPLX>::T;
  __shared__ int32_t cs[kChunk];
  __shared__ VT vs[kChunk];
  __shared__ int64_t rps[kSpmvMaxTileRows + 1];
  __shared__ double sj_s;
  const int tid = threadIdx.x;
  if (tid == 0) sj_s = step_gate(d, j, blockIdx.x == 0);
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;
  const VT* __restrict__ val = static_cast<const VT*>(d.val);
  const int32_t* __restrict__ col = d.col;
  const double2* __restrict__ x = d.V + (int64_t)j * d.ldv;
  const double2* __restrict__ halo = d.halo;
  const int64_t n = d.n;
  constexpr int RPT = kSpmvMaxTileRows / kThreads;
  for (int64_t t = blockIdx.x; t < d.ntiles; t += gridDim.x) {
    const int64_t ra = __ldg(d.tile_row + t), rb = __ldg(d.tile_row + t + 1);
    const int rows = (int)(rb - ra);
    for (int i = tid; i <= rows; i += kThreads) rps[i] = __ldg(d.rowptr + ra + i);
    __syncthreads();
    const int64_t b = rps[0], e = rps[rows];
    double2 acc[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) acc[u] = make_double2(0.0, 0.0);
    for (int64_t cb = b; cb < e; cb += kChunk) {
      const int cnt = (int)min((int64_t)kChunk, e - cb);
#pragma unroll
      for (int u = 0; u < kSpmvE; ++u) {
        const int q = tid + u * kThreads;
        if (q < cnt) { cs[q] = __ldg(col + cb + q); vs[q] = __ldg(val + cb + q); }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int i = tid + u * kThreads;
        if (i < rows) {
          const int lo = (int)(max(rps[i], cb) - cb), hi = (int)(min(rps[i + 1], cb + cnt) - cb);
          int q = lo;
          for (; q + 4 <= hi; q += 4) {
            double2 xx[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) { const int c = cs[q + w]; xx[w] = (c < n) ? __ldg(x + c) : __ldg(halo + (c - n)); }
#pragma unroll
            for (int w = 0; w < 4; ++w) acc[u] = cadd(acc[u], ValT<CPLX>::mul(vs[q + w], xx[w]));
          }
          for (; q < hi; ++q) {
            const int c = cs[q];
            acc[u] = cadd(acc[u], ValT<CPLX>::mul(vs[q], (c < n) ? __ldg(x + c) : __ldg(halo + (c - n))));
          }
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int i = tid + u * kThreads;
      if (i < rows) __stcs(d.W + ra + i, make_double2(acc[u].x * sj, acc[u].y * sj));
    }
    __syncthreads();
  }
}

// SpMV variant 4 (default): the row-tile SpMV software-pipelined with cp.async double buffering.
// While the threads gather x for the rows of tile t (one thread per row, entries from shared
// memory), the rowptr/col/val ranges of tile t+1 are already in flight into the other buffer and
// the descriptors of tile t+2 are being loaded.  A tile whose single row exceeds the buffer is
// summed straight from global memory by the whole block (fixed-order block reduction).
__device__ __forceinline__ void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

struct TileDesc { int64_t ra, rb, b, e; };

template <bool CPLX>
size_t spmv_pipe_smem() {
  using VT = typename ValT<CPLX>::T;
  constexpr int cap = CPLX ? kSpmvTileNnzC : kSpmvTileNnz;
  return 2 * ((size_t)(kSpmvMaxTileRows + 4) * 8 + (size_t)(cap + 4) * 4 + (size_t)(cap + 4) * sizeof(VT));
}

// halo entry hi of step j from the owning rank's V column (uncached: written by another GPU)
__device__ __forceinline__ double2 peer_x(const KDev& d, int j, int hi) {
  const int q = __ldg(d.halo_owner + hi);
  const double2* base = d.peer_base[q];
  return __ldcv(base + (int64_t)j * __ldg(d.peer_ldv + q) + __ldg(d.halo_lidx + hi));
}

// HM: 0 single rank (every column local), 1 multi-rank with the halo staged by the NCCL exchange,
// 2 multi-rank reading halo columns straight from the owning rank's V column (peer memory over
// NVLink; the exchange fused into the SpMV)
template <bool CPLX, int TPR, int HM, int NF>
__global__ void __launch_bounds__(kThreads, 2) k_spmv_pipe(KDev d, int j, int pf) {
  using VT = typename ValT<CPLX>::T;
  extern __shared__ __align__(16) unsigned char smp[];
  // buffer b at smp + b * kBuf: [val kChunk][rowptr kSpmvMaxTileRows+2][col kChunk]
  constexpr int kCap = CPLX ? kSpmvTileNnzC : kSpmvTileNnz;
  constexpr size_t kVal = (size_t)(kCap + 4) * sizeof(VT), kRp = (size_t)(kSpmvMaxTileRows + 4) * 8;
  constexpr size_t kBuf = kVal + kRp + (size_t)(kCap + 4) * 4;
  auto vs_of = [&](int b) { return reinterpret_cast<VT*>(smp + b * kBuf); };
  auto rp_of = [&](int b) { return reinterpret_cast<int64_t*>(smp + b * kBuf + kVal); };
  auto cs_of = [&](int b) { return reinterpret_cast<int32_t*>(smp + b * kBuf + kVal + kRp); };
  __shared__ double sj_s;
  __shared__ double2 red[kWarps];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    sj_s = step_gate(d, j, blockIdx.x == 0);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;
  const uint64_t pol = policy_evict_first();
  const VT* __restrict__ val = static_cast<const VT*>(d.val);
  const int32_t* __restrict__ col = d.col;
  const double2* __restrict__ x = d.V + (int64_t)j * d.ldv;
  asm volatile("" : "+l"(x));  // keep the column base in a register (no per-gather recompute)
  const double2* __restrict__ halo = d.halo;
  const int64_t n = d.n;
  const int64_t G = gridDim.x;
  const int q = tid % TPR, grp = tid / TPR;  // TPR lanes per row (tiles hold <= kThreads/TPR rows)

  auto desc = [&](int64_t t) {
    TileDesc td{0, 0, 0, 0};
    if (t < d.ntiles) {
      td.ra = __ldg(d.tile_row + t);
      td.rb = __ldg(d.tile_row + t + 1);
      td.b = __ldg(d.rowptr + td.ra);
      td.e = __ldg(d.rowptr + td.rb);
    }
    return td;
  };
  // bulk copies (TMA engine, one thread) of the 16-byte-aligned supersets of the tile's rowptr /
  // col / val ranges into buffer bsel; completion counted on bar[bsel]
  auto issue = [&](const TileDesc& td, int bsel, int64_t t) {
    if (tid == 0 && t < d.ntiles) {
      const int64_t cnt = td.e - td.b;
      const int64_t r0 = td.ra & ~1LL, r1 = (td.rb + 2) & ~1LL;
      unsigned br = (unsigned)((r1 - r0) * 8), bc = 0, bv = 0;
      int64_t c0 = 0, v0 = 0;
      if (cnt <= kCap) {
        constexpr int64_t VA = 16 / (int64_t)sizeof(VT);
        c0 = td.b & ~3LL;
        v0 = td.b & ~(VA - 1);
        bc = (unsigned)((((td.e + 3) & ~3LL) - c0) * 4);
        bv = (unsigned)((((td.e + VA - 1) & ~(VA - 1)) - v0) * sizeof(VT));
      }
      mbar_expect_tx(&bar[bsel], br + bc + bv);
      bulk_g2s(rp_of(bsel), d.rowptr + r0, br, &bar[bsel], pol);
      if (bc) bulk_g2s(cs_of(bsel), col + c0, bc, &bar[bsel], pol);
      if (bv) bulk_g2s(vs_of(bsel), val + v0, bv, &bar[bsel], pol);
    }
  };
  const int64_t t0 = blockIdx.x;
  TileDesc cur = desc(t0);
  TileDesc nxt = desc(t0 + G);
  issue(cur, 0, t0);
  for (int64_t it = 0;; ++it) {
    const int64_t t = t0 + it * G;
    if (t >= d.ntiles) break;
    const int bsel = (int)(it & 1);
    issue(nxt, bsel ^ 1, t + G);                // tile t+G in flight during this tile's gathers
    const TileDesc nn = desc(t + 2 * G);        // descriptor loads in flight as well
    mbar_wait(&bar[bsel], (unsigned)((it >> 1) & 1));
    const int rows = (int)(cur.rb - cur.ra);
    const int64_t cnt = cur.e - cur.b;
    if (cnt <= kCap) {
      constexpr int64_t VA = 16 / (int64_t)sizeof(VT);
      const int64_t* rp = rp_of(bsel) + (cur.ra & 1);
      const int32_t* cc = cs_of(bsel) + (cur.b & 3);
      const VT* vv = vs_of(bsel) + (cur.b & (VA - 1));
      {  // group grp owns row grp of the tile (tiles hold <= kThreads/TPR rows); lane q takes
         // entries lo+q, lo+q+TPR, ... (NF gathers in flight: 16 for real values, 8 for complex
         // ones, whose registers are twice as wide), then a fixed-order xor reduction
        const int i = grp;
        const bool act = i < rows;
        const int lo = act ? (int)(rp[i] - cur.b) : 0, hi = act ? (int)(rp[i + 1] - cur.b) : 0;
        double2 acc = make_double2(0.0, 0.0);
        for (int q0 = lo + q; q0 < hi; q0 += NF * TPR) {
          double2 xx[NF];
#pragma unroll
          for (int w = 0; w < NF; ++w) {
            const int e = q0 + w * TPR;
            if (e < hi) {
              const int c = cc[e];
              if (HM == 1) xx[w] = ((uint32_t)c < (uint32_t)n) ? __ldg(x + c) : __ldg(halo + (c - (int)n));
              else if (HM == 2) xx[w] = ((uint32_t)c < (uint32_t)n) ? __ldg(x + c) : peer_x(d, j, c - (int)n);
              else xx[w] = __ldg(x + c);   // single rank: every column is local
            }
          }
          // values are re-read from shared memory here rather than held in registers across the
          // gathers (under the 128-register cap ptxas still issues the gathers in groups of 4-6
          // ahead of their products; the reverse accumulation order is kept from that experiment)
#pragma unroll
          for (int w = NF - 1; w >= 0; --w)
            if (q0 + w * TPR < hi) acc = cadd(acc, ValT<CPLX>::mul(vv[q0 + w * TPR], xx[w]));
        }
        if (TPR > 1) acc = group_sum<TPR>(acc);
        if (act && q == 0) __stcs(d.W + cur.ra + i, make_double2(acc.x * sj, acc.y * sj));
      }
      // L2 prefetch of tile t+2G's entries (its descriptor arrived during this tile): one more
      // tile of DRAM reads in flight per CTA without shared memory
      if (pf && tid == 32 && t + 2 * G < d.ntiles) {
        prefetch_range(col, (size_t)nn.b * 4, (size_t)nn.e * 4);
        prefetch_range(val, (size_t)nn.b * sizeof(VT), (size_t)nn.e * sizeof(VT));
      }
    } else {  // one long row, straight from global memory
      double2 acc = make_double2(0.0, 0.0);
      for (int64_t q = cur.b + tid; q < cur.e; q += kThreads) {
        const int c = __ldg(col + q);
        const double2 xv = (c < n) ? __ldg(x + c) : (HM == 2 ? peer_x(d, j, (int)(c - n)) : __ldg(halo + (c - n)));
        acc = cadd(acc, ValT<CPLX>::mul(__ldg(val + q), xv));
      }
      acc = warp_sum(acc);
      if ((tid & 31) == 0) red[tid >> 5] = acc;
      __syncthreads();
      if (tid == 0) {
        double2 s = red[0];
        for (int w = 1; w < kWarps; ++w) s = cadd(s, red[w]);
        __stcs(d.W + cur.ra, make_double2(s.x * sj, s.y * sj));
      }
    }
    __syncthreads();                            // buffer bsel free for tile t+2G
    if (tid == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    cur = nxt;
    nxt = nn;
  }
}

// SpMV variant 7 (warp-specialised ring): one producer warp issues the bulk copies of tiles into
// a kRingStages-deep shared-memory ring (full/empty mbarriers); 15 consumer warps process every tile
// (TPR lanes per row, <= 480/TPR rows per tile) and release a stage per warp, so warps are never
// joined by a block barrier: the extra gather round of a long row delays one warp, not the tile.
// Tile descriptors {first row, end row, first entry, end entry} come from a host table; the
// producer copies each into its stage.  A row longer than a tile is summed by one consumer warp
// straight from global memory.
// STG stages of kCap entries: 4 x 4096 (real) / 2048 (complex), or 3 x 5632 / 2816 (te_api picks
// per matrix: the deeper ring for short real rows, the larger tiles otherwise)
constexpr int kRingConsumers = 15;
constexpr int kRingThreads = (kRingConsumers + 1) * 32;

template <bool CPLX, int STG>
struct RingLayout {
  using VT = typename ValT<CPLX>::T;
  static constexpr int kCap = STG == 3 ? (CPLX ? kRingNnzC3 : kRingNnz3) : (CPLX ? kRingNnzC4 : kRingNnz4);
  static constexpr size_t kVal = (size_t)(kCap + 4) * sizeof(VT);
  static constexpr size_t kRp = (size_t)(kRingConsumers * 32 + 4) * 8;
  static constexpr size_t kCol = (size_t)(kCap + 4) * 4;
  static constexpr size_t kStage = kVal + kRp + kCol;
  static constexpr size_t kBytes = STG * kStage;
};
template <bool CPLX, int STG>
size_t spmv_ring_smem() { return RingLayout<CPLX, STG>::kBytes; }

template <bool CPLX, int TPR, int HM, int NF, int STG>
__global__ void __launch_bounds__(kRingThreads, 1) k_spmv_ring(KDev d, int j) {
  using VT = typename ValT<CPLX>::T;
  using LY = RingLayout<CPLX, STG>;
  constexpr int kRingStages = STG;
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[kRingStages], empty[kRingStages];
  __shared__ int64_t desc[kRingStages][4];
  __shared__ double sj_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    sj_s = step_gate(d, j, blockIdx.x == 0);
    for (int k = 0; k < kRingStages; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], kRingConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;
  const int64_t G = gridDim.x;
  if (warp == kRingConsumers) {  // ------------------------------------------------ producer
    if (lane != 0) return;
    const uint64_t pol = policy_evict_first();
    constexpr int64_t VA = 16 / (int64_t)sizeof(VT);
    for (int64_t it = 0;; ++it) {
      const int64_t t = blockIdx.x + it * G;
      const int st = (int)(it % kRingStages);
      if (it >= kRingStages) mbar_wait(&empty[st], (unsigned)(((it / kRingStages) - 1) & 1));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (t >= d.ntiles_ring) {  // tell the consumers there is nothing more
        desc[st][0] = -1;
        mbar_expect_tx(&full[st], 0);
        break;
      }
      const longlong2 a = __ldg(reinterpret_cast<const longlong2*>(d.tile_ring + 4 * t));
      const longlong2 b = __ldg(reinterpret_cast<const longlong2*>(d.tile_ring + 4 * t) + 1);
      desc[st][0] = a.x; desc[st][1] = a.y; desc[st][2] = b.x; desc[st][3] = b.y;
      const int64_t cnt = b.y - b.x;
      const int64_t r0 = a.x & ~1LL, r1 = (a.y + 2) & ~1LL;
      unsigned br = (unsigned)((r1 - r0) * 8), bc = 0, bv = 0;
      int64_t c0 = 0, v0 = 0;
      if (cnt <= LY::kCap) {
        c0 = b.x & ~3LL;
        v0 = b.x & ~(VA - 1);
        bc = (unsigned)((((b.y + 3) & ~3LL) - c0) * 4);
        bv = (unsigned)((((b.y + VA - 1) & ~(VA - 1)) - v0) * sizeof(VT));
      } else {
        br = 0;
      }
      unsigned char* base = sm + (size_t)st * LY::kStage;
      mbar_expect_tx(&full[st], br + bc + bv);
      if (br) bulk_g2s(base + LY::kVal, d.rowptr + r0, br, &full[st], pol);
      if (bc) bulk_g2s(base + LY::kVal + LY::kRp, d.col + c0, bc, &full[st], pol);
      if (bv) bulk_g2s(base, static_cast<const VT*>(d.val) + v0, bv, &full[st], pol);
    }
    return;
  }
  // --------------------------------------------------------------------------------- consumers
  const double2* __restrict__ x = d.V + (int64_t)j * d.ldv;
  asm volatile("" : "+l"(x));
  const double2* __restrict__ halo = d.halo;
  const int n = (int)d.n;
  const int q = tid % TPR, grp = tid / TPR;  // consumer threads 0 .. 32*kRingConsumers-1
  auto gx = [&](int c) -> double2 {
    if (HM == 1) return ((uint32_t)c < (uint32_t)n) ? __ldg(x + c) : __ldg(halo + (c - n));
    if (HM == 2) return ((uint32_t)c < (uint32_t)n) ? __ldg(x + c) : peer_x(d, j, c - n);
    return __ldg(x + c);
  };
  for (int64_t it = 0;; ++it) {
    const int st = (int)(it % kRingStages);
    mbar_wait(&full[st], (unsigned)((it / kRingStages) & 1));
    const int64_t ra = desc[st][0];
    if (ra < 0) break;
    const int64_t rb = desc[st][1], b = desc[st][2], e = desc[st][3];
    const int64_t cnt = e - b;
    const int64_t t = blockIdx.x + it * G;
    if (cnt <= LY::kCap) {
      constexpr int64_t VA = 16 / (int64_t)sizeof(VT);
      const unsigned char* base = sm + (size_t)st * LY::kStage;
      const int64_t* rp = reinterpret_cast<const int64_t*>(base + LY::kVal) + (ra & 1);
      const int32_t* cc = reinterpret_cast<const int32_t*>(base + LY::kVal + LY::kRp) + (b & 3);
      const VT* vv = reinterpret_cast<const VT*>(base) + (b & (VA - 1));
      const int rows = (int)(rb - ra);
      const int i = grp;
      const bool act = i < rows;
      const int lo = act ? (int)(rp[i] - b) : 0, hi = act ? (int)(rp[i + 1] - b) : 0;
      double2 acc = make_double2(0.0, 0.0);
      for (int q0 = lo + q; q0 < hi; q0 += NF * TPR) {
        double2 xx[NF];
#pragma unroll
        for (int w = 0; w < NF; ++w) {
          const int ee = q0 + w * TPR;
          if (ee < hi) xx[w] = gx(cc[ee]);
        }
#pragma unroll
        for (int w = NF - 1; w >= 0; --w)
          if (q0 + w * TPR < hi) acc = cadd(acc, ValT<CPLX>::mul(vv[q0 + w * TPR], xx[w]));
      }
      if (TPR > 1) acc = group_sum<TPR>(acc);
      if (act && q == 0) __stcs(d.W + ra + i, make_double2(acc.x * sj, acc.y * sj));
    } else if (warp == (int)(t % kRingConsumers)) {  // one long row: one warp, from global memory
      const VT* __restrict__ val = static_cast<const VT*>(d.val);
      double2 acc = make_double2(0.0, 0.0);
      for (int64_t k = b + lane; k < e; k += 32) acc = cadd(acc, ValT<CPLX>::mul(__ldg(val + k), gx(__ldg(d.col + k))));
      acc = warp_sum(acc);
      if (lane == 0) __stcs(d.W + ra, make_double2(acc.x * sj, acc.y * sj));
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
}

// SpMV variant 5 (async gather).  The x gathers of a tile are cp.async copies into shared
// memory, so a whole tile's gathers (<= kAgCap) are in flight at once without holding registers,
// and they overlap the products of the previous tile:
//   iteration it:  bulk copy (TMA engine) of tile it+2's rowptr/col/val   [3-stage ring]
//                  cp.async gathers x[col] of tile it+1                   [2-stage ring]
//                  products + per-row sums of tile it from shared memory
// Tile descriptors {ra, rb, b, e} come from a host-built table (te_api: kAgCap entries, <=
// kThreads/TPR rows per tile) through a 4-slot shared ring that thread 0 fills one iteration
// ahead.  Per row: TPR lanes, in-order partial sums, fixed xor reduction (deterministic).
__device__ __forceinline__ void cp_async16_ca(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <bool CPLX>
struct AgLayout {
  using VT = typename ValT<CPLX>::T;
  static constexpr size_t kVal = (size_t)(kAgCap + 4) * sizeof(VT);
  static constexpr size_t kRp = (size_t)(kAgMaxRows + 4) * 8;
  static constexpr size_t kCol = (size_t)(kAgCap + 4) * 4;
  static constexpr size_t kStage = kVal + kRp + kCol;
  static constexpr size_t kBytes = 3 * kStage + 2 * (size_t)kAgCap * 16;
};

template <bool CPLX>
size_t spmv_ag_smem() { return AgLayout<CPLX>::kBytes; }

template <bool CPLX, int TPR, bool HALO>
__global__ void __launch_bounds__(kThreads, CPLX ? 2 : 3) k_spmv_ag(KDev d, int j) {
  using VT = typename ValT<CPLX>::T;
  using LY = AgLayout<CPLX>;
  extern __shared__ __align__(16) unsigned char sm[];
  auto vs_of = [&](int st) { return reinterpret_cast<const VT*>(sm + st * LY::kStage); };
  auto rp_of = [&](int st) { return reinterpret_cast<const int64_t*>(sm + st * LY::kStage + LY::kVal); };
  auto cs_of = [&](int st) { return reinterpret_cast<const int32_t*>(sm + st * LY::kStage + LY::kVal + LY::kRp); };
  auto xg_of = [&](int b) { return reinterpret_cast<double2*>(sm + 3 * LY::kStage) + (size_t)b * kAgCap; };
  __shared__ double sj_s;
  __shared__ double2 red[kWarps];
  __shared__ __align__(8) uint64_t bar[3];
  __shared__ int64_t ring[4][4];  // descriptors of iterations it..it+3 (slot it & 3); ra < 0: none
  const int tid = threadIdx.x;
  const int64_t G = gridDim.x, t0 = blockIdx.x;
  const int64_t* __restrict__ tab = d.tile_ag;
  const uint64_t pol = policy_evict_first();
  auto load_desc = [&](int64_t it, int64_t (&o)[4]) {
    const int64_t t = t0 + it * G;
    if (t < d.ntiles_ag) {
      const longlong2 a = __ldg(reinterpret_cast<const longlong2*>(tab + 4 * t));
      const longlong2 b = __ldg(reinterpret_cast<const longlong2*>(tab + 4 * t) + 1);
      o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
    } else {
      o[0] = -1; o[1] = -1; o[2] = 0; o[3] = 0;
    }
  };
  // bulk copy of one tile's rowptr / col / val (16-byte-aligned supersets) into stage st
  auto issue = [&](const int64_t* td, int st) {
    if (td[0] < 0) return;
    const int64_t cnt = td[3] - td[2];
    const int64_t r0 = td[0] & ~1LL, r1 = (td[1] + 2) & ~1LL;
    unsigned br = (unsigned)((r1 - r0) * 8), bc = 0, bv = 0;
    int64_t c0 = 0, v0 = 0;
    constexpr int64_t VA = 16 / (int64_t)sizeof(VT);
    if (cnt <= kAgCap) {
      c0 = td[2] & ~3LL;
      v0 = td[2] & ~(VA - 1);
      bc = (unsigned)((((td[3] + 3) & ~3LL) - c0) * 4);
      bv = (unsigned)((((td[3] + VA - 1) & ~(VA - 1)) - v0) * sizeof(VT));
    }
    unsigned char* base = sm + st * LY::kStage;
    mbar_expect_tx(&bar[st], br + bc + bv);
    bulk_g2s(base + LY::kVal, d.rowptr + r0, br, &bar[st], pol);
    if (bc) bulk_g2s(base + LY::kVal + LY::kRp, d.col + c0, bc, &bar[st], pol);
    if (bv) bulk_g2s(base, static_cast<const VT*>(d.val) + v0, bv, &bar[st], pol);
  };
  if (tid == 0) {
    sj_s = step_gate(d, j, blockIdx.x == 0);
    for (int k = 0; k < 3; ++k) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k < 3; ++k) {
      int64_t o[4];
      load_desc(k, o);
      for (int q = 0; q < 4; ++q) ring[k][q] = o[q];
    }
    if (sj_s != 0.0) {
      issue(ring[0], 0);
      issue(ring[1], 1);
    }
  }
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;
  const double2* __restrict__ x = d.V + (int64_t)j * d.ldv;
  asm volatile("" : "+l"(x));
  const double2* __restrict__ halo = d.halo;
  const int64_t n = d.n;
  // gathers of iteration k's tile (stage k % 3 must have landed) into xg[k & 1]
  auto gather = [&](int64_t k) {
    const int64_t* td = ring[k & 3];
    if (td[0] < 0) return;
    const int64_t b = td[2], cnt = td[3] - b;
    if (cnt > kAgCap) return;  // long row: summed from global memory in the compute phase
    const int st = (int)(k % 3);
    mbar_wait(&bar[st], (unsigned)((k / 3) & 1));
    const int32_t* cc = cs_of(st) + (b & 3);
    double2* xb = xg_of((int)(k & 1));
    for (int e = tid; e < (int)cnt; e += kThreads) {
      const int c = cc[e];
      const double2* src;
      if (HALO) src = ((uint32_t)c < (uint32_t)n) ? x + c : halo + (c - (int)n);
      else src = x + c;
      cp_async16_ca(xb + e, src);
    }
  };
  gather(0);
  cp_async_commit();
  const int q = tid % TPR, grp = tid / TPR;
  for (int64_t it = 0;; ++it) {
    const int64_t ra = ring[it & 3][0];
    if (ra < 0) break;
    int64_t nd[4];
    if (tid == 0) {
      load_desc(it + 3, nd);               // lands during this iteration
      issue(ring[(it + 2) & 3], (int)((it + 2) % 3));
    }
    gather(it + 1);
    cp_async_commit();
    cp_async_wait1();                      // this thread's gathers of tile it are complete
    __syncthreads();                       // ... and every thread's
    const int64_t rb = ring[it & 3][1], b = ring[it & 3][2], e = ring[it & 3][3];
    const int64_t cnt = e - b;
    const int st = (int)(it % 3);
    if (cnt <= kAgCap) {
      constexpr int64_t VA = 16 / (int64_t)sizeof(VT);
      const int64_t* rp = rp_of(st) + (ra & 1);
      const VT* vv = vs_of(st) + (b & (VA - 1));
      const double2* xb = xg_of((int)(it & 1));
      const int rows = (int)(rb - ra);
      const int i = grp;
      const bool act = i < rows;
      const int lo = act ? (int)(rp[i] - b) : 0, hi = act ? (int)(rp[i + 1] - b) : 0;
      double2 acc = make_double2(0.0, 0.0);
      for (int k = lo + q; k < hi; k += TPR) acc = cadd(acc, ValT<CPLX>::mul(vv[k], xb[k]));
      if (TPR > 1) acc = group_sum<TPR>(acc);
      if (act && q == 0) __stcs(d.W + ra + i, make_double2(acc.x * sj, acc.y * sj));
    } else {  // one long row, straight from global memory (its stage holds only rowptr)
      const VT* __restrict__ val = static_cast<const VT*>(d.val);
      double2 acc = make_double2(0.0, 0.0);
      for (int64_t k = b + tid; k < e; k += kThreads) {
        const int c = __ldg(d.col + k);
        const double2 xv = (!HALO || (uint32_t)c < (uint32_t)n) ? __ldg(x + c) : __ldg(halo + (c - (int)n));
        acc = cadd(acc, ValT<CPLX>::mul(__ldg(val + k), xv));
      }
      acc = warp_sum(acc);
      if ((tid & 31) == 0) red[tid >> 5] = acc;
      __syncthreads();
      if (tid == 0) {
        double2 s2 = red[0];
        for (int w = 1; w < kWarps; ++w) s2 = cadd(s2, red[w]);
        __stcs(d.W + ra, make_double2(s2.x * sj, s2.y * sj));
      }
    }
    if (tid == 0)
      for (int k = 0; k < 4; ++k) ring[(it + 3) & 3][k] = nd[k];
    __syncthreads();                       // stage it % 3, xg[it & 1] and ring slot it & 3 free
    if (tid == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  cp_async_wait0();
}

// SpMV variant 6: SELL-C-sigma (C = 32).  Rows sorted by length (descending, stable) inside
// windows of kSellSigma rows, cut into slices of 32; a slice stores its entries column-major
// (entry k of lane l at sptr[s] + 32 k + l, zero-padded to the slice width with the lane's own
// row as column), so a warp streams its slice with fully coalesced loads and no shared-memory
// staging or block barriers.  One lane per row, entries in CSR order: each row's sum is the
// sequential sum of its products.  Built on the device from the CSR (te_api: build_sell).
template <bool CPLX>
__global__ void k_sell_build(int64_t npos, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                             const void* __restrict__ val_, const int32_t* __restrict__ perm,
                             const int64_t* __restrict__ sptr, const int32_t* __restrict__ slen,
                             int32_t* __restrict__ scol, void* __restrict__ sval_) {
  using VT = typename ValT<CPLX>::T;
  const VT* val = static_cast<const VT*>(val_);
  VT* sval = static_cast<VT*>(sval_);
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npos; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = p >> 5;
    const int l = (int)(p & 31);
    const int r = perm[p];
    const int w = slen[s];
    const int64_t base = sptr[s] + l;
    int64_t a = 0, len = 0;
    if (r >= 0) {
      a = rowptr[r];
      len = rowptr[r + 1] - a;
    }
    const int pc = r >= 0 ? r : 0;
    for (int k = 0; k < w; ++k) {
      const int64_t o = base + (int64_t)k * 32;
      if (k < len) {
        scol[o] = col[a + k];
        sval[o] = val[a + k];
      } else {
        scol[o] = pc;
        sval[o] = VT{};
      }
    }
  }
}

template <bool CPLX>
void launch_sell_build(int64_t npos, const int64_t* rowptr, const int32_t* col, const void* val, const int32_t* perm,
                       const int64_t* sptr, const int32_t* slen, int32_t* scol, void* sval, cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(65535, (npos + kThreads - 1) / kThreads));
  k_sell_build<CPLX><<<grid, kThreads, 0, st>>>(npos, rowptr, col, val, perm, sptr, slen, scol, sval);
}
void launch_sell_build(bool cplx, int64_t npos, const int64_t* rowptr, const int32_t* col, const void* val,
                       const int32_t* perm, const int64_t* sptr, const int32_t* slen, int32_t* scol, void* sval,
                       cudaStream_t st) {
  if (cplx) launch_sell_build<true>(npos, rowptr, col, val, perm, sptr, slen, scol, sval, st);
  else launch_sell_build<false>(npos, rowptr, col, val, perm, sptr, slen, scol, sval, st);
}

template <bool CPLX, bool HALO, int U>
__global__ void __launch_bounds__(kThreads, 2) k_spmv_sell(KDev d, int j) {
  using VT = typename ValT<CPLX>::T;
  __shared__ double sj_s;
  if (threadIdx.x == 0) sj_s = step_gate(d, j, blockIdx.x == 0);
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;
  const double2* __restrict__ x = d.V + (int64_t)j * d.ldv;
  asm volatile("" : "+l"(x));
  const double2* __restrict__ halo = d.halo;
  const int n = (int)d.n;
  const int32_t* __restrict__ scol = d.scol;
  const VT* __restrict__ sval = static_cast<const VT*>(d.sval);
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  auto gx = [&](int c) -> double2 {
    if (HALO) return __ldg(((uint32_t)c < (uint32_t)n) ? x + c : halo + (c - n));
    return __ldg(x + c);
  };
  // software pipeline over batches of U entries per lane: in iteration b the gathers of batch
  // b+1 and the column/value loads of batch b+2 are issued before batch b's products, so both
  // latencies stay hidden across the loop back-edge; entries past the slice width read column 0
  // with value 0 (predicated, no padding to a multiple of U)
  for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < d.nslices; s += nw) {
    const int64_t base = __ldg(d.sptr + s) + lane;
    const int w = __ldg(d.slen + s);
    const int r = __ldg(d.sperm + s * 32 + lane);
    const int nb = (w + U - 1) / U;
    auto ldcv = [&](int b, int (&c)[U], VT (&v)[U]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = b * U + u;
        if (k < w) {
          c[u] = __ldg(scol + base + (int64_t)k * 32);
          v[u] = __ldg(sval + base + (int64_t)k * 32);
        } else {
          c[u] = 0;
          v[u] = VT{};
        }
      }
    };
    int cB[U];
    VT vA[U], vB[U];
    double2 xA[U];
    if (nb > 0) {
      int cA[U];
      ldcv(0, cA, vA);
#pragma unroll
      for (int u = 0; u < U; ++u) xA[u] = gx(cA[u]);
    }
    if (nb > 1) ldcv(1, cB, vB);
    double2 acc = make_double2(0.0, 0.0);
    for (int b = 0; b < nb; ++b) {
      double2 xB[U];
      int cC[U];
      VT vC[U];
      if (b + 1 < nb) {
#pragma unroll
        for (int u = 0; u < U; ++u) xB[u] = gx(cB[u]);
      }
      if (b + 2 < nb) ldcv(b + 2, cC, vC);
#pragma unroll
      for (int u = 0; u < U; ++u) acc = cadd(acc, ValT<CPLX>::mul(vA[u], xA[u]));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        xA[u] = xB[u];
        vA[u] = vB[u];
        cB[u] = cC[u];
        vB[u] = vC[u];
      }
    }
    if (r >= 0) __stcs(d.W + r, make_double2(acc.x * sj, acc.y * sj));
  }
}

// Standalone SpMV p = s_j H V_j -> W (CSR-vector, TPR lanes per row, high occupancy).
template <bool CPLX, int TPR>
__global__ void __launch_bounds__(kThreads) k_spmv(KDev d, int j) {
  using VT = typename ValT<CPLX>::T;
  __shared__ double sj_s;
  const int tid = threadIdx.x, q = tid % TPR, grp = tid / TPR;
  constexpr int RPB = kThreads / TPR;
  if (tid == 0) sj_s = step_gate(d, j, blockIdx.x == 0);
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;
  const VT* __restrict__ val = static_cast<const VT*>(d.val);
  const int32_t* __restrict__ col = d.col;
  const double2* __restrict__ x = d.V + (int64_t)j * d.ldv;
  const double2* __restrict__ halo = d.halo;
  const int64_t n = d.n;
  for (int64_t rb = (int64_t)blockIdx.x * RPB; rb < n; rb += (int64_t)gridDim.x * RPB) {
    const int64_t r = rb + grp;
    double2 sum = make_double2(0.0, 0.0);
    if (r < n) {
      const int64_t lo = __ldg(d.rowptr + r), hi = __ldg(d.rowptr + r + 1);
      int64_t e = lo + q;
      for (; e + TPR < hi; e += 2 * TPR) {  // two entries in flight per lane
        const int c0 = __ldg(col + e), c1 = __ldg(col + e + TPR);
        const VT w0 = __ldg(val + e), w1 = __ldg(val + e + TPR);
        const double2 x0 = (c0 < n) ? __ldg(x + c0) : __ldg(halo + (c0 - n));
        const double2 x1 = (c1 < n) ? __ldg(x + c1) : __ldg(halo + (c1 - n));
        sum = cadd(sum, ValT<CPLX>::mul(w0, x0));
        sum = cadd(sum, ValT<CPLX>::mul(w1, x1));
      }
      if (e < hi) {
        const int c0 = __ldg(col + e);
        const VT w0 = __ldg(val + e);
        const double2 x0 = (c0 < n) ? __ldg(x + c0) : __ldg(halo + (c0 - n));
        sum = cadd(sum, ValT<CPLX>::mul(w0, x0));
      }
    }
    sum = group_sum<TPR>(sum);
    if (r < n && q == 0) __stcs(d.W + r, make_double2(sum.x * sj, sum.y * sj));
  }
}

// --------------------------------------------------------------------------------------
// K3: sweep-2 update + norm; writes p'' as (unnormalised) column j+1
// --------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_update_norm(KDev d, int j, int write, int pf) {
  __shared__ double2 coef[kMaxCols];
  __shared__ int go_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncols = j + 1;
  if (tid == 0) {
    go_s = (d.flag[0] == 0);
    if (go_s && blockIdx.x == 0) {  // alpha_j = Re(c1_j + c2_j) (reading C2)
      const double sj = d.s[j];
      d.alpha[j] = sj * (d.g1[j].x + d.g2[j].x);
    }
  }
  if (tid < ncols) {
    const double sk = d.s[tid];
    const double2 g = d.g2[tid];
    coef[tid] = make_double2(sk * sk * g.x, sk * sk * g.y);
  }
  __syncthreads();
  if (!go_s) return;
  const int64_t n = d.n, ldv = d.ldv;
  double2* out = write ? d.V + (int64_t)(j + 1) * ldv : nullptr;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  auto pf_rows = [&](int64_t rbp) {
    if (rbp >= n) return;
    const unsigned bytes = (unsigned)min((int64_t)kThreads, n - rbp) * 16u;
    for (int k = lane; k <= ncols; k += 32)
      prefetch_l2(k < ncols ? (const void*)(d.V + rbp + (int64_t)k * ldv) : (const void*)(d.W + rbp), bytes);
  };
  if (warp == 0)
    for (int i = 0; i < pf; ++i) pf_rows((int64_t)blockIdx.x * kThreads + i * stride);
  double nrm = 0.0;
  for (int64_t rb = (int64_t)blockIdx.x * kThreads; rb < n; rb += stride) {
    if (pf > 0 && warp == 0) pf_rows(rb + pf * stride);
    const int64_t r = rb + tid;
    if (r >= n) continue;
    double2 a = make_double2(0.0, 0.0);
    const double2* Vr = d.V + r;
    int k = 0;
    for (; k + 8 <= ncols; k += 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ld_stream(Vr + (int64_t)(k + u) * ldv);
#pragma unroll
      for (int u = 0; u < 8; ++u) a = cfma(v[u], coef[k + u], a);
    }
    for (; k < ncols; ++k) a = cfma(ld_stream(Vr + (int64_t)k * ldv), coef[k], a);
    const double2 w = __ldcs(d.W + r);
    const double2 p = make_double2(w.x - a.x, w.y - a.y);
    if (out) out[r] = p;
    nrm = fma(p.x, p.x, fma(p.y, p.y, nrm));
  }
  finish_scalar(d, nrm, 2, d.nrm2 + j);
}

// --------------------------------------------------------------------------------------
// Paper-literal 3-term Lanczos recurrence (Eq. 8; Alg. 1):
//   p' = p - beta_{j-1} v_{j-1};  a = v_j^H p';  p'' = p' - a v_j;  alpha_j = Re(a)
// with v_k = s_k V_k.  Two streaming kernels after the SpMV (p' is recomputed, not stored).
// --------------------------------------------------------------------------------------
__device__ __forceinline__ void finish_complex(const KDev& d, double2 v, int ctr, double2* out) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __shared__ double2 ws[kWarps];
  v = warp_sum(v);
  if (lane == 0) ws[warp] = v;
  __syncthreads();
  if (tid == 0) {
    double2 t = ws[0];
    for (int w = 1; w < kWarps; ++w) t = cadd(t, ws[w]);
    d.part[(size_t)blockIdx.x * kMaxCols] = t;
  }
  __threadfence();
  __syncthreads();
  __shared__ int last;
  if (tid == 0) last = (atomicAdd(&d.counter[ctr], 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double2 seg[kThreads];
  const int G = gridDim.x;
  const int per = (G + kThreads - 1) / kThreads;
  double2 s = make_double2(0.0, 0.0);
  const int b0 = tid * per, b1 = min(G, b0 + per);
  for (int b = b0; b < b1; ++b) s = cadd(s, ld_cg(d.part + (size_t)b * kMaxCols));
  seg[tid] = s;
  __syncthreads();
  if (tid == 0) {
    double2 t = make_double2(0.0, 0.0);
    for (int i = 0; i < kThreads; ++i) t = cadd(t, seg[i]);
    *out = t;
    d.counter[ctr] = 0u;
  }
}

__global__ void __launch_bounds__(kThreads) k_lanczos_dot(KDev d, int j) {
  __shared__ int go_s;
  __shared__ double cb_s, sj_s;
  const int tid = threadIdx.x;
  if (tid == 0) {
    go_s = (d.flag[0] == 0);
    cb_s = j > 0 ? d.beta[j - 1] * d.s[j - 1] : 0.0;  // beta_{j-1} v_{j-1} = beta_{j-1} s_{j-1} V_{j-1}
    sj_s = d.s[j];
  }
  __syncthreads();
  if (!go_s) return;
  const double cb = cb_s;
  const int64_t n = d.n, ldv = d.ldv;
  const double2* Vp = d.V + (int64_t)(j > 0 ? j - 1 : 0) * ldv;
  const double2* Vj = d.V + (int64_t)j * ldv;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t r = (int64_t)blockIdx.x * kThreads + tid; r < n; r += (int64_t)gridDim.x * kThreads) {
    double2 p = __ldg(d.W + r);
    if (j > 0) {
      const double2 vp = ld_stream(Vp + r);
      p = make_double2(p.x - cb * vp.x, p.y - cb * vp.y);
    }
    acc = cfma_conj(ld_stream(Vj + r), p, acc);
  }
  finish_complex(d, acc, 0, d.g1 + j);  // raw sum; a = s_j * g1[j]
}

__global__ void __launch_bounds__(kThreads) k_lanczos_update(KDev d, int j, int write) {
  __shared__ int go_s;
  __shared__ double cb_s;
  __shared__ double2 ca_s;
  const int tid = threadIdx.x;
  if (tid == 0) {
    go_s = (d.flag[0] == 0);
    const double sj = d.s[j];
    const double2 g = d.g1[j];
    cb_s = j > 0 ? d.beta[j - 1] * d.s[j - 1] : 0.0;
    ca_s = make_double2(sj * sj * g.x, sj * sj * g.y);  // a v_j = (s_j g) (s_j V_j)
    if (go_s && blockIdx.x == 0) d.alpha[j] = sj * g.x;  // alpha_j = Re(a)
  }
  __syncthreads();
  if (!go_s) return;
  const double cb = cb_s;
  const double2 ca = ca_s;
  const int64_t n = d.n, ldv = d.ldv;
  const double2* Vp = d.V + (int64_t)(j > 0 ? j - 1 : 0) * ldv;
  const double2* Vj = d.V + (int64_t)j * ldv;
  double2* out = write ? d.V + (int64_t)(j + 1) * ldv : nullptr;
  double nrm = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * kThreads + tid; r < n; r += (int64_t)gridDim.x * kThreads) {
    double2 p = __ldcs(d.W + r);
    if (j > 0) {
      const double2 vp = ld_stream(Vp + r);
      p = make_double2(p.x - cb * vp.x, p.y - cb * vp.y);
    }
    const double2 vj = ld_stream(Vj + r);
    const double2 av = make_double2(ca.x * vj.x - ca.y * vj.y, ca.x * vj.y + ca.y * vj.x);
    p = make_double2(p.x - av.x, p.y - av.y);
    if (out) out[r] = p;
    nrm = fma(p.x, p.x, fma(p.y, p.y, nrm));
  }
  finish_scalar(d, nrm, 2, d.nrm2 + j);
}

void launch_lanczos_dot(const KDev& d, int j, const Launch& L) {
  k_lanczos_dot<<<L.grid_k3, kThreads, 0, L.stream>>>(d, j);
}
void launch_lanczos_update(const KDev& d, int j, bool write, const Launch& L) {
  k_lanczos_update<<<L.grid_k3, kThreads, 0, L.stream>>>(d, j, write ? 1 : 0);
}

// ||p''_{m-1}||^2 -> beta_{m-1} = h_{m+1,m} and the final breakdown test (Alg. 1)
__global__ void k_finalize(KDev d, int j) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (d.flag[0] != 0) return;
  const double b = sqrt(d.nrm2[j]);
  d.beta[j] = b;
  d.flag[1] = j + 1;
  if (!isfinite(b)) d.flag[0] = 2;
  else if (b < d.tol_rate) d.flag[0] = 1;
}

__global__ void k_restart_init(KDev d) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    d.flag[0] = 0;
    d.flag[1] = 0;
    d.s[0] = 1.0;
  }
}

// --------------------------------------------------------------------------------------
// K4: w = sum_k V_k coef_k (coef_k = s_k omega_k), in place into column 0 (Eq. 11)
// --------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_combine(const double2* __restrict__ Vbase, int64_t n, int64_t ldv,
                                                      const double2* __restrict__ coefg, int m_eff, double2* out) {
  __shared__ double2 coef[kMaxCols];
  if (threadIdx.x < m_eff) coef[threadIdx.x] = coefg[threadIdx.x];
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x; r < n; r += (int64_t)gridDim.x * kThreads) {
    double2 a = make_double2(0.0, 0.0);
    const double2* Vr = Vbase + r;
    int k = 0;
    for (; k + 8 <= m_eff; k += 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(Vr + (int64_t)(k + u) * ldv);
#pragma unroll
      for (int u = 0; u < 8; ++u) a = cfma(v[u], coef[k + u], a);
    }
    for (; k < m_eff; ++k) a = cfma(__ldcs(Vr + (int64_t)k * ldv), coef[k], a);
    out[r] = a;
  }
}

__global__ void __launch_bounds__(kThreads) k_norm2(KDev d, const double2* __restrict__ x, double* out) {
  double nrm = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x; r < d.n; r += (int64_t)gridDim.x * kThreads) {
    const double2 v = __ldg(x + r);
    nrm = fma(v.x, v.x, fma(v.y, v.y, nrm));
  }
  finish_scalar(d, nrm, 3, out);
}

__global__ void k_copy(const double2* __restrict__ src, double2* __restrict__ dst, int64_t n) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    dst[r] = src[r];
}

__global__ void k_pack(const double2* __restrict__ x, const int32_t* __restrict__ idx, int64_t cnt,
                       double2* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = __ldg(x + idx[t]);
}

// --------------------------------------------------------------------------------------
// setup: CSR validation, Hermiticity, ||H||_1 (= max row abs sum for Hermitian H)
// --------------------------------------------------------------------------------------
template <bool CPLX>
__global__ void k_csr_check(int64_t n, int64_t ncl, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                            const void* valv, int herm, int* err, unsigned long long* norm1_bits) {
  using VT = typename ValT<CPLX>::T;
  const VT* val = static_cast<const VT*>(valv);
  const double eps = 2.220446049250313e-16;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = rowptr[r], hi = rowptr[r + 1];
    int64_t prev = -1;
    double rs = 0.0;
    int e = 0;
    for (int64_t q = lo; q < hi; ++q) {
      const int64_t c = col[q];
      // strictly increasing columns are required of single-rank handles (the Hermiticity search
      // needs them); a distributed handle's local columns keep the caller's global order, which
      // the halo remap does not preserve (validated on the host before the remap, dist.cpp)
      if (c < 0 || c >= ncl || (herm && c <= prev)) { e |= 1; prev = c; continue; }
      prev = c;
      double2 v;
      if constexpr (CPLX) v = val[q]; else v = make_double2(val[q], 0.0);
      const double av = hypot(v.x, v.y);
      rs += av;
      if (!isfinite(av)) e |= 2;
      if (!herm) continue;
      if (c == r) {
        if (fabs(v.y) > 8.0 * eps * av) e |= 2;
        continue;
      }
      int64_t a = rowptr[c], b = rowptr[c + 1] - 1;
      bool found = false;
      while (a <= b) {
        const int64_t mid = (a + b) >> 1;
        const int64_t cm = col[mid];
        if (cm == r) {
          double2 w;
          if constexpr (CPLX) w = val[mid]; else w = make_double2(val[mid], 0.0);
          const double aw = hypot(w.x, w.y);
          if (hypot(v.x - w.x, v.y + w.y) > 8.0 * eps * fmax(av, aw)) e |= 2;
          found = true;
          break;
        }
        if (cm < r) a = mid + 1; else b = mid - 1;
      }
      if (!found) e |= 2;
    }
    if (e) atomicOr(err, e);
    // row abs sums are non-negative: the bit pattern orders like the value (order-free max)
    atomicMax(norm1_bits, (unsigned long long)__double_as_longlong(rs));
  }
}

// --------------------------------------------------------------------------------------
// launchers
// --------------------------------------------------------------------------------------
#define TE_DISPATCH_NCW(ncw, ...)                 \
  switch (ncw) {                                 \
    case 1: { constexpr int NCW = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int NCW = 2; __VA_ARGS__; } break; \
    case 3: { constexpr int NCW = 3; __VA_ARGS__; } break; \
    case 4: { constexpr int NCW = 4; __VA_ARGS__; } break; \
    case 5: { constexpr int NCW = 5; __VA_ARGS__; } break; \
    case 6: { constexpr int NCW = 6; __VA_ARGS__; } break; \
    case 7: { constexpr int NCW = 7; __VA_ARGS__; } break; \
    default: { constexpr int NCW = 8; __VA_ARGS__; } break; \
  }

int kernel_attributes(int which, int* regs, int* max_threads, int* static_smem, int* max_dyn_smem) {
  const void* f = nullptr;
  switch (which) {
    case 0: f = (const void*)k_spmv_tile<false>; break;
    case 1: f = (const void*)k_proj_tma<0>; break;
    case 2: f = (const void*)k_proj_tma<1>; break;
    case 3: f = (const void*)k_update_norm; break;
    case 4: f = (const void*)k_spmv_proj_r<false, 4>; break;
    case 5: f = (const void*)k_update_proj_r<8>; break;
    default: return -1;
  }
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, f) != cudaSuccess) return -2;
  *regs = a.numRegs;
  *max_threads = a.maxThreadsPerBlock;
  *static_smem = (int)a.sharedSizeBytes;
  *max_dyn_smem = a.maxDynamicSharedSizeBytes;
  return 0;
}

cudaError_t configure_kernels() {
  static cudaError_t status = cudaErrorNotReady;
  if (status != cudaErrorNotReady) return status;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaError_t err = cudaSuccess;
  auto set = [&](const void* f, size_t want) {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e == cudaSuccess) {
      const size_t lim = (size_t)optin - a.sharedSizeBytes;
      e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::min(want, lim));
    }
    if (e != cudaSuccess && err == cudaSuccess) err = e;
  };
#define TE_SET(NCW)                                                        \
  set((const void*)k_spmv_proj<false, NCW>, kK1Smem);                      \
  set((const void*)k_spmv_proj<true, NCW>, kK1Smem);                       \
  set((const void*)k_update_proj<NCW>, k2_smem_bytes(kMaxCols, nullptr) + 64 * 1024);
  TE_SET(1) TE_SET(2) TE_SET(3) TE_SET(4) TE_SET(5) TE_SET(6) TE_SET(7) TE_SET(8)
#undef TE_SET
  set((const void*)k_proj_tma<0>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<3>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<0, 8>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<3, 8>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<1, 8>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<0, 16>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<3, 16>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<1, 16>, kProjSmemBudget + 1024);
  set((const void*)k_spmv_tma<false>, kProjSmemBudget + 1024);
#define TE_SETRING_S(T, H, S)                                                              \
  set((const void*)k_spmv_ring<false, T, H, 16, S>, spmv_ring_smem<false, S>());          \
  set((const void*)k_spmv_ring<false, T, H, 12, S>, spmv_ring_smem<false, S>());          \
  set((const void*)k_spmv_ring<true, T, H, 12, S>, spmv_ring_smem<true, S>());            \
  set((const void*)k_spmv_ring<true, T, H, 8, S>, spmv_ring_smem<true, S>());
#define TE_SETRING(T, H) TE_SETRING_S(T, H, 3) TE_SETRING_S(T, H, 4)
  TE_SETRING(1, 0) TE_SETRING(2, 0) TE_SETRING(4, 0) TE_SETRING(8, 0)
  TE_SETRING(1, 1) TE_SETRING(2, 1) TE_SETRING(4, 1) TE_SETRING(8, 1)
  TE_SETRING(1, 2) TE_SETRING(2, 2) TE_SETRING(4, 2) TE_SETRING(8, 2)
#undef TE_SETRING
#undef TE_SETRING_S
#define TE_SETAG(T)                                                                      \
  set((const void*)k_spmv_ag<false, T, false>, spmv_ag_smem<false>());                   \
  set((const void*)k_spmv_ag<true, T, false>, spmv_ag_smem<true>());                     \
  set((const void*)k_spmv_ag<false, T, true>, spmv_ag_smem<false>());                    \
  set((const void*)k_spmv_ag<true, T, true>, spmv_ag_smem<true>());
  TE_SETAG(1) TE_SETAG(2) TE_SETAG(4) TE_SETAG(8) TE_SETAG(16) TE_SETAG(32)
#undef TE_SETAG
#define TE_SETP(T)                                                                   \
  set((const void*)k_spmv_pipe<false, T, 0, 12>, spmv_pipe_smem<false>());           \
  set((const void*)k_spmv_pipe<true, T, 0, 8>, spmv_pipe_smem<true>());              \
  set((const void*)k_spmv_pipe<false, T, 1, 12>, spmv_pipe_smem<false>());           \
  set((const void*)k_spmv_pipe<true, T, 1, 8>, spmv_pipe_smem<true>());              \
  set((const void*)k_spmv_pipe<false, T, 2, 12>, spmv_pipe_smem<false>());           \
  set((const void*)k_spmv_pipe<true, T, 2, 8>, spmv_pipe_smem<true>());              \
  set((const void*)k_spmv_pipe<false, T, 0, 16>, spmv_pipe_smem<false>());           \
  set((const void*)k_spmv_pipe<true, T, 0, 12>, spmv_pipe_smem<true>());             \
  set((const void*)k_spmv_pipe<false, T, 1, 16>, spmv_pipe_smem<false>());           \
  set((const void*)k_spmv_pipe<true, T, 1, 12>, spmv_pipe_smem<true>());             \
  set((const void*)k_spmv_pipe<false, T, 2, 16>, spmv_pipe_smem<false>());           \
  set((const void*)k_spmv_pipe<true, T, 2, 12>, spmv_pipe_smem<true>());
  TE_SETP(1) TE_SETP(2) TE_SETP(4) TE_SETP(8)
#undef TE_SETP
  set((const void*)k_spmv_tma<true>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<1>, kProjSmemBudget + 1024);
  status = err;
  return status;
}

static int tpr_for(int ncols, int min_tpr) {
  int t = min_tpr;
  while (t * kCPT < ncols) t <<= 1;
  return t;
}

#define TE_DISPATCH_TPR(tpr, ...)                               \
  switch (tpr) {                                               \
    case 1: { constexpr int TPR = 1; __VA_ARGS__; } break;     \
    case 2: { constexpr int TPR = 2; __VA_ARGS__; } break;     \
    case 4: { constexpr int TPR = 4; __VA_ARGS__; } break;     \
    default: { constexpr int TPR = 8; __VA_ARGS__; } break;    \
  }

void launch_spmv(const KDev& d, bool cplx, int j, const Launch& L) {
  if (L.spmv_tiled == 7 && d.ntiles_ring > 0) {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(L.num_sms, d.ntiles_ring));
#define TE_RING_S(T, H, S)                                                                                      \
  if (cplx) {                                                                                                   \
    if (L.spmv_nf_wide) k_spmv_ring<true, T, H, 12, S><<<grid, kRingThreads, spmv_ring_smem<true, S>(), L.stream>>>(d, j);   \
    else k_spmv_ring<true, T, H, 8, S><<<grid, kRingThreads, spmv_ring_smem<true, S>(), L.stream>>>(d, j);                   \
  } else {                                                                                                      \
    if (L.spmv_nf_wide) k_spmv_ring<false, T, H, 16, S><<<grid, kRingThreads, spmv_ring_smem<false, S>(), L.stream>>>(d, j); \
    else k_spmv_ring<false, T, H, 12, S><<<grid, kRingThreads, spmv_ring_smem<false, S>(), L.stream>>>(d, j);                \
  }
#define TE_RING_H(T, H) \
  if (L.ring_stages == 3) { TE_RING_S(T, H, 3) } else { TE_RING_S(T, H, 4) }
#define TE_RING(T)                                                                                 \
  case T:                                                                                          \
    if (L.halo_peer) { TE_RING_H(T, 2) } else if (d.halo || L.spmv_force_halo) { TE_RING_H(T, 1) } \
    else { TE_RING_H(T, 0) }                                                                       \
    break;
    switch (L.spmv_ring_tpr) {
      TE_RING(1) TE_RING(2) TE_RING(4)
      default: TE_RING(8)
    }
#undef TE_RING
#undef TE_RING_H
#undef TE_RING_S
    return;
  }
  if (L.spmv_tiled == 6 && d.nslices > 0) {
    const bool hal = d.halo || L.spmv_force_halo;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)8 * L.num_sms, (d.nslices + kWarps - 1) / kWarps));
    if (cplx) {
      if (hal) k_spmv_sell<true, true, 4><<<grid, kThreads, 0, L.stream>>>(d, j);
      else k_spmv_sell<true, false, 4><<<grid, kThreads, 0, L.stream>>>(d, j);
    } else {
      if (hal) k_spmv_sell<false, true, 4><<<grid, kThreads, 0, L.stream>>>(d, j);
      else k_spmv_sell<false, false, 4><<<grid, kThreads, 0, L.stream>>>(d, j);
    }
    return;
  }
  if (L.spmv_tiled == 5 && d.ntiles_ag > 0) {
    const bool hal = d.halo || L.spmv_force_halo;
    // persistent grid = co-resident blocks (occupancy API, cached per instantiation)
    auto grid_of = [&](const void* f, size_t smem) {
      static std::vector<std::pair<const void*, int>> cache;
      int per_sm = 0;
      for (auto& c : cache)
        if (c.first == f) per_sm = c.second;
      if (per_sm == 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, kThreads, smem) != cudaSuccess || per_sm < 1)
          per_sm = 1;
        cache.emplace_back(f, per_sm);
      }
      return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * L.num_sms, d.ntiles_ag));
    };
#define TE_AG_H(T, H)                                                                                        \
  if (cplx) {                                                                                                \
    const int grid = grid_of((const void*)k_spmv_ag<true, T, H>, spmv_ag_smem<true>());                     \
    k_spmv_ag<true, T, H><<<grid, kThreads, spmv_ag_smem<true>(), L.stream>>>(d, j);                         \
  } else {                                                                                                   \
    const int grid = grid_of((const void*)k_spmv_ag<false, T, H>, spmv_ag_smem<false>());                   \
    k_spmv_ag<false, T, H><<<grid, kThreads, spmv_ag_smem<false>(), L.stream>>>(d, j);                       \
  }
#define TE_AG(T)                                            \
  case T:                                                   \
    if (hal) { TE_AG_H(T, true) } else { TE_AG_H(T, false) } \
    break;
    switch (L.spmv_ag_tpr) {
      TE_AG(1) TE_AG(2) TE_AG(4) TE_AG(8) TE_AG(16)
      default: TE_AG(32)
    }
#undef TE_AG
#undef TE_AG_H
    return;
  }
  if (L.spmv_tiled == 4 && d.ntiles > 0) {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(2 * L.num_sms, d.ntiles));
    switch (L.spmv_pipe_tpr) {
#define TE_PIPE_NF(T, H, NR, NC)                                                                     \
  if (cplx) k_spmv_pipe<true, T, H, NC><<<grid, kThreads, spmv_pipe_smem<true>(), L.stream>>>(d, j, L.spmv_pf); \
  else k_spmv_pipe<false, T, H, NR><<<grid, kThreads, spmv_pipe_smem<false>(), L.stream>>>(d, j, L.spmv_pf);
#define TE_PIPE(T)                                                                                  \
  case T:                                                                                           \
    if (L.halo_peer) {                                                                              \
      if (L.spmv_nf_wide) { TE_PIPE_NF(T, 2, 16, 12) } else { TE_PIPE_NF(T, 2, 12, 8) }            \
    } else if (d.halo || L.spmv_force_halo) {                                                       \
      if (L.spmv_nf_wide) { TE_PIPE_NF(T, 1, 16, 12) } else { TE_PIPE_NF(T, 1, 12, 8) }            \
    } else {                                                                                        \
      if (L.spmv_nf_wide) { TE_PIPE_NF(T, 0, 16, 12) } else { TE_PIPE_NF(T, 0, 12, 8) }            \
    }                                                                                               \
    break;
      TE_PIPE(1) TE_PIPE(2) TE_PIPE(4)
      default: TE_PIPE(8)
#undef TE_PIPE
#undef TE_PIPE_NF
    }
    return;
  }
  if (L.spmv_tiled == 3 && d.ntiles > 0) {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(8 * L.num_sms, d.ntiles));
    if (cplx) k_spmv_rowtile<true><<<grid, kThreads, 0, L.stream>>>(d, j);
    else k_spmv_rowtile<false><<<grid, kThreads, 0, L.stream>>>(d, j);
    return;
  }
  if (L.spmv_tiled == 2 && d.ntiles_desc > 0) {
    const int S = spmv_slots(cplx);
    if (cplx) k_spmv_tma<true><<<L.num_sms, kProjThreads, spmv_smem_bytes(true), L.stream>>>(d, j, S);
    else k_spmv_tma<false><<<L.num_sms, kProjThreads, spmv_smem_bytes(false), L.stream>>>(d, j, S);
    return;
  }
  if (L.spmv_tiled && d.ntiles > 0) {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(8 * L.num_sms, d.ntiles));
    if (cplx) k_spmv_tile<true><<<grid, kThreads, 0, L.stream>>>(d, j);
    else k_spmv_tile<false><<<grid, kThreads, 0, L.stream>>>(d, j);
    return;
  }
  const int tpr = L.spmv_tpr;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(8 * L.num_sms, (d.n * tpr + kThreads - 1) / kThreads));
    switch (tpr) {
#define TE_SPMV(T)                                                                      \
  case T:                                                                               \
    if (cplx) k_spmv<true, T><<<grid, kThreads, 0, L.stream>>>(d, j);                   \
    else k_spmv<false, T><<<grid, kThreads, 0, L.stream>>>(d, j);                       \
    break;
      TE_SPMV(1) TE_SPMV(2) TE_SPMV(4) TE_SPMV(8) TE_SPMV(16)
      default: TE_SPMV(32)
#undef TE_SPMV
    }
}

static void launch_proj_s(const KDev& d, int j, int mode, const Launch& L) {
  const int tpr = tpr_for(j + 1, 1);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4 * L.num_sms, (d.n * tpr + kThreads - 1) / kThreads));
  TE_DISPATCH_TPR(tpr, {
    if (mode == 0) k_proj_s<0, TPR><<<grid, kThreads, 0, L.stream>>>(d, j);
    else k_proj_s<1, TPR><<<grid, kThreads, 0, L.stream>>>(d, j);
  });
}

// measured on B200 (tools/micro/mb_proj.cu, 16 KB minimum TMA tiles): the register/shuffle kernel
// is faster for the dots up to 4 columns and for the update up to 5 columns, the TMA ring above;
// the TMA ring keeps per-lane register column sums for the smallest of 8 / 16 / 32 columns that
// covers ncols (fewer live registers at small ncols: 8 columns, update 3.7 -> 4.7 TB/s)
constexpr int kShuffleMaxColsDots = 4;
constexpr int kShuffleMaxCols = 5;

#define TE_PROJ_TMA(MODE, ncols, ...)                                                                   \
  do {                                                                                                  \
    if ((ncols) <= 8) k_proj_tma<MODE, 8><<<L.num_sms, kProjThreads, proj_smem_bytes(ncols), L.stream>>>(__VA_ARGS__);      \
    else if ((ncols) <= 16) k_proj_tma<MODE, 16><<<L.num_sms, kProjThreads, proj_smem_bytes(ncols), L.stream>>>(__VA_ARGS__); \
    else k_proj_tma<MODE, 32><<<L.num_sms, kProjThreads, proj_smem_bytes(ncols), L.stream>>>(__VA_ARGS__);                   \
  } while (0)

void launch_proj_dots(const KDev& d, int j, const Launch& L) {
  if (L.proj_tma == 0 || (L.proj_tma == 2 && j + 1 <= kShuffleMaxColsDots)) {
    launch_proj_s(d, j, 0, L);
    return;
  }
  const int S = proj_slots(j + 1), R = proj_rsub(j + 1), C = proj_consumers(j + 1);
  TE_PROJ_TMA(0, j + 1, L.tmaps[j], d, j, S, R, C, 0);
}

void launch_gram_update(const KDev& d, int j, bool write, const Launch& L) {
  const int S = proj_slots(j + 1), R = proj_rsub(j + 1), C = proj_consumers(j + 1);
  TE_PROJ_TMA(3, j + 1, L.tmaps[j], d, j, S, R, C, write ? 1 : 0);
}

void launch_spmv_proj(const KDev& d, bool cplx, int j, const Launch& L) {
  if (L.variant == 2) {
    launch_spmv(d, cplx, j, L);
    launch_proj_dots(d, j, L);
    return;
  }
  if (L.variant == 0) {

    const int tpr = tpr_for(j + 1, 4);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(2 * L.num_sms, (d.n * tpr + kThreads - 1) / kThreads));
    TE_DISPATCH_TPR(tpr, {
      if (cplx)
        k_spmv_proj_r<true, TPR><<<grid, kThreads, 0, L.stream>>>(d, j, L.prefetch);
      else
        k_spmv_proj_r<false, TPR><<<grid, kThreads, 0, L.stream>>>(d, j, L.prefetch);
    });
    return;
  }
  const int ncw = (j + 1 + kWarps - 1) / kWarps;
  TE_DISPATCH_NCW(ncw, {
    if (cplx)
      k_spmv_proj<true, NCW><<<L.grid_k1, kThreads, kK1Smem, L.stream>>>(d, j);
    else
      k_spmv_proj<false, NCW><<<L.grid_k1, kThreads, kK1Smem, L.stream>>>(d, j);
  });
}

void launch_update_proj(const KDev& d, int j, const Launch& L) {
  if (L.variant == 2 && (L.proj_tma == 0 || (L.proj_tma == 2 && j + 1 <= kShuffleMaxCols))) {
    launch_proj_s(d, j, 1, L);
    return;
  }
  if (L.variant == 2) {
    const int S = proj_slots(j + 1), R = proj_rsub(j + 1), C = proj_consumers(j + 1);
    TE_PROJ_TMA(1, j + 1, L.tmaps[j], d, j, S, R, C, 0);
    return;
  }
  if (L.variant == 0) {
    const int tpr = tpr_for(j + 1, 1);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(2 * L.num_sms, (d.n * tpr + kThreads - 1) / kThreads));
    TE_DISPATCH_TPR(tpr, { k_update_proj_r<TPR><<<grid, kThreads, 0, L.stream>>>(d, j, L.prefetch); });
    return;
  }
  int tr = 0;
  const size_t smem = k2_smem_bytes(j + 1, &tr);
  const int64_t ntiles = (d.n + tr - 1) / tr;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(L.grid_k2, ntiles));
  const int ncw = (j + 1 + kWarps - 1) / kWarps;
  TE_DISPATCH_NCW(ncw, { k_update_proj<NCW><<<grid, kThreads, smem, L.stream>>>(d, j, tr); });
}

void launch_update_norm(const KDev& d, int j, bool write, const Launch& L) {
  k_update_norm<<<L.grid_k3, kThreads, 0, L.stream>>>(d, j, write ? 1 : 0, L.prefetch);
}

void launch_finalize(const KDev& d, int j, const Launch& L) { k_finalize<<<1, 32, 0, L.stream>>>(d, j); }

void launch_restart_init(const KDev& d, const Launch& L) { k_restart_init<<<1, 32, 0, L.stream>>>(d); }

void launch_combine(const KDev& d, const double2* coef, int m_eff, double2* out, const Launch& L) {
  k_combine<<<L.grid_k3, kThreads, 0, L.stream>>>(d.V, d.n, d.ldv, coef, m_eff, out);
}

void launch_norm2(const KDev& d, const double2* x, double* out, const Launch& L) {
  k_norm2<<<L.grid_k3, kThreads, 0, L.stream>>>(d, x, out);
}

void launch_copy_col(const double2* src, double2* dst, int64_t n, cudaStream_t st) {
  int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  if (grid < 1) grid = 1;
  k_copy<<<grid, 256, 0, st>>>(src, dst, n);
}

void launch_pack(const double2* x, const int32_t* idx, int64_t cnt, double2* out, cudaStream_t st) {
  if (cnt <= 0) return;
  int grid = (int)std::min<int64_t>((cnt + 255) / 256, 148 * 8);
  k_pack<<<grid, 256, 0, st>>>(x, idx, cnt, out);
}

void launch_csr_check(int64_t n, int64_t ncl, const int64_t* rowptr, const int32_t* col, const void* val, bool cplx,
                      bool hermitian_check, CsrCheck c, cudaStream_t st) {
  int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (grid < 1) grid = 1;
  if (cplx)
    k_csr_check<true><<<grid, 256, 0, st>>>(n, ncl, rowptr, col, val, hermitian_check, c.err, c.norm1_bits);
  else
    k_csr_check<false><<<grid, 256, 0, st>>>(n, ncl, rowptr, col, val, hermitian_check, c.err, c.norm1_bits);
}

}  // namespace te
