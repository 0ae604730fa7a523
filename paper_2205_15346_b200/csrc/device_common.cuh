// Device helpers shared by the hot-path kernels (kernels.cu: projections, update, norm, V.omega;
// spmv.cu: the SpMV variants): complex arithmetic, mbarrier / bulk-copy / 2-D TMA wrappers,
// cp.async wrappers, warp and lane-group reductions, the step gate (beta_{j-1}, scale s_j,
// breakdown flag) and the deterministic last-block reductions.  All inline.
#pragma once
#include "kernels.cuh"

#include <cuda.h>

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
  const double b = sqrt(d.defer ? d.gsync[0].x : d.nrm2[j - 1]);
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

// The step-j gate decision as a pure function (every thread of a deferred update kernel evaluates it
// from the same loads, in parallel with its coefficient loads; block 0 / thread 0 also runs
// step_gate for the side effects, reaching the same decision)
__device__ __forceinline__ double gate_value(const KDev& d, int j, int flag0, double nrm_prev) {
  if (flag0 != 0) return 0.0;
  if (j == 0) return 1.0;
  const double b = sqrt(nrm_prev);
  if (!isfinite(b) || b < d.tol_rate) return 0.0;
  return 1.0 / b;
}

// Gate of the SpMV of step j: in defer mode (CGS2, f2) only the breakdown flag of earlier steps
// (the SpMV writes H V_j unscaled; the update kernel applies s_j), else the full step gate.
__device__ __forceinline__ double spmv_gate(const KDev& d, int j, bool writer) {
  if (d.defer) return d.flag[0] != 0 ? 0.0 : 1.0;
  return step_gate(d, j, writer);
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


// halo entry hi of step j from the owning rank's V column (uncached: written by another GPU)
__device__ __forceinline__ double2 peer_x(const KDev& d, int j, int hi) {
  const int q = __ldg(d.halo_owner + hi);
  const double2* base = d.peer_base[q];
  return __ldcv(base + (int64_t)j * __ldg(d.peer_ldv + q) + __ldg(d.halo_lidx + hi));
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

constexpr int kTileR = 32;          // rows per consumer sub-tile (lane = row)
constexpr int kConsumers = 7;       // consumer warps (+1 producer warp = 256 threads)
constexpr int kMaxSlots = 32;
constexpr int kProjThreads = (kConsumers + 1) * 32;
constexpr size_t kProjSmemBudget = 200 * 1024;

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


}  // namespace te
