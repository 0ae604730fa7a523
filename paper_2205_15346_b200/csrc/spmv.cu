// SpMV kernels for sm_100a: p = s_j H V_j (Eq. 8, first line; columns stored unnormalised,
// s_j applied on the output), CSR with int32 columns and real or complex values, x = column j of
// V (plus, with several ranks, the halo: staged by the NCCL exchange or read from peer memory).
//   7 k_spmv_ring  (default) warp-specialised: producer warp + 15 consumer warps, 3-4 stage
//                  bulk-copy ring of nnz-balanced tiles, per-warp stage release
//   6 k_spmv_sell  SELL-32-sigma copy of H, software-pipelined coalesced loads
//   8 k_spmv_xs    (spmv_xs.cu) the ring with each tile's x windows staged by bulk copies
//   9 k_spmv_sw    (spmv_sw.cu) slot-window SELL-32 with a value dictionary (2 bytes per entry)
//  10 the ring over a column-blocked copy of H: one pass per column block of x (x block
//     L2-resident while the pass gathers from it), passes > 0 accumulate into W
// The variants measured slower in round 1 (CSR-vector, row tiles, TMA slots, block-pipelined,
// async gather; DESIGN.md §6 keeps their numbers) were removed from the library.
// All variants sum each row's products in a fixed order (deterministic); parity-tested against
// the oracle in tests/test_gpu_parity.py; measurements in DESIGN.md §6.
#include "device_common.cuh"

#include <algorithm>
#include <cstdio>
#include <utility>
#include <vector>

namespace te {


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

// row result: W = s_j acc, or W += s_j acc in the passes > 0 of the column-blocked SpMV
__device__ __forceinline__ void ring_out(const KDev& d, int64_t r, double2 acc, double sj) {
  double2 v = make_double2(acc.x * sj, acc.y * sj);
  if (d.accw) v = cadd(__ldcs(d.W + r), v);
  __stcs(d.W + r, v);
}

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
    sj_s = spmv_gate(d, j, blockIdx.x == 0);
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
      // (loading the next descriptor before the wait, as the staged-x producer does, measured no
      // gain on configs 2 / 5 and -7 % on config 6: kept simple)
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
      if (act && q == 0) ring_out(d, ra + i, acc, sj);
    } else if (warp == (int)(t % kRingConsumers)) {  // one long row: one warp, from global memory
      const VT* __restrict__ val = static_cast<const VT*>(d.val);
      double2 acc = make_double2(0.0, 0.0);
      for (int64_t k = b + lane; k < e; k += 32) acc = cadd(acc, ValT<CPLX>::mul(__ldg(val + k), gx(__ldg(d.col + k))));
      acc = warp_sum(acc);
      if (lane == 0) ring_out(d, ra, acc, sj);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
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
  if (threadIdx.x == 0) sj_s = spmv_gate(d, j, blockIdx.x == 0);
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

// Halo part of a distributed SpMV: W[r] += s_j sum_k H_{r,c_k} x_halo[c_k] over the entries of row
// r whose columns live on other ranks (x_halo: the received halo vector, or the owning rank's V
// column through peer memory).  Runs after the local-column SpMV of the same step, so each row's
// sum is (its local entries in CSR order) + (its halo entries in CSR order): deterministic.
template <bool CPLX, bool PEER>
__global__ void __launch_bounds__(kThreads) k_spmv_halo(KDev d, int j) {
  using VT = typename ValT<CPLX>::T;
  __shared__ double sj_s;
  if (threadIdx.x == 0) sj_s = d.flag[0] != 0 ? 0.0 : (d.defer || j == 0 ? 1.0 : d.s[j]);
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;
  const VT* __restrict__ hv = static_cast<const VT*>(d.hval);
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < d.nh; i += (int64_t)gridDim.x * kThreads) {
    const int64_t a = __ldg(d.hrowptr + i), b = __ldg(d.hrowptr + i + 1);
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t k = a; k < b; ++k) {
      const int c = __ldg(d.hcol + k);
      const double2 xv = PEER ? peer_x(d, j, c) : __ldg(d.halo + c);
      acc = cadd(acc, ValT<CPLX>::mul(__ldg(hv + k), xv));
    }
    const int r = __ldg(d.hrow + i);
    const double2 w = d.W[r];
    d.W[r] = make_double2(w.x + sj * acc.x, w.y + sj * acc.y);
  }
}

void launch_spmv_halo(const KDev& d, bool cplx, int j, const Launch& L) {
  if (d.nh <= 0) return;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)8 * L.num_sms, (d.nh + kThreads - 1) / kThreads));
  if (cplx) {
    if (L.halo_peer) k_spmv_halo<true, true><<<grid, kThreads, 0, L.stream>>>(d, j);
    else k_spmv_halo<true, false><<<grid, kThreads, 0, L.stream>>>(d, j);
  } else {
    if (L.halo_peer) k_spmv_halo<false, true><<<grid, kThreads, 0, L.stream>>>(d, j);
    else k_spmv_halo<false, false><<<grid, kThreads, 0, L.stream>>>(d, j);
  }
}

void launch_spmv(const KDev& d, bool cplx, int j, const Launch& L) {
  if (L.spmv_tiled == 9 && d.sw_nslice > 0) {
    launch_spmv_sw(d, cplx, j, L);
    return;
  }
  if (L.spmv_tiled == 8 && d.ntiles_xs > 0) {
    launch_spmv_xs(d, cplx, j, L);
    return;
  }
  if (L.spmv_tiled == 6 && d.nslices > 0) {
    const bool hal = L.spmv_force_halo;
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
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(L.grid_spmv, d.ntiles_ring));
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
    if (L.spmv_force_halo) { TE_RING_H(T, 1) }                                                    \
    else { TE_RING_H(T, 0) }                                                                       \
    break;
  switch (L.spmv_ring_tpr) {
    TE_RING(1) TE_RING(2) TE_RING(4)
    default: TE_RING(8)
  }
#undef TE_RING
#undef TE_RING_H
#undef TE_RING_S
}


void configure_spmv_kernels(void (*set_attr)(const void*, size_t, void*), void* ctx) {
  auto set = [&](const void* f, size_t want) { set_attr(f, want, ctx); };
#define TE_SETRING_S(T, H, S)                                                              \
  set((const void*)k_spmv_ring<false, T, H, 16, S>, spmv_ring_smem<false, S>());          \
  set((const void*)k_spmv_ring<false, T, H, 12, S>, spmv_ring_smem<false, S>());          \
  set((const void*)k_spmv_ring<true, T, H, 12, S>, spmv_ring_smem<true, S>());            \
  set((const void*)k_spmv_ring<true, T, H, 8, S>, spmv_ring_smem<true, S>());
#define TE_SETRING(T, H) TE_SETRING_S(T, H, 3) TE_SETRING_S(T, H, 4)
  TE_SETRING(1, 0) TE_SETRING(2, 0) TE_SETRING(4, 0) TE_SETRING(8, 0)
  TE_SETRING(1, 1) TE_SETRING(2, 1) TE_SETRING(4, 1) TE_SETRING(8, 1)
#undef TE_SETRING
#undef TE_SETRING_S
  configure_xs_kernels(set_attr, ctx, kXsBudget);
}

// the default SpMV as launched for a real matrix with one lane per row (config 2)
// ------------------------------------------------------------------------------------------
// column-blocked CSR build (variant 10): block b holds the entries with columns in
// [b B, (b+1) B); within a row they are a contiguous run of the sorted CSR row
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ int64_t row_lower_bound(const int32_t* __restrict__ col, int64_t lo, int64_t hi, int64_t c) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)col[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__global__ void k_colblk_count(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col, int64_t B,
                               int nb, int32_t* cnt) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = rowptr[r], e = rowptr[r + 1];
    int64_t lo = a;
    for (int b = 0; b < nb; ++b) {
      const int64_t hi = b + 1 < nb ? row_lower_bound(col, lo, e, (int64_t)(b + 1) * B) : e;
      cnt[(int64_t)b * n + r] = (int32_t)(hi - lo);
      lo = hi;
    }
  }
}
template <bool CPLX>
__global__ void k_colblk_fill(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                              const void* __restrict__ val, int64_t B, int b, const int64_t* __restrict__ rowptr_b,
                              int32_t* col_b, void* val_b) {
  using VT = typename ValT<CPLX>::T;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = rowptr[r], e = rowptr[r + 1];
    const int64_t lo = b > 0 ? row_lower_bound(col, a, e, (int64_t)b * B) : a;
    const int64_t hi = row_lower_bound(col, lo, e, (int64_t)(b + 1) * B);
    int64_t o = rowptr_b[r];
    for (int64_t k = lo; k < hi; ++k, ++o) {
      col_b[o] = col[k];
      static_cast<VT*>(val_b)[o] = static_cast<const VT*>(val)[k];
    }
  }
}
void launch_colblk_count(int64_t n, const int64_t* rowptr, const int32_t* col, int64_t B, int nb, int32_t* cnt,
                         cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, (n + 255) / 256));
  k_colblk_count<<<grid, 256, 0, st>>>(n, rowptr, col, B, nb, cnt);
}
void launch_colblk_fill(int64_t n, const int64_t* rowptr, const int32_t* col, const void* val, bool cplx, int64_t B,
                        int b, const int64_t* rowptr_b, int32_t* col_b, void* val_b, cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, (n + 255) / 256));
  if (cplx) k_colblk_fill<true><<<grid, 256, 0, st>>>(n, rowptr, col, val, B, b, rowptr_b, col_b, val_b);
  else k_colblk_fill<false><<<grid, 256, 0, st>>>(n, rowptr, col, val, B, b, rowptr_b, col_b, val_b);
}

const void* spmv_attr_kernel() { return (const void*)k_spmv_ring<false, 1, 0, 16, 4>; }

}  // namespace te
