// SpMV kernels for sm_100a: p = s_j H V_j (Eq. 8, first line; columns stored unnormalised,
// s_j applied on the output), CSR with int32 columns and real or complex values, x = column j of
// V (plus, with several ranks, the halo: staged by the NCCL exchange or read from peer memory).
//   7 k_spmv_ring  (default) warp-specialised: producer warp + 15 consumer warps, 3-4 stage
//                  bulk-copy ring of nnz-balanced tiles, per-warp stage release
//   4 k_spmv_pipe  the same tiles double-buffered per 8-warp block, block barrier per tile
//   6 k_spmv_sell  SELL-32-sigma copy of H, software-pipelined coalesced loads
//   5 k_spmv_ag    x gathers as cp.async copies into shared memory
//   3 k_spmv_rowtile, 1 k_spmv_tile, 2 k_spmv_tma, 0 k_spmv (CSR-vector): earlier variants
// All variants sum each row's products in a fixed order (deterministic); parity-tested against
// the oracle in tests/test_gpu_parity.py; measurements in DESIGN.md §6.
#include "device_common.cuh"

#include <algorithm>
#include <cstdio>
#include <utility>
#include <vector>

namespace te {

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


void configure_spmv_kernels(void (*set_attr)(const void*, size_t, void*), void* ctx) {
  auto set = [&](const void* f, size_t want) { set_attr(f, want, ctx); };
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
}

// the default SpMV as launched for a real matrix with one lane per row (config 2)
const void* spmv_attr_kernel() { return (const void*)k_spmv_ring<false, 1, 0, 16, 4>; }

}  // namespace te
