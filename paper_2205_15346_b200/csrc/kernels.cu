// Hot-path CUDA kernels for sm_100a besides the SpMV (spmv.cu): one Arnoldi/CGS2 step (Eq. 8,
// P:146-162, classical Gram-Schmidt + one re-orthogonalisation, reading C1 of DESIGN.md) after the
// SpMV, and the restart assembly V.omega (Eq. 11):
//   proj_dots   g1 = V^H p                        k_proj_tma<0> (TMA ring) / k_proj_r<0> (registers)
//   update_proj p' = p - V e1, g2 = V^H p'         k_proj_tma<1> / k_proj_r<1>
//   update_norm p'' = p' - V e2 -> column j+1, ||p''||^2      k_update_norm
//   combine     w = V (s omega), in place into column 0          k_combine
// plus the f1 (paper-literal Lanczos) and f2 (Gram second sweep, k_proj_tma<3>) kernels,
// validation and small helpers (round 1's fused kernel sets 0/1 measured slower and were removed).  e_k = s_k^2 g_k (s_k = 1/||V_k||: columns
// are stored unnormalised and scaled on the fly).  Reductions are deterministic: per-CTA partials,
// then the last CTA to finish (integer ticket) sums them in a fixed order; no floating-point atomics.
#include "device_common.cuh"

#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <vector>

namespace te {

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
// Slot s is owned by warp s % C, so unless C divides S some warps own one slot more and process
// more tiles: 9 slots over 7 warps give two warps 2/9 of the tiles (64 % balance).  The slot count
// is rounded down to a multiple of C when that keeps >= 3/4 of the slots (8, 9 -> 7; 11, 12 kept:
// there the deeper ring wins).  Measured (tools/micro/mb_proj.cu, update pass, n = 2^23): 20
// columns 5.4 -> 6.2 TB/s, 24: 5.0 -> 6.5, 40: 4.8 -> 5.7, 48: 4.8 -> 6.2; 8, 16, 32 columns (11-12
// slots) lost 0.4-0.6 TB/s when rounded to 7, so they keep their slots.  g_proj_balance = 0: off.
int g_proj_balance = 1;
int proj_slots(int ncols) {
  int s = (int)(kProjSmemBudget / proj_slot_bytes(ncols));
  s = s > kMaxSlots ? kMaxSlots : (s < 1 ? 1 : s);
  if (g_proj_balance && s > kConsumers) {
    const int sb = s / kConsumers * kConsumers;
    if (4 * sb >= 3 * s) s = sb;
  }
  return s;
}
int proj_consumers(int ncols) {
  const int s = proj_slots(ncols);
  return s < kConsumers ? s : kConsumers;
}
size_t proj_smem_bytes(int ncols) { return (size_t)proj_slots(ncols) * proj_slot_bytes(ncols) + 1024; }

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
// RT: the sub-tile count R as a compile-time constant (0: the runtime argument).  With a constant
// tile stride the column loads of a lane become one base register plus immediate offsets; the
// runtime-R build spends 3 of its ~9 instructions per column on address arithmetic (SASS: LDC R,
// IMAD, IMAD.WIDE per LD.E.128), and the consumers are issue/latency-bound (8 warps per SM).
template <int MODE, int NREG = 32, int MINB = 1, int RT = 0>
__global__ void __launch_bounds__(kProjThreads, MINB)
    k_proj_tma(const __grid_constant__ CUtensorMap tmV, KDev d, int j, int S, int R_arg, int C, int write) {
  const int R = RT > 0 ? RT : R_arg;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxSlots], empty[kMaxSlots];
  __shared__ double2 coef[kMaxCols];
  __shared__ double2 red[kConsumers][kMaxCols];
  __shared__ int go_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncols = j + 1;
  __shared__ double2 c1s[kMaxCols];
  __shared__ double nrm_s[kConsumers];
  __shared__ double sj_s;
  // MODE 1 / 3 run the deferred gate of step j (device_common.cuh step_gate: s_j from the reduced
  // ||p''_{j-1}||^2, breakdown test; block 0 records beta_{j-1}, s_j and, for f2, Gram row j):
  // W holds H V_j unscaled, g1 its raw dots, so p' = s_j (W - V e1') with e1'_k = s_k^2 g1_k
  const double sj = (MODE == 1 || MODE == 3) ? gate_value(d, j, d.flag[0], d.gsync[0].x) : (d.flag[0] == 0 ? 1.0 : 0.0);
  if (tid == 0) {
    if ((MODE == 1 || MODE == 3) && blockIdx.x == 0) step_gate(d, j, true);
    sj_s = sj;
    go_s = sj != 0.0;
  }
  if (MODE == 1 && tid < ncols) {
    const double sk = tid == j ? sj : d.s[tid];
    const double2 g = d.g1[tid];
    coef[tid] = make_double2(sk * sk * g.x, sk * sk * g.y);   // e1'_k = s_k^2 g1_k
  }
  if (MODE == 4) {  // K3 on the TMA ring: p'' = p' - V e2' (e2'_k = s_k^2 g2_k) -> column j + 1, ||p''||^2
    if (tid < ncols) {
      const double sk = d.s[tid];
      const double2 g = d.g2[tid];
      coef[tid] = make_double2(sk * sk * g.x, sk * sk * g.y);
    }
    if (tid == 0 && blockIdx.x == 0 && sj != 0.0) {  // alpha_j = Re(c1_j + c2_j) (reading C2)
      const double s_j = d.s[j];
      d.alpha[j] = s_j * (s_j * d.g1[j].x + d.g2[j].x);
    }
  }
  if (MODE == 3) {  // f2: c1' = s g1, c2' = c1' - G c1', coefficient on raw V_k: s_k (c1'_k + c2'_k)
    if (tid < ncols) {
      const double sk = tid == j ? sj : d.s[tid];
      const double2 g = d.g1[tid];
      c1s[tid] = make_double2(sk * g.x, sk * g.y);
    }
    __syncthreads();
    if (tid < ncols && go_s) {
      // Gram entries: rows/columns < j from earlier gates (global), row/column j formed here from
      // the reduced dots of the previous update pass (the same values block 0's gate stores)
      double2 gc = make_double2(0.0, 0.0);
      for (int l = 0; l < ncols; ++l) {
        double2 G;
        if (l == tid) {
          G = make_double2(1.0, 0.0);
        } else if (tid < j && l < j) {
          G = d.G[tid * kMaxCols + l];
        } else if (l == j) {
          const double sk = d.s[tid] * sj;
          const double2 g = d.g2[tid];
          G = make_double2(sk * g.x, sk * g.y);
        } else {
          const double sk = d.s[l] * sj;
          const double2 g = d.g2[l];
          G = make_double2(sk * g.x, -sk * g.y);
        }
        gc = cfma(G, c1s[l], gc);
      }
      const double2 c1 = c1s[tid];
      const double2 c = make_double2(c1.x + (c1.x - gc.x), c1.y + (c1.y - gc.y));
      const double sk = tid == j ? sj : d.s[tid];
      coef[tid] = make_double2(sk * c.x, sk * c.y);
      if (tid == j && blockIdx.x == 0) d.alpha[j] = sj * c.x;  // Re(c1_j + c2_j) = s_j Re(c1'_j + c2'_j)
    }
  }
  // 1024-B alignment of the slot ring.  Dots and update + norm passes (MODE 0, 4): through an integer
  // cast, so that the consumers read the tiles with generic LD.E.128 — measured faster there than
  // LDS.128 (round 1: dots at 23 columns 6.0 vs 4.2 TB/s; this round with the compile-time tile
  // stride: equal within 1 %).  Update + dots passes (MODE 1, 3): LDS.128 — with the compile-time
  // stride the LDS build no longer spills and wins (config 5: 6.10 -> 6.39 TB/s, config 2: 5.40 -> 5.49);
  // the runtime-R fallback keeps the generic loads (its LDS build spills: 4.3-5.2 TB/s)
  unsigned char* smem;
  if constexpr ((MODE == 1 || MODE == 3) && RT > 0)  // shared address space kept: LDS.128 tile reads (see above)
    smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  else
    smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
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
    double2* outV = ((MODE == 3 || MODE == 4) && write) ? d.V + (int64_t)(j + 1) * d.ldv : nullptr;
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
#pragma unroll 1
        for (int sub = 0; sub < R && MODE != 2; ++sub) {  // MODE 2: streaming only (microbenchmark)
          const int row = sub * kTileR + lane;
          if (sub * kTileR >= rows) break;  // warp-uniform
          double2 p = row < rows ? Ws[row] : make_double2(0.0, 0.0);
          if (MODE == 1 || MODE == 3 || MODE == 4) {
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
            p = make_double2(sj * (p.x - a.x), sj * (p.y - a.y));
            if (row >= rows) p = make_double2(0.0, 0.0);
            else if (MODE == 1) d.W[r0 + row] = p;
            else {
              if (outV) outV[r0 + row] = p;
              nrm = fma(p.x, p.x, fma(p.y, p.y, nrm));
            }
          }
          if constexpr (MODE == 4) continue;  // no dots in the update + norm pass
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
    if constexpr (MODE != 4) {
      const double2 acc0 = colsum_reg<NREG>(aR, aI);
      if (lane < NREG) red[warp][lane] = acc0;
      if (lane < 16) {
        const double2 ab[4] = {accb0, accb1, accb2, accb3};
#pragma unroll
        for (int g = 0; g < 4; ++g)
          if (NREG + 16 * g + lane < kMaxCols) red[warp][NREG + 16 * g + lane] = ab[g];
      }
    }
    if (MODE == 3 || MODE == 4) {
      nrm = warp_sum(nrm);
      if (lane == 0) nrm_s[warp] = nrm;
    }
  }
  __syncthreads();
  // block partial in fixed warp order, then the last-CTA reduction
  double2* out = MODE == 0 ? d.g1 : d.g2;
  const int ctr = MODE == 0 ? 0 : (MODE == 4 ? 2 : 1);
  if (MODE != 4 && tid < ncols) {
    double2 t = red[0][tid];
    for (int w = 1; w < C; ++w) t = cadd(t, red[w][tid]);
    d.part[(size_t)blockIdx.x * kMaxCols + tid] = t;
  }
  if ((MODE == 3 || MODE == 4) && tid == 0) {
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
  if (MODE != 4) {
    const int c = tid & (kMaxCols - 1), sgi = tid >> 6;
    double2 sm = make_double2(0.0, 0.0);
    if (c < ncols) {
      const int b0 = sgi * per, b1 = min(G, b0 + per);
      for (int b = b0; b < b1; ++b) sm = cadd(sm, ld_cg(d.part + (size_t)b * kMaxCols + c));
    }
    seg[sgi][c] = sm;
  }
  __syncthreads();
  if (MODE != 4 && tid < ncols) {
    double2 t = seg[0][tid];
    t = cadd(t, seg[1][tid]);
    t = cadd(t, seg[2][tid]);
    t = cadd(t, seg[3][tid]);
    out[tid] = t;
  }
  if ((MODE == 3 || MODE == 4) && tid == 0) {  // ||p''||^2 in fixed block order
    double t = 0.0;
    for (int b = 0; b < G; ++b) t += __ldcg(d.partn + b);
    d.nrm2[j] = t;
  }
  // ||p''_{j-1}||^2 rides with g1 in the step's first reduction (defer mode)
  if (MODE == 0 && tid == 0) d.gsync[0] = make_double2(j > 0 ? d.nrm2[j - 1] : 0.0, 0.0);
  if (tid == 0) d.counter[ctr] = 0u;
}

// --------------------------------------------------------------------------------------
// Register-accumulator projection kernel (CGS2 passes K1b/K2 up to kRegMaxCols columns):
// plain register streaming like k_update_norm (no shared-memory staging, 16 warps per SM),
// with persistent per-lane column sums.  Lane (rg, q), rg = lane % RG, q = lane / RG
// (RG = 32 / TPR rows per warp iteration) loads the V entries of row r0 + rg in columns
// k = q + TPR c (c < CPL): each column load of a warp is RG consecutive rows (RG x 16 B
// contiguous).  The entries stay in registers for both uses:
//   MODE 1: p' = s_j (p - sum_k V_k e1'_k)   (row sum over the q lanes: log2 TPR xor-shuffles)
//   dots:   acc_c += conj(V_k) p'            (per-lane, across all of the lane's rows)
// The lane sums are reduced over rg once per kernel (log2 RG xor-shuffles per column), then per
// block in fixed warp order and across blocks by the last block (integer ticket): deterministic
// for a given grid.  Per element: one 16-B load and 4 (+4 in MODE 1) FMAs; no shuffles per
// element for the dots (round 1's shuffle kernel reduced every row batch), no 255-register accumulator file
// (k_proj_tma: 8 warps per SM, latency-bound).
//   MODE 0 (sweep-1):  g1 = V^H p            MODE 1 (sweep-2):  p' -> W,  g2 = V^H p'
// --------------------------------------------------------------------------------------
template <int MODE, int TPR, int CPL, int U, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_proj_r(KDev d, int j) {
  constexpr int RG = 32 / TPR;
  __shared__ double2 coef[kMaxCols];
  __shared__ double2 red[kWarps][kMaxCols];
  __shared__ int go_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rg = lane % RG, q = lane / RG;
  const int ncols = j + 1;
  const double sj = MODE == 1 ? gate_value(d, j, d.flag[0], d.gsync[0].x) : (d.flag[0] == 0 ? 1.0 : 0.0);
  if (tid == 0) {
    if (MODE == 1 && blockIdx.x == 0) step_gate(d, j, true);
    go_s = sj != 0.0;
  }
  if (MODE == 1 && tid < ncols) {
    const double sk = tid == j ? sj : d.s[tid];
    const double2 g = d.g1[tid];
    coef[tid] = make_double2(sk * sk * g.x, sk * sk * g.y);  // e1'_k = s_k^2 g1_k
  }
  __syncthreads();
  if (!go_s) return;
  const int64_t n = d.n, ldv = d.ldv;
  double2 acc[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = make_double2(0.0, 0.0);
  // U row chunks per iteration (all loads issued before any use: U (CPL + 1) loads in flight)
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp, tw = (int64_t)gridDim.x * kWarps;
  for (int64_t c0 = gw; c0 * RG < n; c0 += U * tw) {
    double2 v[U][CPL], p[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = (c0 + u * tw) * RG + rg;
      const bool act = r < n;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int k = q + TPR * c;
        v[u][c] = (act && k < ncols) ? ld_stream(d.V + r + (int64_t)k * ldv) : make_double2(0.0, 0.0);
      }
      p[u] = act ? (MODE == 1 ? __ldcs(d.W + r) : __ldg(d.W + r)) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == 1) {
        const int64_t r = (c0 + u * tw) * RG + rg;
        const bool act = r < n;
        double2 a0 = make_double2(0.0, 0.0), a1 = a0;
#pragma unroll
        for (int c = 0; c < CPL; c += 2) {
          const int k = q + TPR * c;
          if (k < ncols) a0 = cfma(v[u][c], coef[k], a0);
          if (c + 1 < CPL && k + TPR < ncols) a1 = cfma(v[u][c + 1], coef[k + TPR], a1);
        }
        double2 a = cadd(a0, a1);
#pragma unroll
        for (int off = RG; off < 32; off <<= 1) {
          a.x += __shfl_xor_sync(0xffffffffu, a.x, off);
          a.y += __shfl_xor_sync(0xffffffffu, a.y, off);
        }
        p[u] = act ? make_double2(sj * (p[u].x - a.x), sj * (p[u].y - a.y)) : make_double2(0.0, 0.0);
        if (act && q == 0) d.W[r] = p[u];
      }
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc[c] = cfma_conj(v[u][c], p[u], acc[c]);
    }
  }
  // lane sums over rg (fixed butterfly), then lane rg == 0 of each q holds the warp's column sums
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
#pragma unroll
    for (int off = 1; off < RG; off <<= 1) {
      acc[c].x += __shfl_xor_sync(0xffffffffu, acc[c].x, off);
      acc[c].y += __shfl_xor_sync(0xffffffffu, acc[c].y, off);
    }
    const int k = q + TPR * c;
    if (rg == 0 && k < kMaxCols) red[warp][k] = acc[c];
  }
  __syncthreads();
  if (tid < ncols) {
    double2 t = red[0][tid];
    for (int w = 1; w < kWarps; ++w) t = cadd(t, red[w][tid]);
    d.part[(size_t)blockIdx.x * kMaxCols + tid] = t;
  }
  __threadfence();
  __syncthreads();
  __shared__ int last;
  const int ctr = MODE == 0 ? 0 : 1;
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
  double2* out = MODE == 0 ? d.g1 : d.g2;
  if (tid < ncols) out[tid] = cadd(cadd(cadd(seg[0][tid], seg[1][tid]), seg[2][tid]), seg[3][tid]);
  if (MODE == 0 && tid == 0) d.gsync[0] = make_double2(j > 0 ? d.nrm2[j - 1] : 0.0, 0.0);
  if (tid == 0) d.counter[ctr] = 0u;
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
    if (go_s && blockIdx.x == 0) {  // alpha_j = Re(c1_j + c2_j) (reading C2); g1 = raw dots of H V_j
      const double sj = d.s[j];
      d.alpha[j] = sj * (sj * d.g1[j].x + d.g2[j].x);
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
  __shared__ double cb_s;
  const int tid = threadIdx.x;
  if (tid == 0) {
    go_s = (d.flag[0] == 0);
    cb_s = j > 0 ? d.beta[j - 1] * d.s[j - 1] : 0.0;  // beta_{j-1} v_{j-1} = beta_{j-1} s_{j-1} V_{j-1}
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
// out may alias column 0 of V (in place): no __restrict__ on either pointer; each thread reads its
// row of every column before it writes that row
__global__ void __launch_bounds__(kThreads) k_combine(const double2* Vbase, int64_t n, int64_t ldv,
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
int kernel_attributes(int which, int* regs, int* max_threads, int* static_smem, int* max_dyn_smem) {
  const void* f = nullptr;
  switch (which) {
    case 0: f = spmv_attr_kernel(); break;
    case 1: f = (const void*)k_proj_tma<0>; break;
    case 2: f = (const void*)k_proj_tma<1>; break;
    case 3: f = (const void*)k_update_norm; break;
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

// dynamic shared memory limit of one kernel: the request capped at the opt-in maximum minus its
// static shared memory; the first failure is kept
void set_attr(const void* f, size_t want, void* ctx) {
  AttrState* s = static_cast<AttrState*>(ctx);
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, f);
  if (e == cudaSuccess) {
    const size_t lim = (size_t)s->optin - a.sharedSizeBytes;
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::min(want, lim));
  }
  if (e != cudaSuccess && s->err == cudaSuccess) s->err = e;
}

cudaError_t configure_kernels() {
  static cudaError_t status = cudaErrorNotReady;
  if (status != cudaErrorNotReady) return status;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  AttrState st{optin, cudaSuccess};
  auto set = [&](const void* f, size_t want) { set_attr(f, want, &st); };
  set((const void*)k_proj_tma<0>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<3>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<0, 8>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<3, 8>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<1, 8>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<0, 16>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<3, 16>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<1, 16>, kProjSmemBudget + 1024);
  configure_spmv_kernels(set_attr, &st);
  set((const void*)k_proj_tma<1>, kProjSmemBudget + 1024);
#define TE_SET_RT(NREG, RT)                                                    \
  set((const void*)k_proj_tma<0, NREG, 1, RT>, kProjSmemBudget + 1024);        \
  set((const void*)k_proj_tma<1, NREG, 1, RT>, kProjSmemBudget + 1024);        \
  set((const void*)k_proj_tma<3, NREG, 1, RT>, kProjSmemBudget + 1024);
  TE_SET_RT(16, 4) TE_SET_RT(16, 2) TE_SET_RT(32, 2) TE_SET_RT(32, 1)
#undef TE_SET_RT
  set((const void*)k_proj_tma<4, 8, 1, 0>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<4, 8, 1, 1>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<4, 8, 1, 2>, kProjSmemBudget + 1024);
  set((const void*)k_proj_tma<4, 8, 1, 4>, kProjSmemBudget + 1024);
  status = st.err;
  return status;
}

// measured on B200 (tools/micro/mb_proj.cu, n = 2^20 and 2^23): the register-accumulator kernel
// is faster than the TMA ring up to 8 columns (e.g. 4 columns, n = 2^20: dots 4.7 vs 2.9 TB/s),
// the TMA ring above (lane groups of 4+ rows per column load lose coalescing: 64-B chunks);
// the TMA ring keeps per-lane register column sums for the smallest of 8 / 16 / 32 columns that
// covers ncols (fewer live registers at small ncols: 8 columns, update 3.7 -> 4.7 TB/s)
constexpr int kRegMaxCols = 8;

// (NREG, R) pairs of the default tiling get compile-time R: 9-14 columns (16, 4), 15-16 (16, 2),
// 17-30 (32, 2), 31-64 (32, 1); anything else (forced TMA below 9 columns, other g_proj_min_tile)
// runs the runtime-R build
#define TE_PROJ_TMA_L(MODE, NREG, RT, ncols, ...) \
  k_proj_tma<MODE, NREG, 1, RT><<<L.num_sms, kProjThreads, proj_smem_bytes(ncols), L.stream>>>(__VA_ARGS__)
#define TE_PROJ_TMA(MODE, ncols, ...)                                                       \
  do {                                                                                      \
    const int rsub_ = L.proj_const_r ? proj_rsub(ncols) : 0;                                \
    if ((ncols) <= 8) TE_PROJ_TMA_L(MODE, 8, 0, ncols, __VA_ARGS__);                        \
    else if ((ncols) <= 16) {                                                               \
      if (rsub_ == 4) TE_PROJ_TMA_L(MODE, 16, 4, ncols, __VA_ARGS__);                       \
      else if (rsub_ == 2) TE_PROJ_TMA_L(MODE, 16, 2, ncols, __VA_ARGS__);                  \
      else TE_PROJ_TMA_L(MODE, 16, 0, ncols, __VA_ARGS__);                                  \
    } else {                                                                                \
      if (rsub_ == 2) TE_PROJ_TMA_L(MODE, 32, 2, ncols, __VA_ARGS__);                       \
      else if (rsub_ == 1) TE_PROJ_TMA_L(MODE, 32, 1, ncols, __VA_ARGS__);                  \
      else TE_PROJ_TMA_L(MODE, 32, 0, ncols, __VA_ARGS__);                                  \
    }                                                                                       \
  } while (0)

// register-accumulator kernel: CPL = 4 columns per lane, TPR = the smallest power of two with
// TPR * CPL >= ncols, U = 2 row chunks per iteration (10 loads in flight per lane), 2 CTAs per SM
constexpr int kProjRCpl = 4;
constexpr int kProjRU = 2;
constexpr int kProjRMinb = 2;
int proj_r_tpr(int ncols) {
  int t = 1;
  while (t * kProjRCpl < ncols) t <<= 1;
  return t;
}
static void launch_proj_r(const KDev& d, int j, int mode, const Launch& L) {
  const int grid = L.num_sms * kProjRMinb;
  switch (proj_r_tpr(j + 1)) {
#define TE_PROJ_R_CASE(T)                                                                                \
  case T:                                                                                                \
    if (mode == 0) k_proj_r<0, T, kProjRCpl, kProjRU, kProjRMinb><<<grid, kThreads, 0, L.stream>>>(d, j); \
    else k_proj_r<1, T, kProjRCpl, kProjRU, kProjRMinb><<<grid, kThreads, 0, L.stream>>>(d, j);           \
    break;
    TE_PROJ_R_CASE(1)
    TE_PROJ_R_CASE(2)
    TE_PROJ_R_CASE(4)
    TE_PROJ_R_CASE(8)
    default:
    TE_PROJ_R_CASE(16)
#undef TE_PROJ_R_CASE
  }
}

static bool use_reg(const Launch& L, int ncols) {
  return L.proj_tma == 3 || (L.proj_tma == 2 && ncols <= kRegMaxCols);
}

void launch_proj_dots(const KDev& d, int j, const Launch& L) {
  if (use_reg(L, j + 1)) {
    launch_proj_r(d, j, 0, L);
    return;
  }
  const int S = proj_slots(j + 1), R = proj_rsub(j + 1), C = proj_consumers(j + 1);
  TE_PROJ_TMA(0, j + 1, L.tmaps[j], d, j, S, R, C, 0);
}

void launch_gram_update(const KDev& d, int j, bool write, const Launch& L) {
  const int S = proj_slots(j + 1), R = proj_rsub(j + 1), C = proj_consumers(j + 1);
  TE_PROJ_TMA(3, j + 1, L.tmaps[j], d, j, S, R, C, write ? 1 : 0);
}

void launch_update_proj(const KDev& d, int j, const Launch& L) {
  if (use_reg(L, j + 1)) {
    launch_proj_r(d, j, 1, L);
    return;
  }
  const int S = proj_slots(j + 1), R = proj_rsub(j + 1), C = proj_consumers(j + 1);
  TE_PROJ_TMA(1, j + 1, L.tmaps[j], d, j, S, R, C, 0);
}

// K3: above 8 columns the update + norm pass runs on the TMA ring too (k_proj_tma<4>: the ring reads
// V at 7.1 TB/s where plain register streaming reaches 6.5; tools/micro/mb_proj.cu), else the
// register-streaming kernel
void launch_update_norm(const KDev& d, int j, bool write, const Launch& L) {
  const int ncols = j + 1;
  if (L.norm_tma && !use_reg(L, ncols)) {
    const int S = proj_slots(ncols), R = proj_rsub(ncols), C = proj_consumers(ncols);
    const int rt = L.proj_const_r ? R : 0;
#define TE_NORM_TMA(RT) \
  k_proj_tma<4, 8, 1, RT><<<L.num_sms, kProjThreads, proj_smem_bytes(ncols), L.stream>>>(L.tmaps[j], d, j, S, R, C, write ? 1 : 0)
    if (rt == 1) TE_NORM_TMA(1);
    else if (rt == 2) TE_NORM_TMA(2);
    else if (rt == 4) TE_NORM_TMA(4);
    else TE_NORM_TMA(0);
#undef TE_NORM_TMA
    return;
  }
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
