// Staged-x ring SpMV (TE_OPT_SPMV = 8): p = s_j H V_j (Eq. 8, first line), the product the
// paper names as the only operation on the large space.
//
// The ring SpMV (spmv.cu) streams H through a bulk-copy ring but gathers x entry by entry with
// LDG: every gather is a dependent L1/L2/DRAM round trip held in registers, so the kernel is bound
// by gather latency (ncu: 70 % long-scoreboard stalls, 16 warps per SM) rather than by HBM.  For
// the structured Hamiltonians of the paper (spin chains, bosons, its §5 model) the columns a tile
// of rows touches form a few dozen contiguous x windows (XXZ: r XOR bond mask).  This variant
// moves those windows with the TMA engine as well:
//   * create time (k_xs_plan, one CTA per tile): sort the tile's columns, merge them into ranges
//     (gaps of < kXsGap unused entries are bridged), stage every range with >= 2 distinct columns
//     and >= 1/4 density while the tile's slot budget lasts; every entry gets a 16-bit slot in the
//     tile's staged x (0xFFFF: not staged, gathered from global memory like the ring SpMV does);
//   * run time (k_spmv_xs): one producer warp bulk-copies rowptr, values, the 16-bit slots and
//     the tile's x ranges (32 lanes issue the range copies) into a 2-3 stage shared-memory ring
//     (descriptors loaded one tile ahead);
//     15 consumer warps read x from shared memory, so the gathers no longer wait on L2/DRAM.
// Arithmetic per row: TPR lanes, lane q sums entries q, q+TPR, ... in order, then a fixed xor
// reduction (deterministic, parity-tested against the oracle like every variant).
#include "device_common.cuh"

#include <algorithm>

namespace te {

namespace {
constexpr int kPlanThreads = 512;
constexpr int kPlanMax = 8192;  // entries a tile may have to be planned (longer: all global)
constexpr int kXsThreads = (kXsConsumers + 1) * 32;

__host__ __device__ constexpr size_t rnd16(size_t b) { return (b + 15) & ~(size_t)15; }

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_nohint(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
}  // namespace

// ------------------------------------------------------------------------------------------
// plan: one CTA per tile.  keys = (column << 13 | position in tile), bitonic-sorted in shared
// memory; thread 0 walks the sorted columns twice (ranges + decisions, then slots); ranges are
// cut at ncol_stage (columns >= it belong to the halo of a distributed handle: never staged).
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kPlanThreads) k_xs_plan(const int64_t* __restrict__ tiles, const int32_t* __restrict__ col,
                                                          int64_t ncol_stage, int xcap, int rmax, int gap, int4* meta,
                                                          int2* rng, uint16_t* lcol) {
  extern __shared__ __align__(16) unsigned char psm[];
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(psm);          // kPlanMax
  int* base = reinterpret_cast<int*>(psm + 8 * kPlanMax);                          // per range: first slot or -1
  uint16_t* slot = reinterpret_cast<uint16_t*>(psm + 12 * kPlanMax);               // per position
  const int64_t t = blockIdx.x;
  const int64_t e0 = tiles[4 * t + 2], e1 = tiles[4 * t + 3];
  const int cnt = (int)(e1 - e0);
  const int tid = threadIdx.x;
  if (cnt > kPlanMax) {  // a single long row: the kernel's global-memory path
    for (int64_t e = e0 + tid; e < e1; e += kPlanThreads) lcol[e] = 0xFFFFu;
    if (tid == 0) meta[t] = make_int4(0, 0, cnt, 0);
    return;
  }
  int P = 1;
  while (P < cnt) P <<= 1;
  for (int i = tid; i < P; i += kPlanThreads)
    keys[i] = i < cnt ? (((unsigned long long)(uint32_t)col[e0 + i]) << 13) | (unsigned long long)i : ~0ull;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1)
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int i = tid; i < P; i += kPlanThreads) {
        const int ixj = i ^ jj;
        if (ixj > i) {
          const unsigned long long a = keys[i], b = keys[ixj];
          if ((a > b) == ((i & k) == 0)) {
            keys[i] = b;
            keys[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  if (tid == 0) {
    // pass A: ranges in column order; decide each when it closes
    int nr = 0, nrng = 0, nslot = 0;
    int64_t rs = 0, rl = 0, hits = 0, prev = -1;
    auto close = [&]() {
      const int64_t len = rl - rs + 1;
      const bool ok = rs < ncol_stage && hits >= 2 && 4 * hits >= len && nslot + len <= xcap && nrng < rmax;
      if (ok) {
        base[nr] = nslot;
        rng[t * rmax + nrng] = make_int2((int)rs, (int)len);
        nslot += (int)len;
        ++nrng;
      } else {
        base[nr] = -1;
      }
      ++nr;
    };
    for (int i = 0; i < cnt; ++i) {
      const int64_t c = (int64_t)(keys[i] >> 13);
      if (prev < 0) {
        rs = rl = c;
        hits = 1;
      } else if (c == prev) {
        // same column again (several rows of the tile): same slot
      } else if (c > prev + gap || (prev < ncol_stage && c >= ncol_stage)) {
        close();
        rs = rl = c;
        hits = 1;
      } else {
        rl = c;
        ++hits;
      }
      prev = c;
    }
    if (cnt > 0) close();
    // pass B: the same walk, slot of every entry
    int r = -1, ng = 0;
    prev = -1;
    int64_t cur_rs = 0;
    for (int i = 0; i < cnt; ++i) {
      const int64_t c = (int64_t)(keys[i] >> 13);
      const int pos = (int)(keys[i] & 8191ull);
      if (prev < 0 || (c != prev && (c > prev + gap || (prev < ncol_stage && c >= ncol_stage)))) {
        ++r;
        cur_rs = c;
      }
      prev = c;
      const int b = base[r];
      if (b >= 0) {
        slot[pos] = (uint16_t)(b + (int)(c - cur_rs));
      } else {
        slot[pos] = 0xFFFFu;
        ++ng;
      }
    }
    meta[t] = make_int4(nrng, nslot, ng, 0);
  }
  __syncthreads();
  for (int i = tid; i < cnt; i += kPlanThreads) lcol[e0 + i] = slot[i];
}

size_t xs_plan_smem() { return (size_t)kPlanMax * (8 + 4 + 2); }

void launch_xs_plan(const int64_t* tiles, int64_t ntiles, const int32_t* col, int64_t ncol_stage, int xcap, int rmax,
                    int gap, int4* meta, int2* rng, uint16_t* lcol, cudaStream_t st) {
  if (ntiles <= 0) return;
  k_xs_plan<<<(unsigned)ntiles, kPlanThreads, xs_plan_smem(), st>>>(tiles, col, ncol_stage, xcap, rmax, gap, meta, rng,
                                                                     lcol);
}

// ------------------------------------------------------------------------------------------
// the SpMV
// ------------------------------------------------------------------------------------------
// stage layout: [x slots | values | rowptr | 16-bit slots]
template <bool CPLX, int TPR>
struct XsLayout {
  using VT = typename ValT<CPLX>::T;
  static constexpr int kRcap = 32 * kXsConsumers / TPR;
  __host__ __device__ static size_t xb(int xcap) { return (size_t)xcap * 16; }
  __host__ __device__ static size_t vb(int ecap) { return rnd16((size_t)(ecap + 2) * sizeof(VT)); }
  __host__ __device__ static size_t rb() { return rnd16((size_t)(kRcap + 4) * 8); }
  __host__ __device__ static size_t lb(int ecap) { return rnd16((size_t)(ecap + 16) * 2); }
  __host__ __device__ static size_t stage(int ecap, int xcap) { return xb(xcap) + vb(ecap) + rb() + lb(ecap); }
};

template <bool CPLX, int TPR, int HM, int NF, int STG>
__global__ void __launch_bounds__(kXsThreads, 1) k_spmv_xs(KDev d, int j) {
  using VT = typename ValT<CPLX>::T;
  using LY = XsLayout<CPLX, TPR>;
  constexpr int C = kXsConsumers;
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[STG], empty[STG];
  __shared__ int64_t desc[STG][4];
  __shared__ int gcount[STG];
  __shared__ double sj_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ecap = d.xs_ecap, xcap = d.xs_xcap;
  const size_t oX = 0, oV = LY::xb(xcap), oR = oV + LY::vb(ecap), oL = oR + LY::rb();
  const size_t stage_bytes = LY::stage(ecap, xcap);
  if (tid == 0) {
    sj_s = spmv_gate(d, j, blockIdx.x == 0);
    for (int k = 0; k < STG; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], C);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;
  const int64_t G = gridDim.x;
  const double2* __restrict__ x = d.V + (int64_t)j * d.ldv;
  if (warp == C) {  // ------------------------------------------------------------ producer warp
    const uint64_t pol = policy_evict_first();  // H: streamed once
    const uint64_t polx = policy_evict_last();
    constexpr int64_t VA = 16 / (int64_t)sizeof(VT);
    const int2* rngs = reinterpret_cast<const int2*>(d.xs_rng);
    // descriptor, meta and x ranges of tile t: loaded one tile ahead (before the wait for a free
    // stage), so their latency is off the path from "stage free" to "copies issued"
    struct Desc {
      longlong2 a, b;
      int4 mt;
      int2 r0, r1;
    };
    auto load = [&](int64_t t) {
      Desc q{};
      if (t < d.ntiles_xs) {
        q.a = __ldg(reinterpret_cast<const longlong2*>(d.tile_xs + 4 * t));
        q.b = __ldg(reinterpret_cast<const longlong2*>(d.tile_xs + 4 * t) + 1);
        q.mt = __ldg(d.xs_meta + t);
        q.r0 = __ldg(rngs + t * d.xs_rmax + lane);  // unused slots hold {0, 0}
        q.r1 = __ldg(rngs + t * d.xs_rmax + 32 + lane);
      }
      return q;
    };
    Desc cur = load(blockIdx.x);
    for (int64_t it = 0;; ++it) {
      const int64_t t = blockIdx.x + it * G;
      const int st = (int)(it % STG);
      const Desc nxt = load(t + G);
      if (it >= STG) mbar_wait(&empty[st], (unsigned)(((it / STG) - 1) & 1));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (t >= d.ntiles_xs) {
        if (lane == 0) {
          desc[st][0] = -1;
          mbar_expect_tx(&full[st], 0);
        }
        break;
      }
      const longlong2 a = cur.a, b = cur.b;
      const int4 mt = cur.mt;
      const int64_t cnt = b.y - b.x;
      const bool staged = cnt <= ecap;
      unsigned char* base = sm + (size_t)st * stage_bytes;
      const int2 r0 = staged ? cur.r0 : make_int2(0, 0), r1 = staged ? cur.r1 : make_int2(0, 0);
      if (lane == 0) {
        desc[st][0] = a.x; desc[st][1] = a.y; desc[st][2] = b.x; desc[st][3] = b.y;
        gcount[st] = mt.z;
        unsigned br = 0, bv = 0, bl = 0;
        int64_t r0i = 0, v0 = 0, l0 = 0;
        if (staged) {
          r0i = a.x & ~1LL;
          br = (unsigned)((((a.y + 2) & ~1LL) - r0i) * 8);
          v0 = b.x & ~(VA - 1);
          bv = (unsigned)((((b.y + VA - 1) & ~(VA - 1)) - v0) * sizeof(VT));
          l0 = b.x & ~7LL;
          bl = (unsigned)((((b.y + 7) & ~7LL) - l0) * 2);
        }
        mbar_expect_tx(&full[st], br + bv + bl + (staged ? (unsigned)mt.y * 16u : 0u));
        if (br) bulk_g2s(base + oR, d.rowptr + r0i, br, &full[st], pol);
        if (bv) bulk_g2s(base + oV, static_cast<const VT*>(d.val) + v0, bv, &full[st], pol);
        if (bl) bulk_g2s(base + oL, d.lcol + l0, bl, &full[st], pol);
      }
      __syncwarp();
      if (staged) {
        // exclusive prefix of the range lengths (ranges lane, then lane + 32)
        int s0 = r0.y, s1 = r1.y;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int u0 = __shfl_up_sync(0xffffffffu, s0, off);
          const int u1 = __shfl_up_sync(0xffffffffu, s1, off);
          if (lane >= off) { s0 += u0; s1 += u1; }
        }
        const int tot0 = __shfl_sync(0xffffffffu, s0, 31);
        const int b0 = s0 - r0.y, b1 = tot0 + s1 - r1.y;
        if (d.xs_xpol) {  // x kept in L2 ahead of the streamed H (evict_first)
          if (r0.y > 0) bulk_g2s(base + oX + (size_t)b0 * 16, x + r0.x, (unsigned)r0.y * 16u, &full[st], polx);
          if (r1.y > 0) bulk_g2s(base + oX + (size_t)b1 * 16, x + r1.x, (unsigned)r1.y * 16u, &full[st], polx);
        } else {
          if (r0.y > 0) bulk_g2s_nohint(base + oX + (size_t)b0 * 16, x + r0.x, (unsigned)r0.y * 16u, &full[st]);
          if (r1.y > 0) bulk_g2s_nohint(base + oX + (size_t)b1 * 16, x + r1.x, (unsigned)r1.y * 16u, &full[st]);
        }
      }
      cur = nxt;
    }
    return;
  }
  // ------------------------------------------------------------------------------------ consumers
  const double2* __restrict__ halo = d.halo;
  const int n = (int)d.n;
  const int q = tid % TPR, grp = tid / TPR;
  auto gx = [&](int c) -> double2 {
    if (HM == 1) return ((uint32_t)c < (uint32_t)n) ? __ldg(x + c) : __ldg(halo + (c - n));
    if (HM == 2) return ((uint32_t)c < (uint32_t)n) ? __ldg(x + c) : peer_x(d, j, c - n);
    return __ldg(x + c);
  };
  for (int64_t it = 0;; ++it) {
    const int st = (int)(it % STG);
    mbar_wait(&full[st], (unsigned)((it / STG) & 1));
    const int64_t ra = desc[st][0];
    if (ra < 0) break;
    const int64_t rb = desc[st][1], b = desc[st][2], e = desc[st][3];
    const int64_t t = blockIdx.x + it * G;
    if (e - b <= ecap) {
      constexpr int64_t VA = 16 / (int64_t)sizeof(VT);
      const unsigned char* base = sm + (size_t)st * stage_bytes;
      const double2* xs = reinterpret_cast<const double2*>(base + oX);
      const VT* vv = reinterpret_cast<const VT*>(base + oV) + (b & (VA - 1));
      const int64_t* rp = reinterpret_cast<const int64_t*>(base + oR) + (ra & 1);
      const uint16_t* lc = reinterpret_cast<const uint16_t*>(base + oL) + (b & 7);
      const int rows = (int)(rb - ra);
      const int i = grp;
      const bool act = i < rows;
      const int lo = act ? (int)(rp[i] - b) : 0, hi = act ? (int)(rp[i + 1] - b) : 0;
      double2 acc = make_double2(0.0, 0.0);
      if (gcount[st] == 0) {  // every x of the tile is in shared memory
        for (int q0 = lo + q; q0 < hi; q0 += NF * TPR) {
          double2 xx[NF];
#pragma unroll
          for (int w = 0; w < NF; ++w) {
            const int ee = q0 + w * TPR;
            if (ee < hi) xx[w] = xs[lc[ee]];
          }
#pragma unroll
          for (int w = 0; w < NF; ++w)
            if (q0 + w * TPR < hi) acc = cadd(acc, ValT<CPLX>::mul(vv[q0 + w * TPR], xx[w]));
        }
      } else {
        for (int q0 = lo + q; q0 < hi; q0 += NF * TPR) {
          double2 xx[NF];
#pragma unroll
          for (int w = 0; w < NF; ++w) {
            const int ee = q0 + w * TPR;
            if (ee < hi) {
              const unsigned s = lc[ee];
              xx[w] = (s != 0xFFFFu) ? xs[s] : gx(__ldg(d.col + b + ee));
            }
          }
#pragma unroll
          for (int w = 0; w < NF; ++w)
            if (q0 + w * TPR < hi) acc = cadd(acc, ValT<CPLX>::mul(vv[q0 + w * TPR], xx[w]));
        }
      }
      if (TPR > 1) acc = group_sum<TPR>(acc);
      if (act && q == 0) __stcs(d.W + ra + i, make_double2(acc.x * sj, acc.y * sj));
    } else if (warp == (int)(t % C)) {  // one long row: one warp, from global memory (val kept)
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

size_t spmv_xs_smem(bool cplx, int tpr, int ecap, int xcap, int stages) {
  switch (tpr) {
#define TE_XS_SM(T) \
  case T:           \
    return stages * (cplx ? XsLayout<true, T>::stage(ecap, xcap) : XsLayout<false, T>::stage(ecap, xcap));
    TE_XS_SM(1) TE_XS_SM(2) TE_XS_SM(4)
    default: TE_XS_SM(8)
#undef TE_XS_SM
  }
}

void launch_spmv_xs(const KDev& d, bool cplx, int j, const Launch& L) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(L.grid_spmv, d.ntiles_xs));
  const size_t smem = spmv_xs_smem(cplx, L.spmv_xs_tpr, d.xs_ecap, d.xs_xcap, L.xs_stages);
#define TE_XS_NF(T, H, S, NF)                                                                  \
  if (cplx) k_spmv_xs<true, T, H, NF, S><<<grid, kXsThreads, smem, L.stream>>>(d, j);          \
  else k_spmv_xs<false, T, H, NF, S><<<grid, kXsThreads, smem, L.stream>>>(d, j);
#define TE_XS_S(T, H, S) \
  if (L.xs_nf == 16) { TE_XS_NF(T, H, S, 16) } else { TE_XS_NF(T, H, S, 8) }
#define TE_XS_H(T, H) \
  if (L.xs_stages == 3) { TE_XS_S(T, H, 3) } else { TE_XS_S(T, H, 2) }
#define TE_XS(T)                                                                                 \
  case T:                                                                                        \
    if (L.spmv_force_halo) { TE_XS_H(T, 1) }                                                    \
    else { TE_XS_H(T, 0) }                                                                       \
    break;
  switch (L.spmv_xs_tpr) {
    TE_XS(1) TE_XS(2) TE_XS(4)
    default: TE_XS(8)
  }
#undef TE_XS
#undef TE_XS_H
#undef TE_XS_S
#undef TE_XS_NF
}

void configure_xs_kernels(void (*set_attr)(const void*, size_t, void*), void* ctx, size_t budget) {
  auto set = [&](const void* f, size_t want) { set_attr(f, want, ctx); };
  set((const void*)k_xs_plan, xs_plan_smem());
#define TE_SETXS_NF(T, H, NF)                                       \
  set((const void*)k_spmv_xs<false, T, H, NF, 2>, budget);          \
  set((const void*)k_spmv_xs<true, T, H, NF, 2>, budget);           \
  set((const void*)k_spmv_xs<false, T, H, NF, 3>, budget);          \
  set((const void*)k_spmv_xs<true, T, H, NF, 3>, budget);
#define TE_SETXS(T, H) TE_SETXS_NF(T, H, 8) TE_SETXS_NF(T, H, 16)
  TE_SETXS(1, 0) TE_SETXS(2, 0) TE_SETXS(4, 0) TE_SETXS(8, 0)
  TE_SETXS(1, 1) TE_SETXS(2, 1) TE_SETXS(4, 1) TE_SETXS(8, 1)
#undef TE_SETXS
#undef TE_SETXS_NF
}

// x slots per tile that fit the shared-memory budget next to the tile's H part
int xs_xcap_for(bool cplx, int tpr, int ecap, size_t budget, int stages) {
  size_t h = 0;
#define TE_XS_H0(T) h = cplx ? XsLayout<true, T>::stage(ecap, 0) : XsLayout<false, T>::stage(ecap, 0);
  switch (tpr) {
    case 1: TE_XS_H0(1) break;
    case 2: TE_XS_H0(2) break;
    case 4: TE_XS_H0(4) break;
    default: TE_XS_H0(8) break;
  }
#undef TE_XS_H0
  const size_t per_stage = budget / stages;
  if (per_stage <= h + 16) return 0;
  return (int)std::min<size_t>((per_stage - h) / 16, 65535 - 1);
}

}  // namespace te
