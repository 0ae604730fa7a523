// SpMV variant 9: slot-window SELL-32 with a value dictionary.  p = s_j H V_j (Eq. 8, first line,
// P:153), the only operation on the large space.
//
// Why: the model Hamiltonians of the paper (spin chains, its §5 model) have few distinct
// off-diagonal values and strongly aligned column patterns.  In a spin chain, rows r of an aligned
// 32-row slice share their high spin bits, so a bond acting on high sites maps the whole slice to
// another aligned 32-column window (r XOR mask), for every lane at once.  The CSR SpMV streams
// 12 bytes per entry (8-byte value + int32 column) and gathers x entry by entry; here each entry
// is 2 bytes:
//   * slices of 32 rows (lane = row); a row's off-diagonal entries are grouped by the 32-column
//     window c >> 5 of their column; the windows of a slice are merged across its 32 rows in
//     ascending order and each window gets as many slots as its largest per-row count (a slot =
//     one entry per lane, padded with code 255 where a row has fewer);
//   * per slot: the window's first column (int32, one per slot, broadcast to the warp);
//   * per (slot, lane): 16 bits = 8-bit value code (index into the sorted dictionary of the
//     distinct off-diagonal values; 255 = padding) | 8-bit offset of the column in the window;
//   * the diagonal as a dense per-row array (added first).
// A slot's x loads are then 32 lanes reading one aligned 32-entry window (512 B, coalesced) for
// every bond that moves the slice as a block.  Applicable when the off-diagonal values take at
// most 255 distinct values and the padding stays small (te_api.cu decides at create); the
// product order per row is: diagonal, then the slots in window order (fixed, deterministic).
#include "device_common.cuh"

#include <algorithm>

namespace te {

namespace {

template <bool CPLX>
__device__ __forceinline__ int dict_code(const double2* __restrict__ dk, int nd, double re, double im) {
  const unsigned long long kr = (unsigned long long)__double_as_longlong(re);
  const unsigned long long ki = (unsigned long long)__double_as_longlong(im);
  int lo = 0, hi = nd - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const unsigned long long mr = (unsigned long long)__double_as_longlong(dk[mid].x);
    const unsigned long long mi = (unsigned long long)__double_as_longlong(dk[mid].y);
    if (mr < kr || (mr == kr && mi < ki)) lo = mid + 1;
    else hi = mid;
  }
  const bool hit = (unsigned long long)__double_as_longlong(dk[lo].x) == kr &&
                   (unsigned long long)__double_as_longlong(dk[lo].y) == ki;
  return hit ? lo : -1;
}
}  // namespace

// ------------------------------------------------------------------------------------------
// value dictionary (create time): the distinct off-diagonal values of H, bit for bit (exact), into
// an open-addressing hash table; at most 255 of them (the couplings of a model Hamiltonian: XXZ
// 2-3, Bose-Hubbard <= 156) become the 8-bit codes of the slot-window format.
// ------------------------------------------------------------------------------------------
struct DictSlot {
  unsigned state;  // 0 empty, 1 being written, 2 ready
  unsigned pad;
  double re, im;
};

__global__ void k_dict_insert(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                              const void* __restrict__ val, bool cplx, DictSlot* table, int cap, unsigned* count) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    if (*(volatile unsigned*)count > 255u) return;
    for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
      if (col[k] == (int32_t)r) continue;
      double re, im = 0.0;
      if (cplx) {
        const double2 v = static_cast<const double2*>(val)[k];
        re = v.x;
        im = v.y;
      } else {
        re = static_cast<const double*>(val)[k];
      }
      const unsigned long long kr = (unsigned long long)__double_as_longlong(re);
      const unsigned long long ki = (unsigned long long)__double_as_longlong(im);
      unsigned long long hsh = kr * 0x9E3779B97F4A7C15ull ^ (ki + 0x632BE59BD9B4E019ull) * 0xBF58476D1CE4E5B9ull;
      hsh ^= hsh >> 29;
      for (int probe = 0; probe < cap; ++probe) {
        DictSlot* sl = table + ((hsh + probe) & (unsigned long long)(cap - 1));
        unsigned st = *(volatile unsigned*)&sl->state;
        if (st == 0u) {
          if (atomicCAS(&sl->state, 0u, 1u) == 0u) {
            sl->re = re;
            sl->im = im;
            __threadfence();
            atomicExch(&sl->state, 2u);
            atomicAdd(count, 1u);
            break;
          }
          st = 1u;
        }
        while (st == 1u) st = *(volatile unsigned*)&sl->state;
        if ((unsigned long long)__double_as_longlong(*(volatile double*)&sl->re) == kr &&
            (unsigned long long)__double_as_longlong(*(volatile double*)&sl->im) == ki)
          break;
      }
    }
  }
}

void launch_dict_insert(int64_t n, const int64_t* rowptr, const int32_t* col, const void* val, bool cplx, void* table,
                        int cap, unsigned* count, cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (n + 255) / 256));
  k_dict_insert<<<grid, 256, 0, st>>>(n, rowptr, col, val, cplx, static_cast<DictSlot*>(table), cap, count);
}
size_t dict_slot_bytes() { return sizeof(DictSlot); }

// Build, one warp per slice.  FILL = false: slot count of each slice (rounded up to kSwGroup);
// FILL = true: window bases, 16-bit entries and the diagonal.  dk: the nd dictionary values sorted
// by (re bits, im bits).  err bit 1: an off-diagonal value missing from the dictionary.
// B8: 8-bit entries (3-bit code | 5-bit offset; dictionaries of <= 7 values, code 7 = padding) in
// groups of 8 slots per lane; else 16-bit entries (8-bit code | 8-bit offset) in groups of 4.
template <bool CPLX, bool FILL, bool B8>
__global__ void __launch_bounds__(256) k_sw_build(int64_t n, const int64_t* __restrict__ rowptr,
                                                  const int32_t* __restrict__ col, const void* __restrict__ val,
                                                  const double2* __restrict__ dk, int nd, const int64_t* __restrict__ sptr,
                                                  int32_t* nslot, int32_t* base, uint16_t* ent, void* diag, int* err,
                                                  int pass, int ka) {
  constexpr int GRP = B8 ? 8 : kSwGroup;
  uint8_t* ent8 = reinterpret_cast<uint8_t*>(ent);
  auto put = [&](int64_t K, int lane_, unsigned code, unsigned off) {
    if (B8) ent8[((K >> 3) * 32 + lane_) * 8 + (K & 7)] = (uint8_t)(code << 5 | off);
    else ent[((K >> 2) * 32 + lane_) * 4 + (K & 3)] = (uint16_t)(code << 8 | off);
  };
  const unsigned pad_code = B8 ? 7u : 255u;
  using VT = typename ValT<CPLX>::T;
  const VT* v = static_cast<const VT*>(val);
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (n + 31) / 32;
  for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nsl;
       s += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t r = s * 32 + lane;
    int64_t p = r < n ? rowptr[r] : 0, e = r < n ? rowptr[r + 1] : 0;
    int64_t slot = FILL ? sptr[s] : 0;
    const int64_t slot_end = FILL ? sptr[s + 1] : 0;
    double2 dsum = make_double2(0.0, 0.0);
    for (;;) {
      unsigned key = 0xFFFFFFFFu;
      while (p < e && (int64_t)col[p] == r) {  // the diagonal: dense array
        if constexpr (CPLX) dsum = cadd(dsum, v[p]);
        else dsum.x += v[p];
        ++p;
      }
      if (p < e) key = (unsigned)col[p] >> 5;
      const unsigned kmin = __reduce_min_sync(0xFFFFFFFFu, key);
      if (kmin == 0xFFFFFFFFu) break;
      int cnt = 0;
      int64_t q = p;
      while (q < e && ((unsigned)col[q] >> 5) == kmin) {
        if ((int64_t)col[q] != r) ++cnt;
        ++q;
      }
      // panel sweep: pass 1 keeps the windows inside the slice's aligned panel of 2^ka slices,
      // pass 2 the others (s and kmin are warp-uniform; the diagonal's window is always near)
      const bool farw = (((unsigned)s ^ kmin) >> ka) != 0u;
      if ((pass == 1 && farw) || (pass == 2 && !farw)) {
        p = q;
        continue;
      }
      const int w = (int)__reduce_max_sync(0xFFFFFFFFu, (unsigned)cnt);
      if (FILL) {
        int k = 0;
        for (; p < q; ++p) {
          const int32_t c = col[p];
          if ((int64_t)c == r) {
            if constexpr (CPLX) dsum = cadd(dsum, v[p]);
            else dsum.x += v[p];
            continue;
          }
          double re, im = 0.0;
          if constexpr (CPLX) { re = v[p].x; im = v[p].y; } else { re = v[p]; }
          const int code = dict_code<CPLX>(dk, nd, re, im);
          if (code < 0 || code >= (int)pad_code) atomicOr(err, 1);
          put(slot + k, lane, (unsigned)code & (B8 ? 7u : 255u), (unsigned)(c & 31));
          ++k;
        }
        for (; k < w; ++k) put(slot + k, lane, pad_code, 0u);
        if (lane == 0)
          for (int i = 0; i < w; ++i) base[slot + i] = (int32_t)(kmin << 5);
      }
      p = q;
      slot += w;
    }
    if (FILL) {
      for (int64_t K = slot; K < slot_end; ++K) {  // round-up padding of the last group
        put(K, lane, pad_code, 0u);
        if (lane == 0) base[K] = (int32_t)(s * 32);
      }
      if (r < n && diag != nullptr) {
        if constexpr (CPLX) static_cast<double2*>(diag)[r] = dsum;
        else static_cast<double*>(diag)[r] = dsum.x;
      }
    } else if (lane == 0) {
      nslot[s] = (int32_t)((slot + GRP - 1) / GRP * GRP);
    }
  }
}

void launch_sw_build(bool fill, bool cplx, bool b8, int pass, int ka, int64_t n, const int64_t* rowptr, const int32_t* col, const void* val,
                     const double2* dk, int nd, const int64_t* sptr, int32_t* nslot, int32_t* base, uint16_t* ent,
                     void* diag, int* err, cudaStream_t st) {
  const int64_t nsl = (n + 31) / 32;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, (nsl + 7) / 8));
#define TE_SWB(C, F, B) k_sw_build<C, F, B><<<grid, 256, 0, st>>>(n, rowptr, col, val, dk, nd, sptr, nslot, base, ent, diag, err, pass, ka)
  if (b8) {
    if (cplx) { if (fill) TE_SWB(true, true, true); else TE_SWB(true, false, true); }
    else { if (fill) TE_SWB(false, true, true); else TE_SWB(false, false, true); }
  } else {
    if (cplx) { if (fill) TE_SWB(true, true, false); else TE_SWB(true, false, false); }
    else { if (fill) TE_SWB(false, true, false); else TE_SWB(false, false, false); }
  }
#undef TE_SWB
}

// ------------------------------------------------------------------------------------------
// the SpMV: one warp per slice (lane = row), persistent grid-stride over slices; U groups of
// kSwGroup slots per iteration (4U entry codes and x loads in flight per lane)
// ------------------------------------------------------------------------------------------
template <bool CPLX>
__device__ __forceinline__ typename ValT<CPLX>::T ld_dict(uint32_t addr) {
  if constexpr (CPLX) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
  } else {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
  }
}

// Pass 2 of the panel sweep: slice visited at position i of the sweep (the outer bits slowest)
__device__ __forceinline__ int64_t sw_perm(const KDev& d, int64_t i) {
  const int lo = d.sw_lo, ob = d.sw_ob, ib = d.sw_sb - ob;  // ib inner bits: lo low ones, ib - lo high ones
  const int64_t low = i & ((int64_t(1) << lo) - 1);
  const int64_t mid = (i >> lo) & ((int64_t(1) << (ib - lo)) - 1);
  const int64_t out = i >> ib;
  return low | (out << lo) | (mid << (lo + ob));
}

template <bool CPLX, int U, int XM = 0, int MINB = 1, bool PB = false>
__global__ void __launch_bounds__(kThreads, MINB) k_spmv_sw(KDev d, int j) {
  using VT = typename ValT<CPLX>::T;
  __shared__ __align__(16) VT dict_s[256];
  __shared__ double sj_s;
  const int tid = threadIdx.x, lane = tid & 31;
  // codes >= ndict (255: padding) read 0: padding entries are multiplied out instead of branched
  // around (their x index is a valid column of the slot's window)
  for (int i = tid; i < 256; i += blockDim.x) {
    VT z;
    if constexpr (CPLX) z = make_double2(0.0, 0.0); else z = 0.0;
    dict_s[i] = i < d.sw_ndict ? static_cast<const VT*>(d.sw_dict)[i] : z;
  }
  if (tid == 0) sj_s = spmv_gate(d, j, !PB && blockIdx.x == 0);
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;
  const double2* __restrict__ x = d.V + (int64_t)j * d.ldv;
  asm volatile("" : "+l"(x));  // column base pinned in a register (not recomputed per load)
  uint32_t dict_base = smem_u32(dict_s);
  asm volatile("" : "+r"(dict_base));
  constexpr uint32_t kVB = (uint32_t)sizeof(VT);
  const VT* __restrict__ diag = static_cast<const VT*>(d.sw_diag);
  const uint2* __restrict__ ent = reinterpret_cast<const uint2*>(d.sw_ent);
  const int4* __restrict__ base = reinterpret_cast<const int4*>(d.sw_base);
  const int64_t n = d.n, nsl = d.sw_nslice;
  const int64_t tw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t iend = PB ? (int64_t(1) << d.sw_sb) : nsl;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + tid) >> 5; i < iend; i += tw) {
    const int64_t s = PB ? sw_perm(d, i) : i;
    if (PB && s >= nsl) continue;
    const int64_t r = s * 32 + lane;
    const bool act = r < n;
    const int64_t g0 = __ldg(d.sw_sptr + s) / kSwGroup, g1 = __ldg(d.sw_sptr + s + 1) / kSwGroup;
    if (PB && g0 == g1) continue;
    double2 acc = make_double2(0.0, 0.0), w0 = make_double2(0.0, 0.0);
    if (PB) { if (act) w0 = __ldcs(d.W + r); }
    else if (act) acc = ValT<CPLX>::mul(ValT<CPLX>::ldcs(diag + r), __ldg(x + r));
    // software pipeline: the entry codes and window bases of batch g + U are loaded while the x
    // loads of batch g are in flight
    uint2 e[U];
    int4 b[U];
    auto load_batch = [&](int64_t g, uint2 (&eo)[U], int4 (&bo)[U]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool live = g + u < g1;
        eo[u] = live ? __ldcs(ent + (g + u) * 32 + lane) : make_uint2(0xFF00FF00u, 0xFF00FF00u);
        bo[u] = live ? __ldg(base + g + u) : make_int4(0, 0, 0, 0);
      }
    };
    load_batch(g0, e, b);
    for (int64_t g = g0; g < g1; g += U) {
      double2 xv[4 * U];
      uint32_t cd[4 * U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t w = k < 2 ? e[u].x : e[u].y;
          const uint32_t h = (k & 1) ? (w >> 16) : (w & 0xFFFFu);
          const uint32_t bb = (uint32_t)(k == 0 ? b[u].x : (k == 1 ? b[u].y : (k == 2 ? b[u].z : b[u].w)));
          cd[4 * u + k] = h >> 8;
          xv[4 * u + k] = XM ? ld_stream(x + (bb + (h & 0xFFu))) : __ldg(x + (bb + (h & 0xFFu)));
        }
      }
      if (g + U < g1) load_batch(g + U, e, b);
#pragma unroll
      for (int q = 0; q < 4 * U; ++q) acc = cadd(acc, ValT<CPLX>::mul(ld_dict<CPLX>(dict_base + cd[q] * kVB), xv[q]));
    }
    if (act) __stcs(d.W + r, make_double2(w0.x + acc.x * sj, w0.y + acc.y * sj));
  }
}

// 8-bit entries: one 8-byte load per lane covers a group of 8 slots; two 16-byte base loads per
// warp; 8 x-window loads per iteration.  Same product order as the 16-bit kernel.
// The kernel is latency-bound (ncu: long-scoreboard stalls ~11 per issue, 24 warps per SM): a
// slice costs one dependent memory round trip per group of 8 slots plus two for its prologue
// (slice pointers -> first entry codes).  The prologue is therefore pipelined across slices: the
// slice pointers of the warp's next slice are loaded when the current slice starts, and its first
// group of codes and window bases while the current slice's last group of x loads is in flight.
// 3 CTAs per SM (79 registers); a 64-register build at 4 CTAs per SM spills and measured 3.6 ms.
template <bool CPLX, bool PB = false>
__global__ void __launch_bounds__(kThreads, 3) k_spmv_sw8(KDev d, int j) {
  using VT = typename ValT<CPLX>::T;
  __shared__ __align__(16) VT dict_s[8];
  __shared__ double sj_s;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < 8) {
    VT z;
    if constexpr (CPLX) z = make_double2(0.0, 0.0); else z = 0.0;
    dict_s[tid] = tid < d.sw_ndict ? static_cast<const VT*>(d.sw_dict)[tid] : z;  // code 7 (padding): 0
  }
  if (tid == 0) sj_s = spmv_gate(d, j, !PB && blockIdx.x == 0);
  __syncthreads();
  const double sj = sj_s;
  if (sj == 0.0) return;
  const double2* __restrict__ x = d.V + (int64_t)j * d.ldv;
  asm volatile("" : "+l"(x));
  uint32_t dict_base = smem_u32(dict_s);
  asm volatile("" : "+r"(dict_base));
  constexpr uint32_t kVB = (uint32_t)sizeof(VT);
  const VT* __restrict__ diag = static_cast<const VT*>(d.sw_diag);
  const uint2* __restrict__ ent = reinterpret_cast<const uint2*>(d.sw_ent);
  const int4* __restrict__ base = reinterpret_cast<const int4*>(d.sw_base);
  const int64_t n = d.n, nsl = d.sw_nslice;
  const int64_t tw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t iend = PB ? (int64_t(1) << d.sw_sb) : nsl;
  // the warp's slices: sweep positions i, i + tw, ... (pass 2: permuted, positions past nsl skipped)
  auto next_slice = [&](int64_t& i, int64_t& s) -> bool {
    for (; i < iend; i += tw) {
      s = PB ? sw_perm(d, i) : i;
      if (!PB || s < nsl) return true;
    }
    return false;
  };
  int64_t i = ((int64_t)blockIdx.x * blockDim.x + tid) >> 5, s = 0;
  bool have = next_slice(i, s);
  int64_t g0 = 0, g1 = 0;
  uint2 e = make_uint2(0u, 0u);
  int4 b0 = make_int4(0, 0, 0, 0), b1 = b0;
  if (have) {
    g0 = __ldg(d.sw_sptr + s) >> 3;
    g1 = __ldg(d.sw_sptr + s + 1) >> 3;
    if (g0 < g1) {
      e = __ldcs(ent + g0 * 32 + lane);
      b0 = __ldg(base + 2 * g0);
      b1 = __ldg(base + 2 * g0 + 1);
    }
  }
  while (have) {
    int64_t i2 = i + tw, s2 = 0;
    const bool have2 = next_slice(i2, s2);
    int64_t ng0 = 0, ng1 = 0;
    if (have2) {  // consumed one slice later
      ng0 = __ldg(d.sw_sptr + s2) >> 3;
      ng1 = __ldg(d.sw_sptr + s2 + 1) >> 3;
    }
    const int64_t r = s * 32 + lane;
    const bool act = r < n;
    double2 acc = make_double2(0.0, 0.0), w0 = make_double2(0.0, 0.0);
    if (PB) { if (act && g0 < g1) w0 = __ldcs(d.W + r); }
    else if (act) acc = ValT<CPLX>::mul(ValT<CPLX>::ldcs(diag + r), __ldg(x + r));
    auto load_next_first = [&]() {  // first group of the warp's next slice, into the freed registers
      if (have2 && ng0 < ng1) {
        e = __ldcs(ent + ng0 * 32 + lane);
        b0 = __ldg(base + 2 * ng0);
        b1 = __ldg(base + 2 * ng0 + 1);
      }
    };
    if (g0 == g1) load_next_first();
    for (int64_t g = g0; g < g1; ++g) {
      double2 xv[8];
      uint32_t cd[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t h = ((k < 4 ? e.x : e.y) >> (8 * (k & 3))) & 0xFFu;
        const int4& bq = k < 4 ? b0 : b1;
        const uint32_t bb = (uint32_t)((k & 3) == 0 ? bq.x : ((k & 3) == 1 ? bq.y : ((k & 3) == 2 ? bq.z : bq.w)));
        cd[k] = h >> 5;
        xv[k] = __ldg(x + (bb + (h & 31u)));
      }
      if (g + 1 < g1) {
        e = __ldcs(ent + (g + 1) * 32 + lane);
        b0 = __ldg(base + 2 * (g + 1));
        b1 = __ldg(base + 2 * (g + 1) + 1);
      } else {
        load_next_first();
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc = cadd(acc, ValT<CPLX>::mul(ld_dict<CPLX>(dict_base + cd[k] * kVB), xv[k]));
    }
    if (act && (!PB || g0 < g1)) __stcs(d.W + r, make_double2(w0.x + acc.x * sj, w0.y + acc.y * sj));
    have = have2;
    i = i2;
    s = s2;
    g0 = ng0;
    g1 = ng1;
  }
}

template <bool CPLX, bool PB = false>
static int sw8_grid(const Launch& L, int64_t nsl) {
  static int per_sm = 0;
  if (per_sm == 0) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_spmv_sw8<CPLX, PB>, kThreads, 0) != cudaSuccess || b < 1) b = 1;
    per_sm = b;
  }
  return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)L.grid_spmv * per_sm, (nsl + kWarps - 1) / kWarps));
}

// persistent grid: exactly the co-resident blocks (a grid-stride loop with more blocks than fit
// runs the surplus blocks' whole share after the first wave: a long tail)
template <bool CPLX, int U, int XM = 0, int MINB = 1, bool PB = false>
static int sw_grid(const Launch& L, int64_t nsl) {
  static int per_sm = 0;
  if (per_sm == 0) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_spmv_sw<CPLX, U, XM, MINB, PB>, kThreads, 0) != cudaSuccess || b < 1) b = 1;
    per_sm = b;
  }
  // (grid_spmv < num_sms leaves SMs free for a concurrent NCCL halo exchange)
  return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)L.grid_spmv * per_sm, (nsl + kWarps - 1) / kWarps));
}

// 16-bit entries: 2 groups of 4 slots per iteration, at most 85 registers (3 CTAs per SM).  Measured
// on config 5 in its DRAM-bound state (16-bit entries, one pass, 3.86 ms per SpMV): 1 or 4 groups,
// 40-register builds at 6 CTAs per SM, x loads without L1 allocation, two-deep x pipelining and L2
// prefetch of the next slice's codes all within +-0.3 %.
void launch_spmv_sw(const KDev& d, bool cplx, int j, const Launch& L) {
#define TE_SW8(C, P) k_spmv_sw8<C, P><<<sw8_grid<C, P>(L, d.sw_nslice), kThreads, 0, L.stream>>>(d, j)
  if (d.sw_pass == 2) {  // far-window pass of the panel sweep: W += ..., permuted slice order
    if (d.sw_bits == 8) {
      if (cplx) TE_SW8(true, true);
      else TE_SW8(false, true);
    } else {
      if (cplx) k_spmv_sw<true, 2, 0, 3, true><<<sw_grid<true, 2, 0, 3, true>(L, d.sw_nslice), kThreads, 0, L.stream>>>(d, j);
      else k_spmv_sw<false, 2, 0, 3, true><<<sw_grid<false, 2, 0, 3, true>(L, d.sw_nslice), kThreads, 0, L.stream>>>(d, j);
    }
    return;
  }
  if (d.sw_bits == 8) {
    if (cplx) TE_SW8(true, false);
    else TE_SW8(false, false);
    return;
  }
#undef TE_SW8
  if (cplx) k_spmv_sw<true, 2, 0, 3><<<sw_grid<true, 2, 0, 3>(L, d.sw_nslice), kThreads, 0, L.stream>>>(d, j);
  else k_spmv_sw<false, 2, 0, 3><<<sw_grid<false, 2, 0, 3>(L, d.sw_nslice), kThreads, 0, L.stream>>>(d, j);
}

}  // namespace te
