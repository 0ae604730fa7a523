// Device-side data of one Krylov engine and the launchers of the hot-path kernels.
// Layout:
//   V   : column-major n x m_cap complex128 (interleaved re/im), column stride ldv
//         (ldv = n rounded up to 32 elements -> every column 512-byte aligned).  Columns are
//         stored UNNORMALISED; s[k] = 1/||V[:,k]|| (s[0] = 1) is applied on the fly.
//   W   : n complex128 work vector (p -> p' in place).
//   H   : CSR, rowptr int64 [n+1], col int32 [nnz] (local column index; columns >= n_loc
//         refer to the halo buffer in distributed handles), val double or double2.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace te {

constexpr int kThreads = 256;        // block size of every hot-path kernel
constexpr int kWarps = kThreads / 32;
constexpr int kMaxCols = 64;         // TE_M_MAX
// warp-specialised ring SpMV tile capacities (entries) for its 4-stage and 3-stage layouts
constexpr int kRingNnz4 = 4096, kRingNnzC4 = 2048;
constexpr int kRingNnz3 = 5632, kRingNnzC3 = 2816;
constexpr int kSellSigma = 4096;       // SELL-32-sigma sorting window (rows)

struct KDev {
  int64_t n;            // local rows
  int64_t ldv;          // column stride of V (elements)
  double2* V;
  double2* W;
  const int64_t* rowptr;
  const int32_t* col;
  const void* val;
  const double2* const* peer_base;  // [nranks] V base of every rank in this address space (halo mode 1)
  const int64_t* peer_ldv;          // [nranks] their column strides
  const int32_t* halo_owner;        // [n_halo] owning rank of each halo entry
  const int32_t* halo_lidx;         // [n_halo] row index of the entry at its owner
  const int32_t* scol;       // SELL-32-sigma (variant 6): padded column-major slices
  const void* sval;
  const int64_t* sptr;       // [nslices+1] slice offsets (entries)
  const int32_t* slen;       // [nslices] slice widths
  const int32_t* sperm;      // [32*nslices] slice position -> row (-1: padding lane)
  int64_t nslices;
  const int64_t* tile_ring;  // [4*ntiles_ring] {first row, end row, first entry, end entry} (variant 7)
  int64_t ntiles_ring;
  // staged-x ring SpMV (variant 8): its own tiles, per-tile x ranges staged into shared memory by
  // bulk copies, and per-entry 16-bit shared-memory slots (0xFFFF: gathered from global memory)
  const int64_t* tile_xs;    // [4*ntiles_xs] {first row, end row, first entry, end entry}
  int64_t ntiles_xs;
  const int4* xs_meta;       // [ntiles_xs] {ranges, staged slots, global entries, 0}
  const int2* xs_rng;        // [ntiles_xs * xs_rmax] {first column, length}; slots follow in order
  const uint16_t* lcol;      // [nnz + 8] slot of each entry in its tile's staged x
  int xs_ecap, xs_xcap, xs_rmax;  // entries per tile, staged x slots per tile, ranges per tile
  int xs_xpol;               // L2 policy of the staged x copies: 0 normal, 1 evict_last
  // slot-window SELL-32 with a value dictionary (variant 9, spmv_sw.cu)
  const int64_t* sw_sptr;    // [nslice+1] first slot of each 32-row slice (multiples of kSwGroup)
  const int32_t* sw_base;    // [slots] first column of each slot's 32-column window
  const uint16_t* sw_ent;    // [slots*32] (code << 8 | offset), groups of kSwGroup slots per lane
  const void* sw_diag;       // [n] diagonal (VT)
  const void* sw_dict;       // [sw_ndict <= 255] off-diagonal values (VT)
  int64_t sw_nslice;
  int sw_ndict;
  int sw_bits;               // 16: code << 8 | offset, groups of 4 slots; 8: code << 5 | offset, groups of 8
  // panel sweep (two passes when x outgrows L2): pass 1 holds the windows inside the slice's aligned
  // panel of 2^sw_ka slices and runs in row order; pass 2 holds the far windows, adds into W and
  // visits the slices with the sw_ob slice bits from sw_lo upwards as the slowest index, so that
  // the columns of one sweep period again form an L2-sized panel
  int sw_pass;               // 0: single pass, 2: far-window pass (sw_sptr/base/ent are that pass's arrays)
  int sw_sb, sw_lo, sw_ob;   // slice index bits, first outer bit, number of outer bits (pass 2)
  int accw;             // SpMV writes W += s_j (H V_j) instead of W = (column-blocked passes > 0)
  const double2* halo;  // received halo entries (distributed, NCCL exchange); nullptr otherwise
  // distributed handles: the entries of local rows whose columns live on other ranks, kept apart
  // from the local CSR (rowptr/col/val above hold local columns only) and added by k_spmv_halo
  const int32_t* hrow;     // [nh] local rows with halo entries
  const int64_t* hrowptr;  // [nh + 1]
  const int32_t* hcol;     // halo index of each entry
  const void* hval;
  int64_t nh;
  double* s;            // [m_cap+1] column scales
  double* alpha;        // [m_cap]
  double* beta;         // [m_cap]
  double2* g1;          // [m_cap] raw sweep-1 sums of step j  (sum_i conj(V_ik) p_i)
  double2* g2;          // [m_cap] raw sweep-2 sums
  double* nrm2;         // [m_cap] ||p''||^2 of step j
  double2* part;        // per-CTA partials [grid x kMaxCols]
  double* partn;        // per-CTA norm partials [grid]
  unsigned* counter;    // [4] last-block-done counters (self-resetting)
  int* flag;            // [0]: 0 running / 1 breakdown / 2 non-finite ; [1]: m_eff
  double tol_rate;
  int m;                // Krylov dimension of the current restart
  int ortho;            // 0 CGS2, 1 Lanczos (f1), 2 CGS2 with Gram-matrix second sweep (f2)
  double2* G;           // [kMaxCols x kMaxCols] Gram matrix <v_k, v_l> of the normalised basis (f2)
  int defer;            // 1 (CGS2, f2): the SpMV writes H V_j unscaled and the step-j gate (s_j, breakdown)
                        // runs in the update kernel after the step's first reduction, which also
                        // carries ||p''_{j-1}||^2 (one allreduce fewer per step on several ranks);
                        // 0 (f1 Lanczos): the SpMV applies the gate itself
  double2* gsync;       // [1] .x = ||p''_{j-1}||^2 as reduced together with g1 (defer mode)
};

struct Launch {
  cudaStream_t stream;
  int num_sms;
  int grid_k3;               // streaming kernels (update_norm, combine, norm): up to 8 blocks per SM
  const CUtensorMap* tmaps;  // [kMaxCols] 2-D maps of V, box = 64R doubles x (k+1) columns
  int spmv_force_halo;  // test hook: run the multi-rank (halo-aware) SpMV instantiation on one rank
  int spmv_nf_wide;     // ring SpMV gathers in flight per lane: 0 -> 12 real / 8 complex, 1 -> 16 / 12
  int halo_peer;        // halo entries read from peer memory (no staged exchange)
  int grid_spmv;        // CTAs of the (persistent) SpMV: num_sms, or fewer so that the NCCL halo
                        // exchange running concurrently on the side stream finds free SMs
  int spmv_ring_tpr;    // lanes per row of the warp-specialised ring SpMV
  int ring_stages;      // its ring depth: 4 (short real rows) or 3 (larger tiles)
  int spmv_xs_tpr;      // lanes per row of the staged-x ring SpMV
  int xs_stages;        // its ring depth (2 or 3)
  int xs_nf;            // its entries in flight per lane (8 or 16)
  int proj_tma;         // 2: hybrid by column count (default), 1: TMA-tiled only, 3: register accumulators only
  int spmv_tiled;       // 10: column-blocked ring, 9: slot-window SELL-32, 8: staged-x ring, 7: ring, 6: SELL-32-sigma
  int prefetch;         // update_norm: L2 bulk-prefetch distance in block iterations (0: off)
  int norm_tma;         // K3 (update + norm) above 8 columns: 1 on the TMA ring (k_proj_tma<4>), 0 k_update_norm
  int proj_const_r;     // TMA projection kernels: 1 (default) the builds with a compile-time sub-tile count, 0 the runtime-R build
};

// hot path (one Krylov step j = 4 launches; see kernels.cu)
void launch_sell_build(bool cplx, int64_t npos, const int64_t* rowptr, const int32_t* col, const void* val,
                       const int32_t* perm, const int64_t* sptr, const int32_t* slen, int32_t* scol, void* sval,
                       cudaStream_t st);
// kernel attribute setup: configure_kernels() (kernels.cu) sets the dynamic shared memory limits
// of every kernel; the SpMV kernels' part lives in spmv.cu
struct AttrState {
  int optin;
  cudaError_t err;
};
void set_attr(const void* f, size_t want, void* ctx);
void configure_spmv_kernels(void (*set_attr)(const void*, size_t, void*), void* ctx);
const void* spmv_attr_kernel();  // the SpMV kernel reported by kernel_attributes(0)
void launch_spmv(const KDev& d, bool cplx, int j, const Launch& L);        // K1a: SpMV only
// column-blocked CSR (variant 10): entries of each B-column block stored as their own CSR (the
// entries of a row keep their order inside each block); count / fill passes on the device
void launch_colblk_count(int64_t n, const int64_t* rowptr, const int32_t* col, int64_t B, int nb, int32_t* cnt,
                         cudaStream_t st);
void launch_colblk_fill(int64_t n, const int64_t* rowptr, const int32_t* col, const void* val, bool cplx, int64_t B,
                        int b, const int64_t* rowptr_b, int32_t* col_b, void* val_b, cudaStream_t st);
void launch_spmv_halo(const KDev& d, bool cplx, int j, const Launch& L);   // K1a': + halo entries (distributed)
// staged-x ring SpMV (spmv_xs.cu): plan (create time) and launch
constexpr int kXsConsumers = 15;
constexpr int kXsRmax = 64;      // x ranges per tile
constexpr int kXsGap = 8;        // bridge gaps of < 8 unused x entries (128 B) inside a range
constexpr size_t kXsBudget = 220 * 1024;  // shared memory of the 2-3 stage ring
size_t spmv_xs_smem(bool cplx, int tpr, int ecap, int xcap, int stages);
int xs_xcap_for(bool cplx, int tpr, int ecap, size_t budget, int stages);
void launch_dict_insert(int64_t n, const int64_t* rowptr, const int32_t* col, const void* val, bool cplx, void* table,
                        int cap, unsigned* count, cudaStream_t st);
size_t dict_slot_bytes();
void launch_xs_plan(const int64_t* tiles, int64_t ntiles, const int32_t* col, int64_t ncol_stage, int xcap, int rmax,
                    int gap, int4* meta, int2* rng, uint16_t* lcol, cudaStream_t st);
void configure_xs_kernels(void (*set_attr)(const void*, size_t, void*), void* ctx, size_t budget);
void launch_spmv_xs(const KDev& d, bool cplx, int j, const Launch& L);
// slot-window SELL-32 SpMV (spmv_sw.cu): build (count / fill passes) and launch
constexpr int kSwGroup = 4;      // slots per 8-byte entry load of a lane
void launch_sw_build(bool fill, bool cplx, bool b8, int pass, int ka, int64_t n, const int64_t* rowptr, const int32_t* col, const void* val,
                     const double2* dict_keys, int nd, const int64_t* sptr, int32_t* nslot, int32_t* base,
                     uint16_t* ent, void* diag, int* err, cudaStream_t st);
void launch_spmv_sw(const KDev& d, bool cplx, int j, const Launch& L);
void launch_proj_dots(const KDev& d, int j, const Launch& L);              // K1b: g1 = V^H p (TMA)
void launch_update_proj(const KDev& d, int j, const Launch& L);            // K2
void launch_gram_update(const KDev& d, int j, bool write, const Launch& L); // f2: p'' = p - V(c1+c2) -> V_{j+1}, V^H p'', ||p''||^2
void launch_update_norm(const KDev& d, int j, bool write, const Launch& L);// K3
void launch_finalize(const KDev& d, int j, const Launch& L);
void launch_lanczos_dot(const KDev& d, int j, const Launch& L);                // f1: a = v_j^H (p - b v_{j-1})
void launch_lanczos_update(const KDev& d, int j, bool write, const Launch& L); // f1: p'' and ||p''||^2               // beta_{m-1}
void launch_combine(const KDev& d, const double2* coef, int m_eff, double2* out, const Launch& L); // K4
void launch_restart_init(const KDev& d, const Launch& L);                  // flag=0, s[0]=1
void launch_norm2(const KDev& d, const double2* x, double* out, const Launch& L);
void launch_copy_col(const double2* src, double2* dst, int64_t n, cudaStream_t st);

// setup
struct CsrCheck { int* err; unsigned long long* norm1_bits; };
void launch_csr_check(int64_t n, int64_t ncol_limit, const int64_t* rowptr, const int32_t* col, const void* val,
                      bool cplx, bool hermitian_check, CsrCheck c, cudaStream_t st);
// distributed halo pack: out[t] = V_j[idx[t]]
void launch_pack(const double2* x, const int32_t* idx, int64_t cnt, double2* out, cudaStream_t st);

int proj_slots(int ncols);
int proj_rsub(int ncols);
int proj_consumers(int ncols);
size_t proj_smem_bytes(int ncols);
cudaError_t configure_kernels();
int kernel_attributes(int which, int* regs, int* max_threads, int* static_smem, int* max_dyn_smem);  // opt-in shared memory sizes (once per process/device)

}  // namespace te
