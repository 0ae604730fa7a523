/*
 * te.h — C ABI of the B200-native restarted-Krylov engine for v(t) = exp(-iHt) v(0)
 * (after Michel & Zell, "TimeEvolver", arXiv:2205.15346).
 *
 * Citations: P:n = line n of the paper's LaTeX source.
 *   Problem statement            Eq. 1, Alg. 1 input/output
 *   Arnoldi/Lanczos basis        Eq. 8, Alg. 1 step 1
 *   Krylov approximation         Eq. 11
 *   Error bound                  Eq. 16, tanh-sinh quadrature
 *   Step size / error rate       Eqs. 18-19, Alg. 1 step 2
 *   Roundoff estimate            Eq. 17, warning
 * Readings of ambiguous passages: DESIGN.md "Readings".
 *
 * Conventions (all functions):
 *  - Everything is extern "C"; no C++ exception crosses the ABI.  Every entry
 *    point that can fail returns a status code (TE_OK = 0) or NULL, and sets a
 *    thread-local status/message readable with te_last_status()/te_last_error().
 *  - Complex numbers are te_c128 = {re, im} doubles (== numpy.complex128 ==
 *    C99 double _Complex layout).  Vectors are dense, contiguous, length n.
 *  - CSR: rowptr int64 [n+1] with rowptr[0] = 0 and non-decreasing; col int32
 *    [nnz] with 0 <= col < n and strictly increasing within a row (duplicates
 *    are rejected); val [nnz].  H must be Hermitian: structurally symmetric
 *    with |H_ij - conj(H_ji)| <= 8 eps max(|H_ij|,|H_ji|) and real diagonal.
 *  - Ownership: every input pointer is borrowed for the duration of the call
 *    and copied; the caller may free it afterwards.  Output arrays are
 *    caller-allocated.  A handle owns all device memory until te_destroy().
 *  - Device: a handle is bound to the CUDA device current at create time.
 *    A handle is not thread-safe; distinct handles may be used concurrently.
 *  - Determinism: identical inputs on the same device give bitwise-identical
 *    outputs (no floating-point atomics; fixed reduction order per grid size).
 */
#ifndef TE_H
#define TE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct te_handle te_handle;
typedef struct te_dist te_dist;
typedef struct { double re, im; } te_c128;

/* ---- status codes ---------------------------------------------------------------- */
enum {
  TE_OK = 0,
  TE_ERR_ARG = 1,             /* NULL pointer, n < 1, t < 0 or non-finite, tol <= 0, m_max < 1 or > TE_M_MAX */
  TE_ERR_CSR = 2,             /* rowptr/col invariants violated                                   */
  TE_ERR_NOT_HERMITIAN = 3,   /* H != H^dagger within tolerance                                    */
  TE_ERR_NOT_NORMALIZED = 4,  /* | ||v0||_2 - 1 | > 1e-8 (v(0) normalised)                  */
  TE_ERR_STEP_COLLAPSE = 5,   /* step size fell below 1e-13 t (m too small for the requested tol)   */
  TE_ERR_NUMERICAL = 6,       /* NaN/Inf in the Arnoldi recurrence                                  */
  TE_ERR_OOM = 7,             /* device allocation failed                                           */
  TE_ERR_CUDA = 8,            /* CUDA runtime error (incl. no device)                               */
  TE_ERR_NCCL = 9,            /* NCCL error (distributed handles)                                   */
  TE_ERR_UNSUPPORTED = 10     /* operation not available for this handle kind                     */
};

/* warning bits in te_stats.warnings — never errors (a warning does not abort) */
#define TE_WARN_ROUNDOFF   1u   /* roundoff estimate d ||H||_1 eps exceeded a step's error bound */
#define TE_WARN_QUADRATURE 2u   /* error integral not converged after 15 refinements             */

#define TE_M_MAX 64             /* largest supported Krylov dimension m_max                              */

typedef struct {
  double   err_bound;       /* sum over restarts of int_0^{tau_k} f (Eq. 16); <= tol by construction     */
  int64_t  n_restarts;      /* Krylov subspaces built = time steps                                        */
  int64_t  n_krylov_steps;  /* Arnoldi iterations (SpMVs)                                                 */
  int64_t  n_breakdowns;    /* lucky breakdowns (Alg. 1)                                            */
  double   roundoff_step;   /* Eq. 17 per restart: n ||H||_1 2^-52                                         */
  double   roundoff_total;  /* n_restarts * roundoff_step (reading C15)                                   */
  uint32_t warnings;        /* TE_WARN_* bits                                                             */
  uint32_t _pad;
  double   t_step_min, t_step_max;
  double   one_norm;        /* ||H||_1                                                                    */
} te_stats;

/* ---- core three (BASELINE.json north star) ------------------------------------- */

/* Copy a Hermitian CSR matrix with complex values to the device, validate it
 * (CSR invariants, Hermiticity, real diagonal) and compute ||H||_1 (Eq. 17).
 * Returns NULL on error (te_last_status(): TE_ERR_ARG/CSR/NOT_HERMITIAN/OOM/CUDA). */
te_handle* te_create_csr(int64_t n, const int64_t* rowptr, const int32_t* col, const te_c128* val);

/* v_out = Krylov approximation of exp(-iHt) v0 with ||exact - v_out||_2 <= stats.err_bound <= tol
 * (up to roundoff, Eq. 17) — Algorithm 1 with Krylov dimension m_max (fixed m,
 * capped at n; CGS2 orthogonalisation, reading C1).  v0 and v_out are HOST arrays of n
 * elements; v_out may alias v0.  t = 0 returns v0 with bound 0 and 0 restarts.  stats may
 * be NULL.  Returns TE_OK or an error (v_out unspecified on error; stats filled up to it). */
int te_evolve(te_handle* h, const te_c128* v0, double t, double tol, int m_max,
              te_c128* v_out, te_stats* stats);

/* Free all device memory owned by h (NULL is a no-op). */
void te_destroy(te_handle* h);

/* ---- extensions ------------------------------------------------------------------ */

/* As te_create_csr with real (float64) values (Hermitian == real symmetric). */
te_handle* te_create_csr_real(int64_t n, const int64_t* rowptr, const int32_t* col, const double* val);

/* As te_evolve with DEVICE pointers (n complex128 each, 16-byte aligned, may alias) on the
 * CUDA stream `stream` (cudaStream_t; NULL = the handle's own stream, a blocking stream, i.e.
 * ordered with work the caller issued on the legacy default stream).  The call returns after the
 * result is complete on that stream. */
int te_evolve_dev(te_handle* h, const void* d_v0, double t, double tol, int m_max,
                  void* d_vout, te_stats* stats, void* stream);

/* Forced step schedule (parity mode, reading C16): restart k uses step t_steps[k]
 * (clamped to the remaining time) instead of the step search; the error integral of each
 * step is still evaluated and summed into stats.err_bound.  Evolves to t = sum(t_steps).
 * Host arrays. */
int te_evolve_schedule(te_handle* h, const te_c128* v0, int64_t k, const double* t_steps,
                       double tol, int m_max, te_c128* v_out, te_stats* stats);

/* As te_evolve, also returning the states at the n_samples ascending times sample_times[] in
 * [0, t] ("sample its values at intermediate points of time" from the Krylov space of the
 * step that contains them).  samples_out: host, n_samples x n (sample-major); sample_bounds
 * (nullable): the error bound of each sample (bound accumulated before its step + the integral
 * of Eq. 16 up to the sample time). */
int te_evolve_sampled(te_handle* h, const te_c128* v0, double t, double tol, int m_max, int64_t n_samples,
                      const double* sample_times, te_c128* samples_out, double* sample_bounds,
                      te_c128* v_out, te_stats* stats);

/* Schedule of the most recent evolve call: up to cap entries of (tau_k, m_eff_k, e_k).
 * Any output pointer may be NULL.  Returns the number of restarts (may exceed cap). */
int64_t te_get_schedule(const te_handle* h, int64_t cap, double* t_steps, int32_t* m_eff,
                        double* err_steps);

/* One Arnoldi/CGS2 decomposition from the host vector v1 (Eq. 8): alpha[m], beta[m] (the
 * tridiagonal T and beta[m_eff-1] = h_{m+1,m}), *m_eff, *breakdown; V_out (nullable) receives
 * the normalised basis n x m_eff column-major.  Breakdown threshold tol_rate (Alg. 1). */
int te_krylov_basis(te_handle* h, const te_c128* v1, int m, double tol_rate, double* alpha,
                    double* beta, int* m_eff, int* breakdown, te_c128* V_out);

/* Options (value semantics per option): */
enum {
  TE_OPT_PROFILE = 1,        /* 1: record CUDA events around every kernel launch (te_get_profile) */
  TE_OPT_GRAPH = 2,          /* 1 (default): replay each restart's launches as a CUDA graph      */
  TE_OPT_KERNELS = 3,        /* projection kernels (same arithmetic, kept for measured comparison):
                                2 (default): chosen by column count (register-accumulator kernel
                                  up to 8 columns, TMA-tiled above);
                                3: TMA-tiled (2-D tensor boxes) warp-specialised projections only;
                                5: register-accumulator projections only (slower above 16
                                  columns: lane groups of <= 4 rows per column load).  Other
                                values: TE_ERR_ARG (round 1's fused sets 0/1 and the shuffle
                                set 4 were removed)                                               */
  TE_OPT_PREFETCH = 4,       /* update_norm's L2 bulk-prefetch distance (block iterations, 0..16;
                                default 0)                                                          */
  TE_OPT_ORTHO = 6,          /* orthogonalisation: 0 (default) CGS2 against the full basis (reading
                                C1, BASELINE north star); 1 the paper's 3-term Lanczos recurrence as
                                printed (Eq. 8; Alg. 1), B_H + 144n bytes/step;
                                2 CGS2 whose second sweep takes c2 = c1 - (V^H V) c1 from the Gram
                                matrix built in the update pass: two V passes per step */
  TE_OPT_INTEGRATOR = 7,     /* error integral: 0 (default) adaptive tanh-sinh;
                                1 non-adaptive Gauss-Legendre of order 30 ("simpler and faster",
                                for explorative runs)                                                 */
  TE_OPT_HALO = 8,           /* distributed handles: 0 (default) halo staged by an NCCL send/recv
                                exchange before each SpMV; 1 the SpMV reads halo columns straight
                                from the owning rank's V column (peer memory: CUDA IPC over NVLink,
                                or the same address space) — SURVEY f4, the exchange fused into
                                the SpMV.  Used with TE_OPT_SPMV 7 or 8.                       */
  TE_OPT_SPMV = 5            /* SpMV kernel (same arithmetic, measured choice):
                                10 column-blocked ring: a copy of the CSR split into equal column
                                blocks of <= 48 MB of x (env TE_SPMV_COLBLK_MB), the ring (7) run
                                once per block (lanes per row from the block's mean row length),
                                passes after the first accumulating into W; each pass gathers
                                from one L2-resident block.  Built at create and the
                                default when the ring is chosen and x exceeds 160 MB (single
                                rank; TE_SPMV_COLBLK=0 disables); TE_ERR_ARG when selected and
                                x fits one block;
                                9 slot-window SELL-32 with a value dictionary: 32-row slices
                                (lane = row), each row's off-diagonal entries grouped by their
                                32-column window, windows merged across the slice into slots
                                (one int32 window base per slot), 8 bits per entry (3-bit value
                                code | 5-bit column offset) when the dictionary holds <= 7 values,
                                else 16 bits (8-bit code | 8-bit offset), dense diagonal.  Built at create when
                                the off-diagonal values take <= 255 distinct values and the slot
                                entries are <= 2.0x (8-bit) / 1.6x (16-bit) the off-diagonal
                                entries (spin chains); then
                                the default.  TE_ERR_ARG when selected and not applicable.
                                env TE_SPMV_SW_PANEL=k (read when the format is built): two
                                launches per SpMV - windows inside the slice's aligned panel of
                                2^k slices in row order, then the far windows added into W in
                                a permuted slice order (halves the DRAM traffic when x exceeds
                                L2; same time on one B200, so not the default);
                                8 staged-x ring: the ring below, and each tile's x windows (column
                                ranges planned on the device at create: >= 2 distinct columns at
                                >= 1/4 density) bulk-copied into shared memory too; entries are
                                addressed by 16-bit slots (0xFFFF: gathered from global memory).
                                The default when the plan stages >= 95 % of the entries, rows hold
                                <= 40 entries on average, n >= 65536 and the slot-window format
                                does not apply (bosons);
                                7 warp-specialised ring: one producer warp bulk-copies (TMA
                                engine) rowptr/col/val of nnz-balanced tiles into a 3-4 stage
                                shared-memory ring, 15 consumer warps (TPR lanes per row, 8-16
                                register gathers in flight per lane) release stages per warp —
                                no block barrier per tile.  The default otherwise (x <= 160 MB);
                                6 SELL-32-sigma: rows sorted by length in 4096-row windows, 32-row
                                slices stored column-major, one lane per row, software-pipelined
                                loads (a padded copy of H is built on the device when selected;
                                TE_ERR_ARG if padding would exceed the entry count).
                                Other values: TE_ERR_ARG (round 1's slower variants were removed) */
};
int te_set_option(te_handle* h, int option, double value);
/* Read-only plan statistics (te_get_option only; -1 when the handle has no such plan).  Staged-x
 * SpMV: entries gathered from global memory / nnz; tiles with at least one such entry / tiles;
 * bulk-copied x slots / nnz.  Slot-window SELL-32: slot entries (padding included) / off-diagonal
 * entries (reported when the value dictionary exists, also when the padding made it inapplicable);
 * TE_INFO_SW_PANEL: log2 of the slices (32 rows) per panel when the slot-window SpMV runs as a
 * two-pass panel sweep (x larger than L2), 0 when it runs as one pass;
 * TE_INFO_SW_FAR: slots of the far-window pass / all slots. */
enum { TE_INFO_XS_GLOBAL = 101, TE_INFO_XS_GLOBAL_TILES = 102, TE_INFO_XS_X_PER_ENTRY = 103, TE_INFO_SW_FILL = 104,
       TE_INFO_SW_PANEL = 105, TE_INFO_SW_FAR = 106 };
/* Current value of an option (TE_OPT_SPMV reports the kernel the handle runs, e.g. the default
 * chosen at create) or of a TE_INFO_* statistic; TE_ERR_ARG for a null handle/pointer or an
 * unknown option. */
int te_get_option(const te_handle* h, int option, double* value);

/* Per-kernel-class profile accumulated while TE_OPT_PROFILE is on (reset by te_set_option):
 * kernel: 0 spmv (K1a), 1 update_proj (K2), 2 update_norm (K3),
 * 3 combine V.omega (K4), 4 halo pack (distributed), 5 proj_dots (K1b), 6 host step
 * search (eigensolve + quadrature + omega; wall-clock ms, alg_bytes 0).  launches, total device milliseconds (CUDA events on the
 * launching stream) and algorithmic bytes. */
typedef struct { int64_t launches; double total_ms; double alg_bytes; } te_kernel_profile;
int te_get_profile(const te_handle* h, int kernel, te_kernel_profile* out);

/* Number of library kernels launched by this handle since creation. */
int64_t te_launch_count(const te_handle* h);

/* ||H||_1 of the handle's matrix (global for distributed handles). */
double te_one_norm(const te_handle* h);

/* Host-side small problem of one restart, exported for testing without a GPU (the same code
 * te_evolve runs on the host, host_math.cpp):
 * te_small_eig: T = tridiag(beta[0..m-2], alpha, beta[0..m-2]) = U diag(lam) U^T by implicit
 *   symmetric QR; lam[m] unsorted, U[m*m] row-major (column k = eigenvector k).
 * te_step_search: Alg. 1 step 2 (reading O-6 of DESIGN.md) on that T with
 *   h = h_{m+1,m}: the step tau and its error integral err = int_0^tau f (Eq. 16) with
 *   err <= tol_rate tau; integrator 0 tanh-sinh (with the O-5a floor), 1 Gauss-Legendre.
 *   TE_ERR_STEP_COLLAPSE below 1e-13 t_total. */
int te_small_eig(int m, const double* alpha, const double* beta, double* lam, double* U);
int te_step_search(int m, const double* alpha, const double* beta, double h, int breakdown, int first,
                   double tau_prev, double rem, double tol_rate, double t_total, int integrator, double* tau,
                   double* err, int* quad_ok);

/* Diagnostics: compiled attributes of a hot-path kernel (which: 0 spmv (the ring kernel, real
 * values, one lane per row), 1 proj_dots, 2 update_proj (TMA), 3 update_norm). */
int te_kernel_attributes(int which, int* regs, int* max_threads, int* static_smem, int* max_dyn_smem);

/* Thread-local status / message of the last failing call (TE_OK / "" if none). */
int te_last_status(void);
const char* te_last_error(void);

/* Library version string. */
const char* te_version(void);

/* ---- distributed (one process per GPU, rows sharded; NCCL over NVLink) --------------- */

/* Rank 0 draws a 128-byte ncclUniqueId (broadcast it with torch.distributed). */
int te_nccl_unique_id(void* out128);

/* Create the library's own NCCL communicator (ncclCommInitRank) on the current device. */
te_dist* te_dist_init(int nranks, int rank, const void* id128);
void te_dist_destroy(te_dist* d);

/* Local rows [row_begin, row_end) of a global n_global x n_global Hermitian CSR, with
 * GLOBAL column indices (int64).  All ranks call collectively with contiguous, ordered,
 * non-overlapping row blocks covering [0, n_global).  val is complex (te_c128) if
 * val_is_complex else double.  Builds the halo plan (te_halo_plan) and exchanges the
 * per-peer need lists once.  v0/v_out of evolve calls are the local row slices.
 * Each rank's global columns must lie in [0, n_global) and increase strictly within a row
 * (checked on the host); the local columns keep that entry order (so each row's sum has the
 * single-GPU order).  Errors are agreed collectively: if any rank's input is invalid or its
 * local create fails, every rank returns NULL (TE_ERR_CSR / TE_ERR_ARG) instead of blocking. */
te_handle* te_create_csr_dist(te_dist* d, int64_t n_global, int64_t row_begin, int64_t row_end,
                              const int64_t* rowptr_local, const int64_t* col_global,
                              const void* val, int val_is_complex);

/* Host-only halo plan (no GPU needed): given the row partition row_starts[nranks+1] and
 * this rank's global column indices, produce
 *   col_local_out[nnz_local]  local columns: own rows -> [0, n_loc), remote columns ->
 *                             n_loc + position in the halo (peers ascending, index ascending)
 *   recv_counts_out[nranks]   halo entries received from each peer (0 for self)
 *   halo_global_out[cap]      the sorted unique remote global indices (halo order)
 * Returns the halo length (>= 0) or -status on error.  Bit-exact and deterministic. */
int64_t te_halo_plan(int nranks, int rank, const int64_t* row_starts, int64_t nnz_local,
                     const int64_t* col_global, int32_t* col_local_out, int64_t* recv_counts_out,
                     int64_t* halo_global_out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* TE_H */
