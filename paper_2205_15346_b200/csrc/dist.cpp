// Row-sharded distributed handles: contiguous row blocks per rank, one halo
// exchange per SpMV over precomputed gather lists (NCCL send/recv over NVLink), batched
// allreduces of the Gram-Schmidt sums.  The halo plan itself is pure host code and is
// exported (te_halo_plan) so it can be tested bit-exactly without a GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/te.h"
#include "nccl_shim.h"

te_handle* te_internal_create_local(int64_t n_loc, int64_t n_global, int64_t row_begin, const int64_t* rowptr,
                                    const int32_t* col_local, const void* val, bool cplx, te_dist* dist,
                                    int64_t ncol_limit);
struct HaloCsr {  // the entries of the local rows whose columns live on other ranks
  std::vector<int32_t> rows;     // local rows with at least one such entry
  std::vector<int64_t> rowptr;   // [rows.size() + 1]
  std::vector<int32_t> col;      // halo index (position in the received halo vector)
  std::vector<unsigned char> val;  // double or double2 per entry
};
int te_internal_setup_halo(te_handle* h, int64_t n_halo, const std::vector<int64_t>& recv_counts,
                           const std::vector<int64_t>& send_counts, const std::vector<int32_t>& send_idx,
                           double norm1_global, const std::vector<int64_t>& halo_global,
                           const std::vector<int64_t>& row_starts, const HaloCsr& hc);
int te_internal_set_error(int code, const char* msg);
cudaStream_t te_internal_stream(te_handle* h);
double te_internal_local_norm1(te_handle* h);
void te_internal_set_norm1(te_handle* h, double v);
ncclComm_t te_internal_comm(te_dist* d);
int te_internal_nranks(te_dist* d);
int te_internal_rank(te_dist* d);

extern "C" int64_t te_halo_plan(int nranks, int rank, const int64_t* row_starts, int64_t nnz_local,
                                const int64_t* col_global, int32_t* col_local_out, int64_t* recv_counts_out,
                                int64_t* halo_global_out, int64_t cap) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !row_starts || (nnz_local > 0 && (!col_global || !col_local_out)) ||
      !recv_counts_out)
    return -te_internal_set_error(TE_ERR_ARG, "te_halo_plan: bad arguments");
  for (int q = 0; q < nranks; ++q)
    if (row_starts[q + 1] < row_starts[q]) return -te_internal_set_error(TE_ERR_ARG, "row_starts not monotone");
  const int64_t n_global = row_starts[nranks];
  const int64_t rb = row_starts[rank], re = row_starts[rank + 1];
  const int64_t n_loc = re - rb;
  std::vector<int64_t> remote;
  remote.reserve(1024);
  for (int64_t k = 0; k < nnz_local; ++k) {
    const int64_t c = col_global[k];
    if (c < 0 || c >= n_global) return -te_internal_set_error(TE_ERR_CSR, "column index out of range");
    if (c < rb || c >= re) remote.push_back(c);
  }
  std::sort(remote.begin(), remote.end());
  remote.erase(std::unique(remote.begin(), remote.end()), remote.end());
  const int64_t n_halo = (int64_t)remote.size();
  if (n_loc + n_halo > INT32_MAX) return -te_internal_set_error(TE_ERR_ARG, "local index space exceeds int32");
  for (int q = 0; q < nranks; ++q) recv_counts_out[q] = 0;
  int owner = 0;
  for (int64_t i = 0; i < n_halo; ++i) {  // sorted, partitions ordered -> owners ascending
    while (remote[i] >= row_starts[owner + 1]) ++owner;
    recv_counts_out[owner] += 1;
  }
  for (int64_t k = 0; k < nnz_local; ++k) {
    const int64_t c = col_global[k];
    if (c >= rb && c < re) {
      col_local_out[k] = (int32_t)(c - rb);
    } else {
      const int64_t pos = std::lower_bound(remote.begin(), remote.end(), c) - remote.begin();
      col_local_out[k] = (int32_t)(n_loc + pos);
    }
  }
  if (halo_global_out)
    for (int64_t i = 0; i < std::min(cap, n_halo); ++i) halo_global_out[i] = remote[i];
  return n_halo;
}

#define DCK(call)                                                                        \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      te_internal_set_error(TE_ERR_CUDA, cudaGetErrorString(e_));                        \
      goto fail;                                                                         \
    }                                                                                    \
  } while (0)
#define DNK(call)                                                                        \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess) {                                                             \
      te_internal_set_error(TE_ERR_NCCL, te::nccl().GetErrorString(r_));                 \
      goto fail;                                                                         \
    }                                                                                    \
  } while (0)

extern "C" te_handle* te_create_csr_dist(te_dist* d, int64_t n_global, int64_t row_begin, int64_t row_end,
                                         const int64_t* rowptr_local, const int64_t* col_global, const void* val,
                                         int val_is_complex) {
  if (!d || n_global < 1 || row_begin < 0 || row_end <= row_begin || row_end > n_global || !rowptr_local) {
    te_internal_set_error(TE_ERR_ARG, "te_create_csr_dist: bad arguments");
    return nullptr;
  }
  const int P = te_internal_nranks(d), me = te_internal_rank(d);
  const int64_t n_loc = row_end - row_begin;
  const int64_t nnz = rowptr_local[n_loc];
  std::vector<int64_t> row_starts(P + 1, 0);
  std::vector<int64_t> recv_counts(P, 0), send_counts(P, 0), halo;
  std::vector<int32_t> col_local(std::max<int64_t>(1, nnz));
  std::vector<int32_t> send_idx;
  int64_t n_halo = 0, n_send = 0;
  std::vector<int64_t> lrp;
  std::vector<int32_t> lcol;
  std::vector<unsigned char> lval;
  HaloCsr hc;
  double norm_rows = 0.0;
  te_handle* h = nullptr;
  int64_t* dbuf = nullptr;
  cudaStream_t st = nullptr;
  ncclComm_t comm = te_internal_comm(d);
  // 0. local structure check of the caller's global CSR (rowptr non-decreasing from 0, columns in
  //    [0, n_global) and strictly increasing per row); the verdict travels with the row partition
  //    so that every rank fails together instead of leaving peers inside a collective
  int64_t local_bad = (rowptr_local[0] != 0) ? 1 : 0;
  for (int64_t r = 0; r < n_loc && !local_bad; ++r) {
    if (rowptr_local[r + 1] < rowptr_local[r]) { local_bad = 1; break; }
    int64_t prev = -1;
    for (int64_t q = rowptr_local[r]; q < rowptr_local[r + 1]; ++q) {
      const int64_t c = col_global[q];
      if (c < 0 || c >= n_global || c <= prev) { local_bad = 1; break; }
      prev = c;
    }
  }
  if (P == 1 && local_bad) {
    te_internal_set_error(TE_ERR_CSR, "te_create_csr_dist: columns out of range or not strictly increasing");
    return nullptr;
  }
  DCK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  if (P > 1) {
    // 1. row partition (+ every rank's structure verdict)
    DCK(cudaMalloc(&dbuf, sizeof(int64_t) * (16 + 4 * P + P * P)));
    {
      int64_t mine[3] = {row_begin, row_end, local_bad};
      std::vector<int64_t> all(3 * P);
      DCK(cudaMemcpy(dbuf, mine, sizeof mine, cudaMemcpyHostToDevice));
      DNK(te::nccl().AllGather(dbuf, dbuf + 3, 3, ncclInt64, comm, st));
      DCK(cudaStreamSynchronize(st));
      DCK(cudaMemcpy(all.data(), dbuf + 3, sizeof(int64_t) * 3 * P, cudaMemcpyDeviceToHost));
      for (int q = 0; q < P; ++q)
        if (all[3 * q + 2]) {
          te_internal_set_error(TE_ERR_CSR, q == me ? "te_create_csr_dist: columns out of range or not strictly increasing"
                                                    : "te_create_csr_dist: invalid CSR on another rank");
          goto fail;
        }
      for (int q = 0; q < P; ++q) {
        if (all[3 * q] != (q == 0 ? 0 : all[3 * q - 2])) {
          te_internal_set_error(TE_ERR_ARG, "row blocks must be contiguous and ordered by rank");
          goto fail;
        }
        row_starts[q] = all[3 * q];
      }
      row_starts[P] = all[3 * (P - 1) + 1];
      if (row_starts[P] != n_global) {
        te_internal_set_error(TE_ERR_ARG, "row blocks do not cover [0, n_global)");
        goto fail;
      }
    }
  } else {
    row_starts[0] = 0;
    row_starts[1] = n_global;
  }
  // 2. halo plan (host, bit-exact)
  halo.resize(std::max<int64_t>(1, nnz));
  n_halo = te_halo_plan(P, me, row_starts.data(), nnz, col_global, col_local.data(), recv_counts.data(), halo.data(),
                        (int64_t)halo.size());
  if (n_halo < 0) goto fail;
  halo.resize(n_halo);
  if (P > 1) {
    // 3. counts matrix: M[q][p] = entries rank q needs from rank p
    int64_t* dM = dbuf + 2 + 2 * P;
    std::vector<int64_t> M((size_t)P * P);
    DCK(cudaMemcpy(dbuf, recv_counts.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice));
    DNK(te::nccl().AllGather(dbuf, dM, P, ncclInt64, comm, st));
    DCK(cudaStreamSynchronize(st));
    DCK(cudaMemcpy(M.data(), dM, sizeof(int64_t) * P * P, cudaMemcpyDeviceToHost));
    for (int q = 0; q < P; ++q) send_counts[q] = (q == me) ? 0 : M[(size_t)q * P + me];
    for (int q = 0; q < P; ++q) n_send += send_counts[q];
    // 4. exchange need lists (global indices)
    int64_t *dneed = nullptr, *dgive = nullptr;
    DCK(cudaMalloc(&dneed, sizeof(int64_t) * std::max<int64_t>(1, n_halo)));
    DCK(cudaMalloc(&dgive, sizeof(int64_t) * std::max<int64_t>(1, n_send)));
    if (n_halo > 0) DCK(cudaMemcpy(dneed, halo.data(), sizeof(int64_t) * n_halo, cudaMemcpyHostToDevice));
    DNK(te::nccl().GroupStart());
    {
      int64_t ro = 0, so = 0;
      for (int q = 0; q < P; ++q) {
        if (q == me) continue;
        if (recv_counts[q] > 0) DNK(te::nccl().Send(dneed + ro, recv_counts[q], ncclInt64, q, comm, st));
        if (send_counts[q] > 0) DNK(te::nccl().Recv(dgive + so, send_counts[q], ncclInt64, q, comm, st));
        ro += recv_counts[q];
        so += send_counts[q];
      }
    }
    DNK(te::nccl().GroupEnd());
    DCK(cudaStreamSynchronize(st));
    {
      std::vector<int64_t> give(n_send);
      if (n_send > 0) DCK(cudaMemcpy(give.data(), dgive, sizeof(int64_t) * n_send, cudaMemcpyDeviceToHost));
      send_idx.resize(n_send);
      for (int64_t t = 0; t < n_send; ++t) {
        if (give[t] < row_begin || give[t] >= row_end) {
          te_internal_set_error(TE_ERR_CSR, "peer requested a row this rank does not own");
          cudaFree(dneed);
          cudaFree(dgive);
          goto fail;
        }
        send_idx[t] = (int32_t)(give[t] - row_begin);
      }
    }
    cudaFree(dneed);
    cudaFree(dgive);
  }
  // 5. split every row into its local-column entries (the handle's CSR: the SpMV runs on them
  //    while the halo is in flight) and its halo entries (a small CSR over the rows that have
  //    any, added by k_spmv_halo once the halo arrived); ||H||_1 from the full rows.  Local
  //    handle with local column indices (Hermiticity needs the global matrix: not checked)
  {
    const size_t vb = val_is_complex ? 16 : 8;
    const unsigned char* vin = static_cast<const unsigned char*>(val);
    lrp.assign((size_t)n_loc + 1, 0);
    lcol.reserve((size_t)std::max<int64_t>(1, nnz));
    lval.reserve((size_t)std::max<int64_t>(1, nnz) * vb);
    hc.rowptr.push_back(0);
    for (int64_t r = 0; r < n_loc; ++r) {
      double rs = 0.0;
      bool any = false;
      for (int64_t q = rowptr_local[r]; q < rowptr_local[r + 1]; ++q) {
        const int32_t c = col_local[(size_t)q];
        const unsigned char* v = vin + (size_t)q * vb;
        double a = 0.0;
        if (val_is_complex) {
          double re, im;
          std::memcpy(&re, v, 8);
          std::memcpy(&im, v + 8, 8);
          a = std::hypot(re, im);
        } else {
          double re;
          std::memcpy(&re, v, 8);
          a = std::fabs(re);
        }
        rs += a;
        if (c < n_loc) {
          lcol.push_back(c);
          lval.insert(lval.end(), v, v + vb);
        } else {
          hc.col.push_back(c - (int32_t)n_loc);
          hc.val.insert(hc.val.end(), v, v + vb);
          any = true;
        }
      }
      lrp[(size_t)r + 1] = (int64_t)lcol.size();
      if (any) {
        hc.rows.push_back((int32_t)r);
        hc.rowptr.push_back((int64_t)hc.col.size());
      }
      norm_rows = std::max(norm_rows, rs);
    }
  }
  h = te_internal_create_local(n_loc, n_global, row_begin, lrp.data(), lcol.data(), lval.data(), val_is_complex != 0,
                               d, n_loc);
  if (!h && P == 1) goto fail;
  {
    // 6. halo buffers and peer tables first (their allocations can fail too), then
    //    ||H||_1 = max over all rows of the row abs sums (allreduce max), together with a
    //    "local setup failed" flag, so that a failure on one rank fails every rank
    bool local_ok = h != nullptr;
    const double norm_loc = norm_rows;
    if (local_ok &&
        te_internal_setup_halo(h, n_halo, recv_counts, send_counts, send_idx, norm_loc, halo, row_starts, hc) != TE_OK)
      local_ok = false;
    double nv[2] = {norm_loc, local_ok ? 0.0 : 1.0};
    if (P > 1) {
      double* dn = reinterpret_cast<double*>(dbuf);
      DCK(cudaMemcpy(dn, nv, sizeof nv, cudaMemcpyHostToDevice));
      DNK(te::nccl().AllReduce(dn, dn, 2, ncclDouble, ncclMax, comm, st));
      DCK(cudaStreamSynchronize(st));
      DCK(cudaMemcpy(nv, dn, sizeof nv, cudaMemcpyDeviceToHost));
    }
    if (!local_ok) goto fail;  // own error already set by te_internal_create_local / setup_halo
    if (nv[1] != 0.0) {
      te_internal_set_error(TE_ERR_CSR, "te_create_csr_dist: local handle setup failed on another rank");
      goto fail;
    }
    te_internal_set_norm1(h, nv[0]);
  }
  cudaFree(dbuf);
  cudaStreamDestroy(st);
  return h;
fail:
  if (h) te_destroy(h);
  if (dbuf) cudaFree(dbuf);
  if (st) cudaStreamDestroy(st);
  return nullptr;
}
