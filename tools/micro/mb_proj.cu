// Microbenchmark of the hot-path kernels on synthetic data (no library state): times the TMA
// projection kernel in its three modes (0 dots, 1 update+dots, 2 streaming only) and the
// register update_norm kernel for a range of column counts, n = 2^20 rows.
#include "../../paper_2205_15346_b200/csrc/kernels.cu"
#include "../../paper_2205_15346_b200/csrc/spmv.cu"
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
using namespace te;
int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (1 << 20);
  if (argc > 3) g_proj_min_tile = atoll(argv[3]);
  const int mcap = 48;
  const int64_t ldv = (n + 31) / 32 * 32;
  double2 *V, *W, *g, *part; double *small, *partn; unsigned* ctr;
  cudaMalloc(&V, sizeof(double2) * ldv * mcap); cudaMalloc(&W, sizeof(double2) * ldv);
  cudaMemset(V, 0, sizeof(double2) * ldv * mcap); cudaMemset(W, 0, sizeof(double2) * ldv);
  cudaMalloc(&g, sizeof(double2) * 192); cudaMalloc(&small, sizeof(double) * 512); cudaMemset(small, 0, 4096);
  cudaMalloc(&part, sizeof(double2) * 64 * 148 * 8); cudaMalloc(&partn, sizeof(double) * 148 * 8);
  cudaMalloc(&ctr, 64); cudaMemset(ctr, 0, 64);
  KDev d{}; d.n = n; d.ldv = ldv; d.V = V; d.W = W; d.s = small + 130; d.alpha = small; d.beta = small + 64;
  d.flag = (int*)(small + 128); d.nrm2 = small + 196; d.g1 = g; d.g2 = g + 64; d.part = part; d.partn = partn; d.counter = ctr;
  configure_kernels();
  cudaFuncSetAttribute(k_proj_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 205 * 1024);
  // variants: 16 register-accumulated columns, 1 or 2 CTAs per SM (half the slot budget each)
  cudaFuncSetAttribute(k_proj_tma<0, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 205 * 1024);
  cudaFuncSetAttribute(k_proj_tma<1, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 205 * 1024);
  cudaFuncSetAttribute(k_proj_tma<0, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 205 * 1024);
  cudaFuncSetAttribute(k_proj_tma<1, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 205 * 1024);
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int list[] = {2, 4, 5, 6, 8, 9, 12, 16, 17, 20, 23, 24, 28, 32, 33, 41, 48};
  int first = argc > 2 ? atoi(argv[2]) : 0;
  for (int li = first; li < 17; ++li) { const int nc = list[li];
    CUtensorMap tm;
    cuuint64_t gd[2] = {(cuuint64_t)(2 * n), (cuuint64_t)mcap}; cuuint64_t gs[1] = {(cuuint64_t)(ldv * 16)};
    cuuint32_t box[2] = {(cuuint32_t)(64 * proj_rsub(nc)), (cuuint32_t)nc}; cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, V, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int j = nc - 1, S = proj_slots(nc), R = proj_rsub(nc), C = proj_consumers(nc);
    const size_t sm = proj_smem_bytes(nc);
    double ms[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    const int tpr = tpr_for(nc, 1);
    const int gs4 = (int)std::min<int64_t>(4 * sms, (n * tpr + 255) / 256);
    for (int mode = 0; mode < 10; ++mode) {
      for (int it = 0; it < 6; ++it) {
        if (it == 1) cudaEventRecord(e0);
        if (mode == 0) k_proj_tma<0><<<sms, kProjThreads, sm>>>(tm, d, j, S, R, C, 0);
        if (mode == 1) k_proj_tma<1><<<sms, kProjThreads, sm>>>(tm, d, j, S, R, C, 0);
        if (mode == 2) k_proj_tma<2><<<sms, kProjThreads, sm>>>(tm, d, j, S, R, C, 0);
        if (mode == 3) k_update_norm<<<8 * sms, kThreads>>>(d, j, 0, 0);
        if (mode == 4) { TE_DISPATCH_TPR(tpr, { k_proj_s<0, TPR><<<gs4, kThreads>>>(d, j); }); }
        if (mode == 5) { TE_DISPATCH_TPR(tpr, { k_proj_s<1, TPR><<<gs4, kThreads>>>(d, j); }); }
        if (mode == 6) k_proj_tma<0, 8><<<sms, kProjThreads, sm>>>(tm, d, j, S, R, C, 0);
        if (mode == 7) k_proj_tma<1, 8><<<sms, kProjThreads, sm>>>(tm, d, j, S, R, C, 0);
        if (mode == 8) k_proj_tma<0, 16><<<sms, kProjThreads, sm>>>(tm, d, j, S, R, C, 0);
        if (mode == 9) k_proj_tma<1, 16><<<sms, kProjThreads, sm>>>(tm, d, j, S, R, C, 0);
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      { cudaError_t er = cudaGetLastError(); if (er != cudaSuccess) { printf("ncols %d mode %d FAILED: %s\n", nc, mode, cudaGetErrorString(er)); return 1; } }
      float t; cudaEventElapsedTime(&t, e0, e1); ms[mode] = t / 5;
    }
    const double b01 = 16.0 * n * nc + 16.0 * n, b1 = 16.0 * n * nc + 32.0 * n;
    printf("ncols %2d S %2d R %d | tma dots %.0f upd %.0f stream %.0f | norm %.0f | shuffle dots %.0f upd %.0f | "
           "r8 dots %.0f upd %.0f | r16 dots %.0f upd %.0f GB/s | %s\n",
           nc, S, R, b01 / ms[0] / 1e6, b1 / ms[1] / 1e6, b01 / ms[2] / 1e6, b01 / ms[3] / 1e6, b01 / ms[4] / 1e6,
           b1 / ms[5] / 1e6, b01 / ms[6] / 1e6, b1 / ms[7] / 1e6, b01 / ms[8] / 1e6, b1 / ms[9] / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
