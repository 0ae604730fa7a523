// Microbenchmark: register-accumulator projection kernel k_proj_r<MODE, TPR, CPL, U, MINB> against the
// TMA ring (k_proj_tma) and update_norm, synthetic V (random values), n rows (default 2^23, so V
// exceeds L2 at every column count).  Also checks k_proj_r's dots against k_proj_tma's (relative).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -I include -I <nccl>
//        tools/micro/mb_proj.cu -o tools/micro/mb_proj -L/usr/local/cuda/lib64/stubs -lcuda
// Round-2 results (B200, GB/s at n = 2^20 / 2^23): DESIGN.md §6.
#include "../../paper_2205_15346_b200/csrc/kernels.cu"
#include "../../paper_2205_15346_b200/csrc/spmv.cu"
#include "../../paper_2205_15346_b200/csrc/spmv_xs.cu"
#include "../../paper_2205_15346_b200/csrc/spmv_sw.cu"
#include <cudaTypedefs.h>
#include <cmath>
#include <cstdio>
#include <vector>
using namespace te;

__global__ void k_fill(double2* x, int64_t cnt, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    x[i] = make_double2((double)(z >> 11) * 0x1.0p-53 - 0.5, (double)((z * 31) >> 11) * 0x1.0p-53 - 0.5);
  }
}

template <int MODE, int TPR, int CPL, int U, int MINB>
void run_r(const KDev& d, int j, int sms) {
  k_proj_r<MODE, TPR, CPL, U, MINB><<<sms * MINB, kThreads>>>(d, j);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (1 << 23);
  if (argc > 2) g_proj_balance = atoi(argv[2]);
  const int mcap = 64;
  const int64_t ldv = (n + 31) / 32 * 32;
  double2 *V, *W, *W0, *g, *part; double *small, *partn; unsigned* ctr; int* flag; double2* gs;
  cudaMalloc(&V, sizeof(double2) * ldv * mcap); cudaMalloc(&W, sizeof(double2) * ldv); cudaMalloc(&W0, sizeof(double2) * ldv);
  k_fill<<<4096, 256>>>(V, ldv * mcap, 1); k_fill<<<4096, 256>>>(W0, ldv, 2);
  cudaMalloc(&g, sizeof(double2) * 192); cudaMalloc(&small, sizeof(double) * 1024); cudaMemset(small, 0, 8192);
  cudaMalloc(&part, sizeof(double2) * 64 * 148 * 8); cudaMalloc(&partn, sizeof(double) * 148 * 8);
  cudaMalloc(&ctr, 64); cudaMemset(ctr, 0, 64); cudaMalloc(&flag, 64); cudaMemset(flag, 0, 64);
  cudaMalloc(&gs, 64); cudaMemset(gs, 0, 64);
  KDev d{}; d.n = n; d.ldv = ldv; d.V = V; d.W = W; d.s = small + 512; d.alpha = small; d.beta = small + 64;
  d.flag = flag; d.nrm2 = small + 256; d.g1 = g; d.g2 = g + 64; d.part = part; d.partn = partn; d.counter = ctr;
  d.gsync = gs; d.tol_rate = 0.0; d.defer = 0;
  {  // s_k = 1 for every column, nrm2 = 1 (gate value 1)
    std::vector<double> one(300, 1.0);
    cudaMemcpy(d.s, one.data(), 65 * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d.nrm2, one.data(), 64 * 8, cudaMemcpyHostToDevice);
    double2 gsv = make_double2(1.0, 0.0);
    cudaMemcpy(gs, &gsv, 16, cudaMemcpyHostToDevice);
  }
  configure_kernels();
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int list[] = {2, 4, 6, 8, 12, 16, 20, 24, 28, 32, 40, 48, 64};
  const int NL = sizeof(list) / sizeof(list[0]);
  printf("n = %lld; GB/s (algorithmic bytes: dots 16n(ncols+1), update 16n(ncols+2))\n", (long long)n);
  printf("ncols | tma ring dots upd | same, runtime R | update_norm: k_update_norm no write, write, tma ring write | k_proj_r: TPR/CPL/U/MINB dots upd ...\n");
  for (int li = 0; li < NL; ++li) {
    const int nc = list[li], j = nc - 1;
    CUtensorMap tm;
    cuuint64_t gd[2] = {(cuuint64_t)(2 * n), (cuuint64_t)mcap}; cuuint64_t gst[1] = {(cuuint64_t)(ldv * 16)};
    cuuint32_t box[2] = {(cuuint32_t)(64 * proj_rsub(nc)), (cuuint32_t)nc}; cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, V, gd, gst, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int S = proj_slots(nc), R = proj_rsub(nc), C = proj_consumers(nc);
    const size_t sm = proj_smem_bytes(nc);
    const double bd = 16.0 * n * (nc + 1), bu = 16.0 * n * (nc + 2);
    auto timeit = [&](auto&& launch, int reps) {
      launch();
      cudaEventRecord(e0);
      for (int it = 0; it < reps; ++it) {
        cudaMemcpyAsync(W, W0, 16 * n, cudaMemcpyDeviceToDevice);  // not timed separately: subtracted below
        launch();
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float t; cudaEventElapsedTime(&t, e0, e1);
      cudaError_t er = cudaGetLastError();
      if (er != cudaSuccess) { printf("FAILED: %s\n", cudaGetErrorString(er)); exit(1); }
      return (double)t / reps;
    };
    const double tcopy = timeit([&] {}, 5);
    auto gbs = [&](double ms, double b) { return b / ((ms - tcopy) * 1e6); };
    // the library's own dispatch (launch_proj_dots / launch_update_proj / launch_update_norm) with the
    // TMA ring forced at every column count: compile-time-R builds (default) and the runtime-R fallback
    static CUtensorMap tms[kMaxCols];
    tms[j] = tm;
    Launch L{};
    L.stream = 0; L.num_sms = sms; L.grid_k3 = 8 * sms; L.tmaps = tms; L.proj_tma = 1; L.prefetch = 0;
    L.proj_const_r = 1; L.norm_tma = 0;
    (void)S; (void)R; (void)C; (void)sm;
    // reference dots (TMA) for the check
    std::vector<double2> gref(nc), gr(nc);
    cudaMemcpy(W, W0, 16 * n, cudaMemcpyDeviceToDevice);
    launch_proj_dots(d, j, L);
    cudaMemcpy(gref.data(), d.g1, 16 * nc, cudaMemcpyDeviceToHost);
    const double ttd = timeit([&] { launch_proj_dots(d, j, L); }, 5);
    const double ttu = timeit([&] { launch_update_proj(d, j, L); }, 5);
    const double tn = timeit([&] { launch_update_norm(d, j, false, L); }, 5);
    // the same pass writing column j + 1 (as in the restart loop): 16n more bytes
    const double tnw = nc < mcap ? timeit([&] { launch_update_norm(d, j, true, L); }, 5) : tn;
    L.norm_tma = 1;
    const double tnt = nc < mcap ? timeit([&] { launch_update_norm(d, j, true, L); }, 5) : tn;
    L.proj_const_r = 0;
    const double ttd0 = timeit([&] { launch_proj_dots(d, j, L); }, 5);
    const double ttu0 = timeit([&] { launch_update_proj(d, j, L); }, 5);
    printf("%5d | %5.0f %5.0f | %5.0f %5.0f | %5.0f %5.0f %5.0f |", nc, gbs(ttd, bd), gbs(ttu, bu), gbs(ttd0, bd), gbs(ttu0, bu),
           gbs(tn, bd), nc < mcap ? gbs(tnw, bu) : 0.0, nc < mcap ? gbs(tnt, bu) : 0.0);
    auto variant = [&](auto tpr_c, auto cpl_c, auto u_c, auto minb_c) {
      constexpr int TPR = decltype(tpr_c)::value, CPL = decltype(cpl_c)::value, U = decltype(u_c)::value, MINB = decltype(minb_c)::value;
      if (nc > TPR * CPL || (TPR > 1 && nc <= TPR * CPL / 2)) return;
      cudaMemcpy(W, W0, 16 * n, cudaMemcpyDeviceToDevice);
      run_r<0, TPR, CPL, U, MINB>(d, j, sms);
      cudaMemcpy(gr.data(), d.g1, 16 * nc, cudaMemcpyDeviceToHost);
      double err = 0, nr = 0;
      for (int k = 0; k < nc; ++k) {
        err = fmax(err, hypot(gr[k].x - gref[k].x, gr[k].y - gref[k].y));
        nr = fmax(nr, hypot(gref[k].x, gref[k].y));
      }
      const double td = timeit([&] { run_r<0, TPR, CPL, U, MINB>(d, j, sms); }, 5);
      const double tu = timeit([&] { run_r<1, TPR, CPL, U, MINB>(d, j, sms); }, 5);
      printf(" %d/%d/%d/%d %5.0f %5.0f%s |", TPR, CPL, U, MINB, gbs(td, bd), gbs(tu, bu), err <= 1e-11 * (nr + 1) ? "" : " BAD");
    };
    using I1 = std::integral_constant<int, 1>; using I2 = std::integral_constant<int, 2>;
    using I3 = std::integral_constant<int, 3>; using I4 = std::integral_constant<int, 4>;
    using I8 = std::integral_constant<int, 8>; using I16 = std::integral_constant<int, 16>;
    // TPR/CPL/U/MINB
    variant(I1{}, I4{}, I1{}, I4{}); variant(I1{}, I4{}, I2{}, I2{}); variant(I1{}, I8{}, I1{}, I2{});
    variant(I2{}, I4{}, I1{}, I4{}); variant(I2{}, I4{}, I2{}, I2{}); variant(I2{}, I8{}, I1{}, I2{});
    variant(I4{}, I4{}, I1{}, I4{}); variant(I4{}, I4{}, I2{}, I2{}); variant(I4{}, I8{}, I1{}, I2{});
    printf("\n");
  }
  return 0;
}
