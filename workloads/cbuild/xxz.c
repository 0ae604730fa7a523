/* Fast host builder of the XXZ(+NNN) chain CSR (input generator only; no Krylov arithmetic).
 * Identical definition and floating-point operation order as workloads/models.py:xxz_csr:
 * diagonal = 0.0, += (+-) J*Delta*0.25 over bonds in order (NN i=0..L-1, then NNN), then
 * += (+-) 0.5*h_i for i = 0..L-1; off-diagonal 0.5*J at col = row ^ ((1<<a)|(1<<b)) for each
 * antiparallel bond; entries of a row sorted by column.  Compiled without FMA contraction. */
#include <stdint.h>
#include <stdlib.h>

static int nbonds(int L, double J2, int* a, int* b, double* J, double J1) {
  int nb = 0;
  for (int i = 0; i < L; ++i) { a[nb] = i; b[nb] = (i + 1) % L; J[nb] = J1; ++nb; }
  if (J2 != 0.0)
    for (int i = 0; i < L; ++i) { a[nb] = i; b[nb] = (i + 2) % L; J[nb] = J2; ++nb; }
  return nb;
}

/* pass 1: row lengths of rows [r0, r1) -> local rowptr (r1-r0+1, starting at 0) */
void xxz_rowptr(int L, double J1, double J2, int64_t r0, int64_t r1, int64_t* rowptr) {
  int a[128], b[128];
  double J[128];
  const int nb = nbonds(L, J2, a, b, J, J1);
  const int64_t m = r1 - r0;
  rowptr[0] = 0;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    const int64_t r = r0 + i;
    int cnt = 1;
    for (int k = 0; k < nb; ++k) cnt += (int)(((r >> a[k]) ^ (r >> b[k])) & 1);
    rowptr[i + 1] = cnt;
  }
  for (int64_t i = 0; i < m; ++i) rowptr[i + 1] += rowptr[i];
}

/* pass 2: fill col (global indices) / val of rows [r0, r1) */
void xxz_fill(int L, double J1, double J2, double delta, const double* h, int64_t r0, int64_t r1,
              const int64_t* rowptr, int32_t* col, double* val) {
  int a[128], b[128];
  double J[128];
  const int nb = nbonds(L, J2, a, b, J, J1);
#pragma omp parallel for schedule(static)
  for (int64_t r = r0; r < r1; ++r) {
    int64_t cc[130];
    double vv[130];
    int m = 0;
    double diag = 0.0;
    for (int k = 0; k < nb; ++k) {
      const int anti = (int)(((r >> a[k]) ^ (r >> b[k])) & 1);
      const double zz = J[k] * delta * 0.25;
      diag = diag + (anti ? -zz : zz);
      if (anti) {
        cc[m] = r ^ (((int64_t)1 << a[k]) | ((int64_t)1 << b[k]));
        vv[m] = 0.5 * J[k];
        ++m;
      }
    }
    for (int i = 0; i < L; ++i) {
      const double half = 0.5 * h[i];
      diag = diag + (((r >> i) & 1) ? half : -half);
    }
    cc[m] = r;
    vv[m] = diag;
    ++m;
    /* insertion sort by column (distinct columns) */
    for (int i = 1; i < m; ++i) {
      int64_t c = cc[i];
      double v = vv[i];
      int q = i - 1;
      while (q >= 0 && cc[q] > c) { cc[q + 1] = cc[q]; vv[q + 1] = vv[q]; --q; }
      cc[q + 1] = c;
      vv[q + 1] = v;
    }
    int64_t o = rowptr[r - r0];
    for (int i = 0; i < m; ++i) { col[o + i] = (int32_t)cc[i]; val[o + i] = vv[i]; }
  }
}
