#include "host_math.h"

#include <cmath>
#include <mutex>

namespace te {

// ------------------------------------------------------------------------------------------
// Eigen-decomposition of the real symmetric tridiagonal T = tridiag(beta, alpha, beta) (P:331:
// "diagonalise once per restart") by implicit symmetric QR steps with the Wilkinson shift and
// bulge chasing (Golub & Van Loan, Matrix Computations, §8.3: Algorithms 8.3.2-8.3.3), written
// out here: every step applies Givens rotations G in planes (k, k+1), T <- G T G^T, and
// accumulates Z <- Z G^T, so that T = Z diag(lam) Z^T at the end (columns of Z = eigenvectors).
// Deflation: an off-diagonal |b_i| <= 2^-53 (|a_i| + |a_{i+1}|) is set to 0.
// ------------------------------------------------------------------------------------------
bool tridiag_eig(int m, const double* alpha, const double* beta, SmallEig& out) {
  out.m = m;
  std::vector<double> a(alpha, alpha + m), b(m > 1 ? m - 1 : 1, 0.0);
  for (int i = 0; i + 1 < m; ++i) b[i] = beta[i];
  std::vector<double>& Z = out.U;  // row-major m x m
  Z.assign((size_t)m * m, 0.0);
  for (int i = 0; i < m; ++i) Z[(size_t)i * m + i] = 1.0;
  const double tiny = std::ldexp(1.0, -53);
  auto negligible = [&](int i) { return std::fabs(b[i]) <= tiny * (std::fabs(a[i]) + std::fabs(a[i + 1])); };
  int hi = m - 1, steps = 0;
  while (hi > 0) {
    if (negligible(hi - 1)) {  // trailing eigenvalue converged
      b[hi - 1] = 0.0;
      --hi;
      continue;
    }
    int lo = hi - 1;  // the unreduced block [lo, hi]
    while (lo > 0 && !negligible(lo - 1)) --lo;
    if (lo > 0) b[lo - 1] = 0.0;
    if (++steps > 60 * m) return false;
    // Wilkinson shift from the trailing 2 x 2 block of [lo, hi]
    const double dl = 0.5 * (a[hi - 1] - a[hi]);
    const double bh = b[hi - 1];
    const double mu = a[hi] - bh * bh / (dl + (dl >= 0.0 ? 1.0 : -1.0) * std::hypot(dl, bh));
    double x = a[lo] - mu, z = b[lo];
    for (int k = lo; k < hi; ++k) {
      const double r = std::hypot(x, z);
      const double c = r == 0.0 ? 1.0 : x / r, s = r == 0.0 ? 0.0 : z / r;
      if (k > lo) b[k - 1] = r;  // the bulge at (k+1, k-1) is rotated away
      const double app = a[k], aqq = a[k + 1], apq = b[k];
      a[k] = c * c * app + 2.0 * c * s * apq + s * s * aqq;
      a[k + 1] = s * s * app - 2.0 * c * s * apq + c * c * aqq;
      b[k] = c * s * (aqq - app) + (c * c - s * s) * apq;
      if (k + 1 < hi) {  // new bulge at (k+2, k)
        z = s * b[k + 1];
        b[k + 1] *= c;
        x = b[k];
      }
      for (int i = 0; i < m; ++i) {
        double* zr = &Z[(size_t)i * m];
        const double zp = zr[k], zq = zr[k + 1];
        zr[k] = c * zp + s * zq;
        zr[k + 1] = c * zq - s * zp;
      }
    }
  }
  out.lam = a;
  out.c.resize(m);
  for (int k = 0; k < m; ++k) out.c[k] = Z[(size_t)(m - 1) * m + k] * Z[k];
  return true;
}

double integrand(const SmallEig& e, double tau) {
  double re = 0.0, im = 0.0;
  for (int k = 0; k < e.m; ++k) {
    double sn, cs;
    sincos(e.lam[k] * tau, &sn, &cs);
    re += e.c[k] * cs;
    im -= e.c[k] * sn;
  }
  return e.h * std::hypot(re, im);
}

// ------------------------------------------------------------------------------------------
// tanh-sinh node tables on the reference interval, built once per process
// x = a + hw d (u < 0), b - hw d (u > 0), mid (u = 0), with d = 1 - |tanh s| = 2/(1+e^{2|s|}),
// s = pi/2 sinh u; weight hw * (pi/2) cosh u / cosh^2 s.
// ------------------------------------------------------------------------------------------
namespace {
constexpr double kUmax = 3.5;
constexpr int kMaxLevels = 15;
struct Level {
  std::vector<double> d, w;
  std::vector<signed char> side;
};
Level g_levels[kMaxLevels + 1];
std::once_flag g_once[kMaxLevels + 1];

// level tables are built lazily (level 15 alone has 7 * 2^14 nodes)
void build_level(int k) {
  const double half_pi = 0.5 * M_PI;
  const double step = std::ldexp(1.0, -k);
  const long jmax = (long)std::floor(kUmax / step);
  Level& L = g_levels[k];
  for (long j = -jmax; j <= jmax; ++j) {
    if (k > 0 && (j % 2 == 0)) continue;
    const double u = (double)j * step;
    const double s = half_pi * std::sinh(u);
    const double cs = std::cosh(s);
    L.d.push_back(2.0 / (1.0 + std::exp(2.0 * std::fabs(s))));
    L.w.push_back(half_pi * std::cosh(u) / (cs * cs));
    L.side.push_back(u < 0 ? -1 : (u > 0 ? 1 : 0));
  }
}
}  // namespace

QuadResult tanh_sinh(const SmallEig& e, double a, double b, double floor, double rel, int max_levels) {
  if (b == a) return {0.0, true};
  const double c = 0.5 * (a + b), hw = 0.5 * (b - a);
  double total = 0.0, prev = 0.0, cur = 0.0;
  if (max_levels > kMaxLevels) max_levels = kMaxLevels;
  for (int k = 0; k <= max_levels; ++k) {
    std::call_once(g_once[k], build_level, k);
    const Level& L = g_levels[k];
    double s = 0.0;
    for (size_t q = 0; q < L.d.size(); ++q) {
      const double x = L.side[q] < 0 ? a + hw * L.d[q] : (L.side[q] > 0 ? b - hw * L.d[q] : c);
      s += hw * L.w[q] * integrand(e, x);
    }
    total += s;
    cur = total * std::ldexp(1.0, -k);
    if (cur == 0.0) return {cur, true};
    if (k >= 2 && std::fabs(cur - prev) <= rel * std::fmax(std::fabs(cur), floor)) return {cur, true};
    prev = cur;
  }
  return {cur, false};
}

// ------------------------------------------------------------------------------------------
// Gauss-Legendre nodes of order 30 by Newton iteration on P_30 (Abramowitz-Stegun start values)
// ------------------------------------------------------------------------------------------
namespace {
constexpr int kGaussOrder = 30;
double g_gx[kGaussOrder], g_gw[kGaussOrder];
std::once_flag g_gonce;
void build_gauss() {
  const int n = kGaussOrder;
  for (int i = 0; i < n; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-16) break;
    }
    g_gx[i] = x;
    g_gw[i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
}
}  // namespace

QuadResult gauss_legendre(const SmallEig& e, double a, double b) {
  if (b == a) return {0.0, true};
  std::call_once(g_gonce, build_gauss);
  const double c = 0.5 * (a + b), hw = 0.5 * (b - a);
  double s = 0.0;
  for (int i = 0; i < kGaussOrder; ++i) s += g_gw[i] * integrand(e, c + hw * g_gx[i]);
  return {hw * s, true};
}

QuadResult integrate(const SmallEig& e, double a, double b, double tol_rate, int integrator) {
  return integrator == 1 ? gauss_legendre(e, a, b) : tanh_sinh(e, a, b, tol_rate * (b - a));
}

// ------------------------------------------------------------------------------------------
// step search (Alg. 1 step 2, P:303-318 with P:262; reading O-6)
// ------------------------------------------------------------------------------------------
StepResult find_step(const SmallEig& e, bool breakdown, bool first, double tau_prev, double rem,
                     double tol_rate, double t_total, int integrator) {
  bool qok = true;
  auto I = [&](double lo, double hi) {
    QuadResult r = integrate(e, lo, hi, tol_rate, integrator);
    if (!r.converged) qok = false;
    return r.value;
  };
  auto ok = [&](double tau, double err) { return err <= tol_rate * tau; };
  if (breakdown) {  // exact subspace: take the remaining time
    const double err = I(0.0, rem);
    return {rem, err, qok, false};
  }
  double tau, err;
  if (first) {  // initial guess 0.1, doubling while admissible
    tau = std::fmin(0.1, rem);
    err = I(0.0, tau);
    if (ok(tau, err)) {
      while (2.0 * tau <= rem) {
        const double e2 = I(0.0, 2.0 * tau);
        if (!ok(2.0 * tau, e2)) break;
        tau = 2.0 * tau;
        err = e2;
      }
    }
  } else {  // previous step slightly reduced
    tau = std::fmin(0.97 * tau_prev, rem);
    err = I(0.0, tau);
  }
  while (!ok(tau, err)) {  // halve
    tau = tau / 2.0;
    if (tau < 1e-13 * t_total) return {tau, err, qok, true};
    err = I(0.0, tau);
  }
  const double s = tau / 10.0;  // N_SUBSTEPS = 10 (reading C10), extend (C9)
  for (;;) {
    if (tau + s >= rem) {
      const double dlt = I(tau, rem);
      if (ok(rem, err + dlt)) {
        tau = rem;
        err += dlt;
      }
      break;
    }
    const double dlt = I(tau, tau + s);
    if (ok(tau + s, err + dlt)) {
      tau += s;
      err += dlt;
    } else {
      break;
    }
  }
  return {tau, err, qok, false};
}

void omega(const SmallEig& e, double tau, std::complex<double>* out) {
  const int m = e.m;
  std::vector<std::complex<double>> y(m);
  for (int k = 0; k < m; ++k) {
    double sn, cs;
    sincos(e.lam[k] * tau, &sn, &cs);
    y[k] = std::complex<double>(cs, -sn) * e.U[k];  // e^{-i lam_k tau} U[0][k]
  }
  for (int i = 0; i < m; ++i) {
    std::complex<double> acc(0.0, 0.0);
    for (int k = 0; k < m; ++k) acc += e.U[(size_t)i * m + k] * y[k];
    out[i] = acc;
  }
}

}  // namespace te
