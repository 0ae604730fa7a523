#include "host_math.h"

#include <cmath>
#include <mutex>

namespace te {

// ------------------------------------------------------------------------------------------
// implicit QL with Wilkinson-type shifts on a symmetric tridiagonal matrix, accumulating the
// rotations into U (columns = eigenvectors).  Textbook algorithm (Golub & Van Loan §8.3,
// "tql2"/"tqli" family), restated in 0-based form.
// ------------------------------------------------------------------------------------------
bool tridiag_eig(int m, const double* alpha, const double* beta, SmallEig& out) {
  out.m = m;
  std::vector<double> d(alpha, alpha + m), e(m, 0.0);
  for (int i = 0; i + 1 < m; ++i) e[i] = beta[i];
  std::vector<double>& z = out.U;
  z.assign((size_t)m * m, 0.0);
  for (int i = 0; i < m; ++i) z[(size_t)i * m + i] = 1.0;
  for (int l = 0; l < m; ++l) {
    int iter = 0;
    int mm;
    do {
      for (mm = l; mm < m - 1; ++mm) {
        const double dd = std::fabs(d[mm]) + std::fabs(d[mm + 1]);
        if (std::fabs(e[mm]) + dd == dd) break;
      }
      if (mm != l) {
        if (iter++ == 100) return false;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[mm] - d[l] + e[l] / (g + std::copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool deflated = false;
        for (i = mm - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = std::hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[mm] = 0.0;
            deflated = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          for (int k = 0; k < m; ++k) {
            double* zk = &z[(size_t)k * m];
            f = zk[i + 1];
            zk[i + 1] = s * zk[i] + c * f;
            zk[i] = c * zk[i] - s * f;
          }
        }
        if (deflated) continue;
        d[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    } while (mm != l);
  }
  out.lam = d;
  out.c.resize(m);
  for (int k = 0; k < m; ++k) out.c[k] = z[(size_t)(m - 1) * m + k] * z[k];
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
