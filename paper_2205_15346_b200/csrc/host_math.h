// Host-side small-problem numerics of Algorithm 1 step 2, written independently
// of the oracle: symmetric tridiagonal eigensolver (diagonalise H_m once per restart),
// the error integrand of Eq. 16, adaptive tanh-sinh quadrature (P:222, P:261,
// P:406) and the step-size search (Eqs. 18-19).
// Readings of the garbled pseudocode: DESIGN.md "Readings" O-5, O-6, C9-C12, C16, C17.
#pragma once
#include <complex>
#include <vector>

namespace te {

struct SmallEig {
  int m = 0;
  std::vector<double> lam;  // eigenvalues (unsorted)
  std::vector<double> U;    // m x m row-major, column i = eigenvector i
  std::vector<double> c;    // c_k = U[m-1][k] * U[0][k]   (Eq. 16 integrand coefficients)
  double h = 0.0;           // h_{m+1,m}
};

// T = tridiag(beta[0..m-2], alpha[0..m-1], beta[0..m-2]); returns false if the implicit QR
// iteration fails to converge.
bool tridiag_eig(int m, const double* alpha, const double* beta, SmallEig& out);

// f(tau) = h |sum_k c_k e^{-i lam_k tau}|
double integrand(const SmallEig& e, double tau);

struct QuadResult { double value; bool converged; };
// tanh-sinh on [a,b]: level k uses u_j = j 2^-k, |u_j| <= 3.5; stop when I_k == 0 or
// (k >= 2 and |I_k - I_{k-1}| <= rel max(|I_k|, floor)); at most 15 refinements.
// floor = tol_rate (b - a) in the step search (reading O-5a).
QuadResult tanh_sinh(const SmallEig& e, double a, double b, double floor, double rel = 1e-3, int max_levels = 15);

// Non-adaptive Gauss-Legendre rule of order 30 on [a,b] (the paper's optional fast scheme).
QuadResult gauss_legendre(const SmallEig& e, double a, double b);

// integrator: 0 adaptive tanh-sinh (default), 1 Gauss-Legendre
QuadResult integrate(const SmallEig& e, double a, double b, double tol_rate, int integrator);

struct StepResult { double tau, err; bool quad_ok; bool collapse; };
// Largest admissible step: e <= tol_rate * tau (reading O-6); integrals use floor tol_rate (b-a).
StepResult find_step(const SmallEig& e, bool breakdown, bool first, double tau_prev, double rem,
                     double tol_rate, double t_total, int integrator = 0);

// omega = U (e^{-i lam tau} .* U[0,:])  (Eq. 11)
void omega(const SmallEig& e, double tau, std::complex<double>* out);

}  // namespace te
