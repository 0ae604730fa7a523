"""Pins for the oracle (oracle/krylov.py) against things other than itself:
closed forms, the mathematics (dense exponentials, Krylov-space definition,
mpmath), special cases that reduce to textbook results, and the paper's printed
values (tests/golden/).  CPU only.
"""
import json
import math
import os

import mpmath
import numpy as np
import pytest
import scipy.integrate as si
import scipy.linalg as sl
import scipy.sparse as sp

from oracle import krylov as K
from workloads import memory_burden as mb
from workloads import configs, models

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def csr_from_dense(A):
    S = sp.csr_matrix(A)
    S.sort_indices()
    return S.indptr.astype(np.int64), S.indices.astype(np.int32), S.data.astype(A.dtype)


def rand_herm(n, density, seed, complex_=True):
    g = np.random.default_rng(seed)
    A = g.standard_normal((n, n)) + (1j * g.standard_normal((n, n)) if complex_ else 0)
    A = A * (g.random((n, n)) < density)
    A = A + A.conj().T
    np.fill_diagonal(A, np.diag(A).real + 0.1)  # keep an explicit diagonal
    return A if complex_ else A.real


def dense_evolve(A, v0, t):
    lam, U = np.linalg.eigh(A)
    return U @ (np.exp(-1j * lam * t) * (U.conj().T @ v0))


# ---------------------------------------------------------------- spmv / norm

def test_spmv_matches_dense_matvec():
    A = rand_herm(57, 0.1, 1)
    rp, c, v = csr_from_dense(A)
    x = np.random.default_rng(2).standard_normal(57) + 1j
    assert np.allclose(K.spmv(rp, c, v, x), A @ x, rtol=0, atol=1e-13)


def test_spmv_identity_and_permutation():
    rp, c, v = csr_from_dense(np.eye(3, dtype=complex))
    x = np.array([1 + 2j, -3, 0.5j])
    assert np.array_equal(K.spmv(rp, c, v, x), x)
    rp, c, v = csr_from_dense(np.array([[0, 1], [1, 0]], dtype=complex))
    assert np.array_equal(K.spmv(rp, c, v, np.array([1, 0], complex)), np.array([0, 1], complex))


def test_spmv_rows_is_a_row_restriction():
    """Dense mat-vec rows (the definition) on a ragged random matrix, including empty rows."""
    A = rand_herm(50, 0.15, 9)
    A[7, :] = 0
    A[:, 7] = 0
    rp, c, v = csr_from_dense(A)
    x = np.random.default_rng(3).standard_normal(50) + 1j * np.random.default_rng(4).standard_normal(50)
    rows = np.array([0, 7, 13, 49, 13])
    assert np.allclose(K.spmv_rows(rp, c, v, x, rows), (A @ x)[rows], rtol=0, atol=1e-13)


def test_one_norm_hand_values():
    rp, c, v = csr_from_dense(np.array([[0, 1], [1, 0]], dtype=float))
    assert K.one_norm(rp, c, v, 2) == 1.0
    rp, c, v = csr_from_dense(np.diag([2.0, -3.0]))
    assert K.one_norm(rp, c, v, 2) == 3.0
    A = rand_herm(40, 0.2, 3)
    rp, c, v = csr_from_dense(A)
    assert math.isclose(K.one_norm(rp, c, v, 40), np.abs(A).sum(axis=0).max(), rel_tol=1e-14)


def test_one_norm_paper_s5_matrix():
    """The P:527 benchmark matrix (config 6): ||H||_1 = 171.515, computed independently in
    SURVEY.md App. A from the column-sum closed form with 50-digit couplings f_i; the roundoff
    estimate of Eq. 17 for one restart is then d ||H||_1 2^-52 = 5.96e-8 (BASELINE.md §1 note)."""
    c = configs.build(6)
    nrm = K.one_norm(c["rowptr"], c["col"], c["val"], c["n"])
    assert abs(nrm - 171.515) <= 5e-4
    assert abs(c["n"] * nrm * 2.0 ** -52 - 5.96e-8) <= 5e-11


# ---------------------------------------------------------------- Arnoldi

@pytest.mark.parametrize("ortho", ["cgs2", "lanczos3", "cgs2gram"])
def test_arnoldi_relation_and_orthonormality(ortho):
    n, m = 120, 12
    A = rand_herm(n, 0.08, 4)
    v = np.random.default_rng(5).standard_normal(n) + 1j * np.random.default_rng(6).standard_normal(n)
    v /= np.linalg.norm(v)
    kr = K.arnoldi(lambda x: A @ x, v, m, 1e-14, ortho)
    V, a, b = kr["V"], kr["alpha"], kr["beta"]
    T = np.diag(a) + np.diag(b[:-1], 1) + np.diag(b[:-1], -1)
    R = A @ V - V @ T
    # Eq. 9: H V_m = V_m H_m + h v_{m+1} e_m^T -> first m-1 residual columns ~ 0, last has norm h
    norm1 = np.abs(A).sum(axis=0).max()
    assert np.linalg.norm(R[:, :-1]) <= 32 * 2**-52 * n * norm1
    assert math.isclose(np.linalg.norm(R[:, -1]), kr["h"], rel_tol=1e-9)
    if ortho in ("cgs2", "cgs2gram"):
        assert np.abs(V.conj().T @ V - np.eye(m)).max() <= 1e-13


def test_arnoldi_spans_krylov_space():
    """span(V_m) = span{v, Hv, ..., H^{m-1} v} (Eq. 2)."""
    n, m = 60, 6
    A = rand_herm(n, 0.15, 7)
    v = np.random.default_rng(8).standard_normal(n).astype(complex)
    v /= np.linalg.norm(v)
    kr = K.arnoldi(lambda x: A @ x, v, m, 1e-14)
    P = np.stack([np.linalg.matrix_power(A, k) @ v for k in range(m)], axis=1)
    Q, _ = np.linalg.qr(P)
    # projectors onto the two subspaces agree
    assert np.abs(Q @ Q.conj().T - kr["V"] @ kr["V"].conj().T).max() < 1e-9


def test_arnoldi_tridiagonal_matches_projection():
    """H_m = V_m^H H V_m."""
    n, m = 80, 10
    A = rand_herm(n, 0.1, 9)
    v = np.ones(n, complex) / math.sqrt(n)
    kr = K.arnoldi(lambda x: A @ x, v, m, 1e-14)
    V = kr["V"]
    Hm = V.conj().T @ A @ V
    T = np.diag(kr["alpha"]) + np.diag(kr["beta"][:-1], 1) + np.diag(kr["beta"][:-1], -1)
    assert np.abs(Hm - T).max() < 1e-12


def test_breakdown_pauli_pair_and_eigenvector():
    X = np.array([[0, 1], [1, 0]], complex)
    kr = K.arnoldi(lambda x: X @ x, np.array([1, 0], complex), 5, 1e-10)
    assert kr["m_eff"] == 2 and kr["breakdown"]
    assert np.allclose(kr["alpha"], [0, 0]) and kr["beta"][0] == 1.0 and kr["h"] == 0.0
    D = np.diag([2.5, -1.0, 4.0]).astype(complex)
    kr = K.arnoldi(lambda x: D @ x, np.array([1, 0, 0], complex), 3, 1e-10)
    assert kr["m_eff"] == 1 and kr["alpha"][0] == 2.5 and kr["h"] == 0.0


# ---------------------------------------------------------------- small eig / integrand

def test_small_eig_against_mpmath():
    g = np.random.default_rng(10)
    a, b = g.standard_normal(7), np.abs(g.standard_normal(7))
    lam, U = K.small_eig(a, b)
    T = mpmath.matrix(7, 7)
    for i in range(7):
        T[i, i] = a[i]
        if i < 6:
            T[i, i + 1] = T[i + 1, i] = b[i]
    mpmath.mp.dps = 40
    E, Q = mpmath.eigsy(T)
    ev = sorted(float(x) for x in E)
    assert np.allclose(lam, ev, rtol=0, atol=1e-13)
    Tn = np.diag(a) + np.diag(b[:6], 1) + np.diag(b[:6], -1)
    assert np.abs(U @ np.diag(lam) @ U.T - Tn).max() <= 100 * 2**-52 * 7 * np.abs(Tn).max()


def test_integrand_2x2_closed_form():
    a, b, c, h = 0.3, 0.7, -1.1, 0.25
    lam, U = K.small_eig(np.array([a, c]), np.array([b, 0.0]))
    Om = math.sqrt(((a - c) / 2) ** 2 + b ** 2)
    tau = np.linspace(0, 3, 17)
    exact = h * np.abs(b / Om * np.sin(Om * tau))   # |e2^T e^{-iT tau} e1|
    assert np.allclose(K.integrand(lam, U, h, tau), exact, rtol=0, atol=1e-15)


def test_integrand_against_dense_expm():
    g = np.random.default_rng(11)
    a, b = g.standard_normal(8), np.abs(g.standard_normal(8))
    T = np.diag(a) + np.diag(b[:7], 1) + np.diag(b[:7], -1)
    lam, U = K.small_eig(a, b)
    for tau in (0.0, 0.5, 2.3):
        ref = 0.3 * abs(sl.expm(-1j * T * tau)[7, 0])
        assert abs(K.integrand(lam, U, 0.3, tau) - ref) < 1e-12
    assert K.integrand(lam, U, 0.0, 1.7) == 0.0
    assert K.integrand(lam, U, 0.3, 0.0) < 1e-15


def test_omega_against_dense_expm():
    g = np.random.default_rng(12)
    a, b = g.standard_normal(6), np.abs(g.standard_normal(6))
    T = np.diag(a) + np.diag(b[:5], 1) + np.diag(b[:5], -1)
    lam, U = K.small_eig(a, b)
    e1 = np.zeros(6); e1[0] = 1
    assert np.abs(K.omega(lam, U, 0.7) - sl.expm(-1j * T * 0.7) @ e1).max() < 1e-13
    lam, U = K.small_eig(np.zeros(2), np.array([1.0, 0]))       # Pauli: (cos t, -i sin t)
    assert np.allclose(K.omega(lam, U, 0.4), [math.cos(0.4), -1j * math.sin(0.4)], atol=1e-15)


# ---------------------------------------------------------------- quadrature

def test_tanh_sinh_textbook_integrals():
    v, ok = K.tanh_sinh(np.sin, 0.0, math.pi)
    assert ok and abs(v - 2.0) <= 2e-3
    v, ok = K.tanh_sinh(np.sin, 0.0, math.pi, rel=1e-13)
    assert ok and abs(v - 2.0) <= 1e-12
    v, ok = K.tanh_sinh(lambda x: 1 / np.sqrt(x), 0.0, 1.0, rel=1e-10)
    assert abs(v - 2.0) <= 1e-6
    v, ok = K.tanh_sinh(np.exp, 0.0, 1.0, rel=1e-13)
    assert abs(v - (math.e - 1)) <= 1e-12
    v, ok = K.tanh_sinh(lambda x: np.ones_like(x), 0.0, 1.0)
    assert ok and abs(v - 1.0) < 1e-12
    assert K.tanh_sinh(np.sin, 1.0, 1.0) == (0.0, True)


def test_error_integral_2x2_closed_form():
    """int_0^t h |b/Om sin(Om tau)| dtau = h |b| (1 - cos Om t) / Om^2  for Om t <= pi."""
    a, b, c, h = 0.1, 0.9, 0.4, 0.6
    lam, U = K.small_eig(np.array([a, c]), np.array([b, 0.0]))
    Om = math.sqrt(((a - c) / 2) ** 2 + b ** 2)
    t = 0.9 * math.pi / Om
    exact = h * abs(b) * (1 - math.cos(Om * t)) / Om ** 2
    v, ok = K.tanh_sinh(lambda x: K.integrand(lam, U, h, x), 0.0, t)
    assert ok and abs(v - exact) <= 1e-3 * exact
    v, _ = K.tanh_sinh(lambda x: K.integrand(lam, U, h, x), 0.0, t, rel=1e-12)
    assert abs(v - exact) <= 1e-12


def _count_calls(f):
    calls = [0]

    def g(x):
        calls[0] += np.size(x)
        return f(x)
    return g, calls


def test_error_integral_floor_o5a_2x2_closed_form():
    """Reading O-5a: the stop test |I_k - I_{k-1}| <= 1e-3 max(|I_k|, floor) with
    floor = tol_rate (b - a).  Pinned on the closed-form 2x2 error integral
    h |b| (1 - cos Om tau) / Om^2 (Eq. 16; P:406's relative 1e-3 test):
      * floor active (tol_rate tau >> exact): |I - exact| <= 1e-3 tol_rate tau, and the rule stops
        at level 2 (29 nodes: 7 + 8 + 14), where the pure relative test refines further;
      * floor inactive (tol_rate tau << exact): the relative 1e-3 accuracy of P:406 is kept;
      * the floor scales with (b - a): the same tol_rate on a 100x longer interval is inactive
        again for an integral that grows like tau^2."""
    a, b, c, h = 0.1, 0.9, 0.4, 0.6
    lam, U = K.small_eig(np.array([a, c]), np.array([b, 0.0]))
    Om = math.sqrt(((a - c) / 2) ** 2 + b ** 2)

    def exact(t):
        return h * abs(b) * (1 - math.cos(Om * t)) / Om ** 2

    f = lambda x: K.integrand(lam, U, h, x)  # noqa: E731
    # floor active
    tau, tol_rate = 1e-4, 1e-3
    assert tol_rate * tau > 10 * exact(tau)
    g, calls = _count_calls(f)
    v, ok = K.tanh_sinh(g, 0.0, tau, floor=tol_rate * tau)
    assert ok and abs(v - exact(tau)) <= 1e-3 * max(exact(tau), tol_rate * tau)
    assert calls[0] == 29
    g0, calls0 = _count_calls(f)
    v0, ok0 = K.tanh_sinh(g0, 0.0, tau)
    assert ok0 and abs(v0 - exact(tau)) <= 1e-3 * exact(tau)
    assert calls0[0] >= calls[0]
    # floor inactive: same result as the plain relative test
    tau2, tol_rate2 = 0.9 * math.pi / Om, 1e-9
    assert tol_rate2 * tau2 < 1e-3 * exact(tau2)
    v2, ok2 = K.tanh_sinh(f, 0.0, tau2, floor=tol_rate2 * tau2)
    v2r, _ = K.tanh_sinh(f, 0.0, tau2)
    assert ok2 and abs(v2 - exact(tau2)) <= 1e-3 * exact(tau2) and v2 == v2r
    # sub-interval [tau, tau + s] (the step search's substep pieces): floor tol_rate * s
    t0, s = 0.5, 0.05
    piece = exact(t0 + s) - exact(t0)
    v3, ok3 = K.tanh_sinh(f, t0, t0 + s, floor=1e-2 * s)
    assert ok3 and abs(v3 - piece) <= 1e-3 * max(piece, 1e-2 * s)


def test_error_integral_floor_o5a_roundoff_regime():
    """The regime O-5a exists for: for m = 10 and small tau the true integrand is
    h prod(beta) tau^(m-1)/(m-1)! + O(tau^m) (leading Taylor term of e_m^T exp(-iT tau) e_1 for a
    tridiagonal T), far below the roundoff noise h m eps of the eigendecomposition formula.  With
    the floor the rule converges at level 2 and returns the integral within 1e-3 tol_rate tau of
    the true value h prod(beta) tau^m / m!; the evolution's own calls (evolve -> find_step) pass
    the same floor, checked through the 29-node count of a first-restart integral."""
    g = np.random.default_rng(5)
    m = 10
    alpha = g.standard_normal(m)
    beta = np.abs(g.standard_normal(m)) + 0.5
    lam, U = K.small_eig(alpha, beta[: m - 1])
    h = beta[m - 1]
    tau, tol_rate = 1e-3, 1e-11
    true = h * float(np.prod(beta[: m - 1])) * tau ** m / math.factorial(m)
    assert true < 1e-30
    f = lambda x: K.integrand(lam, U, h, x)  # noqa: E731
    gf, calls = _count_calls(f)
    v, ok = K.tanh_sinh(gf, 0.0, tau, floor=tol_rate * tau)
    assert ok and calls[0] == 29
    assert abs(v - true) <= 1e-3 * max(true, tol_rate * tau)
    # without the floor the relative test chases the noise through many more levels
    gf0, calls0 = _count_calls(f)
    K.tanh_sinh(gf0, 0.0, tau)
    assert calls0[0] > 4 * calls[0]


def test_evolve_first_step_error_matches_closed_form():
    """The ledger entry of the first restart of an m = 2 evolution on a 3x3 Hermitian H from e_1
    equals the closed-form 2x2 error integral (Eq. 16; T = [[a, b], [b, c]] built by hand from H:
    a = H_00, b = ||H e_0 - a e_0||, v_1 = (H e_0 - a e_0)/b, c = v_1^H H v_1, h = ||H v_1 - c v_1
    - b e_0||) within the O-5a tolerance 1e-3 max(e, tol_rate tau) — so evolve passes the floor as
    tol_rate (b - a) and integrates [0, tau] (a wrong floor scale or interval shows here)."""
    H = np.array([[0.3, 0.5 - 0.2j, 0.1j], [0.5 + 0.2j, -0.4, 0.25], [-0.1j, 0.25, 0.7]])
    e0 = np.array([1.0, 0.0, 0.0], dtype=np.complex128)
    a = H[0, 0].real
    r = H @ e0 - a * e0
    b = np.linalg.norm(r)
    v1 = r / b
    c = np.vdot(v1, H @ v1).real
    hh = np.linalg.norm(H @ v1 - c * v1 - b * e0)
    Om = math.sqrt(((a - c) / 2) ** 2 + b ** 2)
    rp, col, val = csr_from_dense(H)
    for t, tol in [(0.5, 1e-3), (0.5, 1e-6), (2.0, 1e-2)]:
        res = K.evolve(rp, col, val, e0, t, tol, 2)
        tau, m_eff, e = res["schedule"][0]
        assert m_eff == 2 and Om * tau <= math.pi
        ex = hh * abs(b) * (1 - math.cos(Om * tau)) / Om ** 2
        assert abs(e - ex) <= 1e-3 * max(ex, tol / t * tau)


def test_error_integral_against_mpmath_quad():
    g = np.random.default_rng(13)
    a, b = g.standard_normal(10), np.abs(g.standard_normal(10)) + 0.1
    lam, U = K.small_eig(a, b)
    f = lambda x: K.integrand(lam, U, 0.5, x)  # noqa: E731
    ref = float(mpmath.quad(lambda x: float(f(float(x))), [0, 0.4, 0.8, 1.2]))
    v, ok = K.tanh_sinh(f, 0.0, 1.2)
    assert ok and abs(v - ref) <= 1e-3 * ref


# ---------------------------------------------------------------- step search

def _setup_step(seed, m=8, h=0.3):
    g = np.random.default_rng(seed)
    a, b = g.standard_normal(m), np.abs(g.standard_normal(m)) + 0.2
    lam, U = K.small_eig(a, b)
    f = lambda x: K.integrand(lam, U, h, x)  # noqa: E731
    integ = lambda lo, hi: K.tanh_sinh(f, lo, hi)[0]  # noqa: E731
    return f, integ


def test_step_search_breakdown_takes_remaining_time():
    integ = lambda lo, hi: 0.0  # noqa: E731   h = 0: f == 0
    tau, e = K.find_step(integ, True, False, 0.5, 3.7, 1e-6, 10.0)
    assert tau == 3.7 and e == 0.0
    tau, e = K.find_step(integ, False, True, None, 3.7, 1e-6, 10.0)
    assert tau == 3.7 and e == 0.0


@pytest.mark.parametrize("first", [True, False])
def test_step_search_rate_and_bracket(first):
    f, integ = _setup_step(14)
    tol_rate = 1e-6
    tau, e = K.find_step(integ, False, first, 0.3, 50.0, tol_rate, 100.0)
    # independent integrals (scipy adaptive Gauss-Kronrod)
    E = lambda x: si.quad(f, 0, x, limit=200, epsabs=0, epsrel=1e-12)[0]  # noqa: E731
    assert e <= tol_rate * tau
    assert abs(E(tau) - e) <= 2e-3 * E(tau)
    s = None
    # the step cannot be extended by one more substep (it stops at the first failure)
    # bisection bracket: the rate inequality fails somewhere within (tau, tau + tau/5]
    s = tau / 10 * 2
    assert E(tau + s) > tol_rate * (tau + s) * (1 - 2e-3)


def test_step_search_monotone_in_tol_rate():
    f, integ = _setup_step(15)
    prev = 0.0
    for tr in (1e-9, 1e-8, 1e-7, 1e-6, 1e-5):
        tau, _ = K.find_step(integ, False, True, None, 1e3, tr, 1e3)
        assert tau >= prev
        prev = tau


def test_step_collapse():
    integ = lambda lo, hi: 1.0 * (hi - lo)  # noqa: E731   f == h = 1 (m = 1)
    with pytest.raises(K.StepCollapse):
        K.find_step(integ, False, True, None, 1.0, 1e-3, 1.0)


def test_roundoff_arithmetic():
    rp, c, v = csr_from_dense(np.array([[0, 1], [1, 0]], dtype=float))
    r = K.evolve(rp, c, v, np.array([1, 0], complex), 1.0, 1e-6, 2)
    assert r["roundoff_step"] == 2 * 1.0 * 2 ** -52  # 4.44e-16 (Eq. 17)


# ---------------------------------------------------------------- evolution

def test_evolve_pauli_t_pi():
    rp, c, v = csr_from_dense(np.array([[0, 1], [1, 0]], dtype=complex))
    r = K.evolve(rp, c, v, np.array([1, 0], complex), math.pi, 1e-10, 10)
    assert np.abs(r["v"] - np.array([-1, 0])).max() < 1e-10


def test_evolve_rabi_closed_form():
    """H = (Delta/2) sz + (Om/2) sx: P_1(t) = Om^2/(Om^2+D^2) sin^2(sqrt(Om^2+D^2) t/2)."""
    D, Om, t = 0.7, 1.3, 3.1
    A = np.array([[D / 2, Om / 2], [Om / 2, -D / 2]], complex)
    rp, c, v = csr_from_dense(A)
    r = K.evolve(rp, c, v, np.array([1, 0], complex), t, 1e-10, 10)
    W = math.sqrt(Om ** 2 + D ** 2)
    assert abs(abs(r["v"][1]) ** 2 - Om ** 2 / W ** 2 * math.sin(W * t / 2) ** 2) < 1e-10


def test_evolve_block_rabi_ensemble():
    """Block-diagonal ensemble of independent 2x2 Rabi problems: closed form at any n,
    and the Krylov space is not exact (many distinct frequencies) so real stepping occurs."""
    nb = 300
    g = np.random.default_rng(16)
    D, Om = g.uniform(-1, 1, nb), g.uniform(0.2, 2, nb)
    A = sp.block_diag([np.array([[d / 2, o / 2], [o / 2, -d / 2]]) for d, o in zip(D, Om)]).tocsr()
    A.sort_indices()
    v0 = (g.standard_normal(2 * nb) + 1j * g.standard_normal(2 * nb))
    v0 /= np.linalg.norm(v0)
    t, tol = 6.0, 1e-9
    r = K.evolve(A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data, v0, t, tol, 20)
    exact = np.zeros_like(v0)
    for k in range(nb):
        W = math.sqrt(D[k] ** 2 + Om[k] ** 2)
        Hk = np.array([[D[k] / 2, Om[k] / 2], [Om[k] / 2, -D[k] / 2]])
        # e^{-iHt} = cos(Wt/2) I - i sin(Wt/2) (2H/W)
        Uk = math.cos(W * t / 2) * np.eye(2) - 1j * math.sin(W * t / 2) * (2 * Hk / W)
        exact[2 * k: 2 * k + 2] = Uk @ v0[2 * k: 2 * k + 2]
    err = np.linalg.norm(r["v"] - exact)
    assert r["restarts"] > 1
    assert err <= r["bound"] + 10 * r["roundoff_total"]
    assert r["bound"] <= tol


@pytest.mark.parametrize("seed,n,complex_", [(17, 64, True), (18, 150, False), (19, 200, True)])
def test_evolve_vs_dense_and_bound(seed, n, complex_):
    A = rand_herm(n, 0.05, seed, complex_)
    rp, c, v = csr_from_dense(A)
    g = np.random.default_rng(seed + 100)
    v0 = g.standard_normal(n) + 1j * g.standard_normal(n)
    v0 /= np.linalg.norm(v0)
    t, tol = 5.0, 1e-7
    r = K.evolve(rp, c, v, v0, t, tol, 15)
    ve = dense_evolve(A, v0, t)
    err = np.linalg.norm(r["v"] - ve)
    assert r["bound"] <= tol
    assert err <= r["bound"] + 10 * r["roundoff_total"]          # bound validity (Eq. 16)
    assert abs(np.linalg.norm(r["v"]) - 1) <= r["bound"] + 10 * r["roundoff_total"]
    e0 = np.vdot(v0, A @ v0).real
    e1 = np.vdot(r["v"], A @ r["v"]).real
    assert abs(e1 - e0) <= 2 * np.abs(A).sum(0).max() * (r["bound"] + r["roundoff_total"])
    assert math.fsum(s[0] for s in r["schedule"]) == pytest.approx(t, rel=0, abs=1e-12)
    assert sum(s[1] for s in r["schedule"]) == r["krylov_steps"]


def test_evolve_time_reversal_and_determinism():
    A = rand_herm(90, 0.06, 20)
    rp, c, v = csr_from_dense(A)
    v0 = np.ones(90, complex) / math.sqrt(90)
    r1 = K.evolve(rp, c, v, v0, 4.0, 1e-8, 12)
    r1b = K.evolve(rp, c, v, v0, 4.0, 1e-8, 12)
    assert np.array_equal(r1["v"], r1b["v"]) and r1["schedule"] == r1b["schedule"]
    r2 = K.evolve(rp, c, -v, r1["v"] / np.linalg.norm(r1["v"]), 4.0, 1e-8, 12)
    assert np.linalg.norm(r2["v"] - v0) <= 2e-8


def test_evolve_edge_cases():
    rp, c, v = csr_from_dense(np.diag([1.0, 2.0]))
    v0 = np.array([1, 0], complex)
    r = K.evolve(rp, c, v, v0, 0.0, 1e-8, 5)
    assert r["restarts"] == 0 and np.array_equal(r["v"], v0) and r["bound"] == 0
    with pytest.raises(K.NotNormalized):
        K.evolve(rp, c, v, np.array([1, 1], complex), 1.0, 1e-8, 5)
    # eigenvector: one restart, breakdown at j=0, exact phase
    r = K.evolve(rp, c, v, v0, 3.0, 1e-8, 5)
    assert r["restarts"] == 1 and r["breakdowns"] == 1
    assert abs(r["v"][0] - np.exp(-3j)) < 1e-14
    # m_max > n: capped at n
    A = rand_herm(5, 0.5, 21)
    rp, c, v = csr_from_dense(A)
    v0 = np.ones(5, complex) / math.sqrt(5)
    r = K.evolve(rp, c, v, v0, 2.0, 1e-9, 40)
    assert np.linalg.norm(r["v"] - dense_evolve(A, v0, 2.0)) < 1e-9


def test_lanczos3_agrees_with_cgs2_within_bounds():
    A = rand_herm(100, 0.05, 22)
    rp, c, v = csr_from_dense(A)
    v0 = np.ones(100, complex) / 10
    ra = K.evolve(rp, c, v, v0, 3.0, 1e-9, 10, ortho="cgs2")
    rb = K.evolve(rp, c, v, v0, 3.0, 1e-9, 10, ortho="lanczos3")
    assert np.linalg.norm(ra["v"] - rb["v"]) <= ra["bound"] + rb["bound"] + 1e-12


def test_xxz_one_magnon_exact():
    """One-magnon sector of the XXZ(+NNN) chain is an L x L problem (SURVEY §8(c) pin):
    exact L x L exponential vs the oracle on the full 2^L space."""
    L = 10
    h = models.xxz_fields(L, 5)
    J1, J2, Dl = 1.0, 0.5, 1.0
    rp, c, v = models.xxz_csr(L, J1, Dl, h, J2=J2)
    # reference state all-down has diagonal energy E_ref
    E_ref = (J1 * L + J2 * L) * Dl / 4 - 0.5 * h.sum()
    M = np.zeros((L, L))
    for k in range(L):
        M[k, k] = E_ref - J1 * Dl - J2 * Dl + h[k]
        M[k, (k + 1) % L] = M[(k + 1) % L, k] = J1 / 2
        M[k, (k + 2) % L] = M[(k + 2) % L, k] = J2 / 2
    g = np.random.default_rng(23)
    a = g.standard_normal(L) + 1j * g.standard_normal(L)
    a /= np.linalg.norm(a)
    v0 = np.zeros(1 << L, complex)
    v0[[1 << k for k in range(L)]] = a
    t = 3.0
    r = K.evolve(rp, c, v, v0, t, 1e-10, 30)
    exact = sl.expm(-1j * M * t) @ a
    out = r["v"][[1 << k for k in range(L)]]
    assert np.linalg.norm(out - exact) <= r["bound"] + 1e-13
    mask = np.ones(1 << L, bool)
    mask[[1 << k for k in range(L)]] = False
    assert np.all(r["v"][mask] == 0)      # other Sz sectors stay exactly zero


# ---------------------------------------------------------------- paper's printed values

def test_paper_forward_backward_p509():
    gold = json.load(open(os.path.join(GOLDEN, "paper_p509_forward_backward.json")))
    H = mb.hamiltonian()
    assert H["n"] == gold["dimension"]
    v0 = np.zeros(H["n"], complex)
    v0[H["init_index"]] = 1
    t, tol = gold["t"], gold["err_max_each_way"]
    r1 = K.evolve(H["rowptr"], H["col"], H["val"], v0, t, tol, 40)
    r2 = K.evolve(H["rowptr"], H["col"], -H["val"], r1["v"], t, tol, 40)
    err = np.linalg.norm(r2["v"] - v0)
    assert err <= gold["requested_bound"]
    assert r1["bound"] + r2["bound"] <= gold["requested_bound"]
    # true forward error against the dense exponential of the d = 588 matrix
    Hd = sp.csr_matrix((H["val"], H["col"], H["rowptr"])).toarray()
    assert np.linalg.norm(sl.expm(-1j * t * Hd) @ v0 - r1["v"]) <= r1["bound"] + 1e-12


def test_paper_dimensions_p527_p535():
    gold = json.load(open(os.path.join(GOLDEN, "paper_dimensions.json")))
    for case in gold["cases"]:
        p = dict(mb.DEFAULTS, **case["params"])
        assert mb.dimension(p) == case["d"]
    occ, _, _ = mb.basis(mb.DEFAULTS)
    assert occ.shape[0] == 588


def test_gauss_legendre_exactness():
    """Order-30 Gauss-Legendre (P:406 option) is exact for polynomials of degree <= 59."""
    v, ok = K.gauss_legendre(lambda x: x ** 59 + 3 * x ** 2, 0.0, 1.0)
    assert abs(v - (1 / 60 + 1.0)) < 1e-13
    v, _ = K.gauss_legendre(np.exp, 0.0, 1.0)
    assert abs(v - (math.e - 1)) < 1e-13
    assert K.gauss_legendre(np.sin, 2.0, 2.0) == (0.0, True)


@pytest.mark.parametrize("integrator", ["tanh-sinh", "gauss"])
def test_intermediate_samples_vs_dense(integrator):
    """states sampled inside a step from that step's Krylov space; each sample is within
    its own bound of the exact exp(-iH t_s) v0, and the sample at t equals the final state."""
    A = rand_herm(120, 0.06, 31)
    rp, c, v = csr_from_dense(A)
    v0 = np.ones(120, complex) / math.sqrt(120)
    ts = [0.0, 0.3, 1.1, 2.0, 2.9, 3.0]
    r = K.evolve(rp, c, v, v0, 3.0, 1e-8, 10, samples=ts, integrator=integrator)
    assert r["restarts"] > 1
    assert np.array_equal(r["samples"][0], v0)
    assert np.array_equal(r["samples"][-1], r["v"])
    for tsi, s, b in zip(ts, r["samples"], r["sample_bounds"]):
        assert np.linalg.norm(s - dense_evolve(A, v0, tsi)) <= b + 1e-12
    assert r["sample_bounds"][-1] == pytest.approx(r["bound"], rel=1e-9)


def test_cgs2gram_equals_cgs2_to_roundoff():
    """f2: the Gram-corrected second sweep reproduces CGS2 (same T, same basis) to roundoff,
    also deep into a restart where plain CGS would lose orthogonality."""
    A = rand_herm(400, 0.02, 41)
    v0 = np.random.default_rng(42).standard_normal(400) + 0j
    v0 /= np.linalg.norm(v0)
    a = K.arnoldi(lambda x: A @ x, v0, 40, 1e-14, "cgs2")
    b = K.arnoldi(lambda x: A @ x, v0, 40, 1e-14, "cgs2gram")
    assert np.abs(a["alpha"] - b["alpha"]).max() < 1e-12 * np.abs(a["alpha"]).max()
    assert np.abs(a["beta"] - b["beta"]).max() < 1e-12 * np.abs(a["beta"]).max()
    assert np.linalg.norm(a["V"] - b["V"]) < 1e-11
    assert np.abs(b["V"].conj().T @ b["V"] - np.eye(40)).max() < 1e-13
