"""ORACLE — plain, slow, single-threaded CPU implementation of TimeEvolver's
restarted Krylov method (Michel & Zell, arXiv:2205.15346).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code with the CUDA library ``paper_2205_15346_b200``
(and never imports it); the library never imports this.

Citations: ``P:n`` = line n of the paper's LaTeX source; the
readings of ambiguous passages are SURVEY.md §8(c) O-1..O-9 / C1..C18 and are
listed in DESIGN.md "Readings".  Everything is complex128 / float64.

Functions and what pins them (tests/test_oracle_pins.py):
  spmv            y = H x, row by row (Eq. 8 first line)
                  pinned: dense mat-vec, identity/permutation.
  spmv_rows       the same definition for listed rows only (sampled full-size checks)
                  pinned: dense mat-vec rows, empty rows.
  one_norm        ||H||_1 = max column abs sum (Eq. 17)
                  pinned: hand values, scaling.
  arnoldi         Eq. 8 / Alg. 1 step 1 with ortho
                  'cgs2' (C1, parity reference) or 'lanczos3' (paper-literal)
                  pinned: Arnoldi relation, orthonormality, breakdown examples.
  small_eig       diagonalise T once per restart — numpy eigh
                  pinned: reconstruction, mpmath eigsy.
  integrand       f(tau) = h |e_m^T exp(-i T tau) e_1| (Eq. 16)
                  pinned: 2x2 closed form, dense expm, f(0)=0, h=0.
  tanh_sinh       double-exponential quadrature, rel 1e-3, <= 15 levels
                  (reading O-5/C14)
                  pinned: int sin = 2, int x^-1/2 = 2, int e^x = e-1, closed-form
                  2x2 integral, mpmath.quad.
  find_step       Alg. 1 step 2 + P:262 + P:332-333 (reading O-6/C9/C11/C12)
                  pinned: breakdown -> remaining time, rate inequality,
                  monotone in tol_rate, bisection bracket within one substep.
  evolve          Alg. 1: restart loop, V.omega (Eq. 11),
                  ledger, roundoff warning (Eq. 17)
                  pinned: dense exp(-iHt) v, Rabi closed form, Pauli t=pi,
                  block-diagonal Rabi ensemble, bound >= true error,
                  norm/energy conservation, time reversal, partition of t.
"""
from __future__ import annotations

import math

import numpy as np

EPS = 2.0 ** -52          # machine epsilon used in Eq. 17 (reading C15)
T_GUESS = 0.1             # Alg. 1 line 1: t_step = 0.1
SHRINK = 0.97             # Alg. 1 step 2: t_step := 0.97 t_step
N_SUBSTEPS = 10           # named N_SUBSTEPS; value per reading C10
QUAD_REL = 1e-3           # relative error estimate below 1e-3
QUAD_MAX_LEVELS = 15      # "with 15 refinements"
QUAD_UMAX = 3.5           # truncation of the tanh-sinh u-axis (reading O-5)
COLLAPSE = 1e-13          # step-collapse threshold tau < 1e-13 t (reading C17)

WARN_ROUNDOFF = 1         # roundoff estimate exceeds the analytic bound
WARN_QUADRATURE = 2       # integral not converged after 15 refinements


class StepCollapse(RuntimeError):
    pass


class NotNormalized(ValueError):
    pass


# ---------------------------------------------------------------------------
# sparse matrix helpers (the only large-space operation)
# ---------------------------------------------------------------------------

def spmv(rowptr, col, val, x):
    """y_i = sum_k val[k] x[col[k]] over row i's entries (Eq. 8, ``w_j = H v_j``).

    Written as the plain definition: form every product, then add each product
    into its row with ``np.add.at`` (unbuffered, in storage order).
    """
    n = rowptr.shape[0] - 1
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    y = np.zeros(n, dtype=np.complex128)
    np.add.at(y, rows, val * x[col])
    return y


def spmv_rows(rowptr, col, val, x, rows):
    """(H x)_r for the listed rows r only: the definition of ``spmv`` restricted to those rows
    (sampled full-size checks, where the full product is too slow for the oracle)."""
    rows = np.asarray(rows, dtype=np.int64)
    y = np.zeros(rows.shape[0], dtype=np.complex128)
    for i, r in enumerate(rows):
        a, b = int(rowptr[r]), int(rowptr[r + 1])
        y[i] = np.sum(val[a:b] * x[col[a:b]])
    return y


def one_norm(rowptr, col, val, n):
    """||H||_1 = max_j sum_i |H_ij| (Eq. 17)."""
    s = np.zeros(n, dtype=np.float64)
    np.add.at(s, col, np.abs(val))
    return float(s.max()) if n else 0.0


# ---------------------------------------------------------------------------
# Step 1: Arnoldi / Lanczos (Eq. 8; Alg. 1)
# ---------------------------------------------------------------------------

def arnoldi_step(matvec, V, beta, j, ortho="cgs2"):
    """One iteration j of Eq. 8 on the basis columns V[:, :j+1]; returns the
    orthogonalised vector p, alpha_j and beta_j = ||p||_2 (see ``arnoldi``)."""
    p = matvec(V[:, j])
    if ortho == "cgs2":
        Vj = V[:, : j + 1]
        c1 = Vj.conj().T @ p
        p = p - Vj @ c1
        c2 = Vj.conj().T @ p
        p = p - Vj @ c2
        a = (c1[j] + c2[j]).real
    elif ortho == "lanczos3":
        if j > 0:
            p = p - beta[j - 1] * V[:, j - 1]
        aa = np.vdot(V[:, j], p)
        p = p - aa * V[:, j]
        a = aa.real
    elif ortho == "cgs2gram":
        # SURVEY f2 (low-synchronisation CGS2): the second sweep's coefficients from the Gram
        # matrix, c2 = V^H (p - V c1) = c1 - (V^H V) c1, then one update with c1 + c2
        Vj = V[:, : j + 1]
        c1 = Vj.conj().T @ p
        G = Vj.conj().T @ Vj
        c2 = c1 - G @ c1
        p = p - Vj @ (c1 + c2)
        a = (c1[j] + c2[j]).real
    else:
        raise ValueError(ortho)
    b = math.sqrt(np.vdot(p, p).real)
    if not math.isfinite(b):
        raise FloatingPointError("non-finite value in the Arnoldi recurrence")
    return p, a, b


def arnoldi(matvec, v1, m, tol_rate, ortho="cgs2"):
    """Build the Krylov basis from v_1 = w (no renormalisation, C13).

    Works with A = H and a real symmetric tridiagonal T (reading O-3/C4:
    algebraically identical to the paper's A = -iH, anti-Hermitian M).

    ortho="cgs2"     classical Gram-Schmidt against all previous columns plus
                     one re-orthogonalisation pass (BASELINE north star; C1):
                        c1 = V^H p ; p -= V c1 ; c2 = V^H p ; p -= V c2
                        alpha_j = Re(c1_j + c2_j)               (C2, C3)
    ortho="lanczos3" the paper's recurrence as printed:
                        p -= beta_{j-1} v_{j-1} ; a = v_j^H p ; p -= a v_j
    ortho="cgs2gram" SURVEY f2: c1 = V^H p ; c2 = c1 - (V^H V) c1 ; p -= V (c1 + c2)
                     (equal to CGS2 in exact arithmetic; one update pass instead of two)

    beta_j = ||p||_2 (Eq. 8 ``h_{j+1,j}``).  Lucky breakdown when
    beta_j < tol_rate (Alg. 1; reading C6/C7): stop with m_eff = j+1 and
    keep h = beta_j.  Otherwise v_{j+1} = p / beta_j, and at j = m-1
    h = beta_{m-1}.
    """
    n = v1.shape[0]
    m = min(m, n)
    V = np.zeros((n, m), dtype=np.complex128)
    alpha = np.zeros(m)
    beta = np.zeros(m)
    V[:, 0] = v1
    m_eff = m
    breakdown = False
    for j in range(m):
        p, alpha[j], b = arnoldi_step(matvec, V, beta, j, ortho)
        beta[j] = b
        if b < tol_rate:
            m_eff = j + 1
            breakdown = True
            break
        if j < m - 1:
            V[:, j + 1] = p / b
    return dict(V=V[:, :m_eff], alpha=alpha[:m_eff], beta=beta[:m_eff],
                h=float(beta[m_eff - 1]), m_eff=m_eff, breakdown=breakdown)


# ---------------------------------------------------------------------------
# Step 2: small problem, error integrand, quadrature, step search
# ---------------------------------------------------------------------------

def small_eig(alpha, beta):
    """T = tridiag(beta[0..m-2], alpha, beta[0..m-2]) = U diag(lam) U^T
    (diagonalise once per restart)."""
    m = alpha.shape[0]
    T = np.diag(alpha)
    if m > 1:
        T = T + np.diag(beta[: m - 1], 1) + np.diag(beta[: m - 1], -1)
    lam, U = np.linalg.eigh(T)
    return lam, U


def integrand(lam, U, h, tau):
    """f(tau) = h |e_m^T exp(-i T tau) e_1| = h |sum_k U_{m,k} U_{1,k} e^{-i lam_k tau}|
    (Eq. 16; Alg. 1)."""
    m = lam.shape[0]
    c = U[m - 1, :] * U[0, :]
    tau = np.asarray(tau, dtype=np.float64)
    s = np.exp(-1j * np.multiply.outer(tau, lam)) @ c
    return h * np.abs(s)


def tanh_sinh(f, a, b, rel=QUAD_REL, max_levels=QUAD_MAX_LEVELS, umax=QUAD_UMAX, floor=0.0):
    """Adaptive tanh-sinh quadrature of f on [a, b].

    Textbook Takahasi-Mori form (reading O-5):
      x(u) = (a+b)/2 + (b-a)/2 tanh(pi/2 sinh u), evaluated as the distance
             (b-a)/2 * 2/(1+e^{2|s|}) from the nearer endpoint, s = pi/2 sinh u
      w(u) = (b-a)/2 (pi/2) cosh u / cosh^2(pi/2 sinh u)
      I_k  = 2^-k sum_{|j 2^-k| <= umax} w(u_j) f(x(u_j)),  u_j = j 2^-k
    Level k adds the odd j.  Stop when I_k == 0, or k >= 2 and
    |I_k - I_{k-1}| <= rel max(|I_k|, floor).  Returns (I, converged).

    ``floor`` (reading O-5a): the step search passes tol_rate (b - a), the
    size below which a piece of the error integral cannot change any decision
    e <= tol_rate tau; without it, integrands at the roundoff floor (tiny tau,
    f ~ h m eps noise) only converge after ~13 refinements.
    """
    if b == a:
        return 0.0, True
    c = 0.5 * (a + b)
    hw = 0.5 * (b - a)

    def nodes(level):
        step = 2.0 ** -level
        jmax = int(math.floor(umax / step))
        j = np.arange(-jmax, jmax + 1)
        if level > 0:
            j = j[j % 2 != 0]
        u = j * step
        s = 0.5 * math.pi * np.sinh(u)
        # distance to the nearer endpoint, 1 -+ tanh(s) = 2 / (1 + e^{+-2s}),
        # so nodes never collapse onto an endpoint singularity
        d = 2.0 / (1.0 + np.exp(2.0 * np.abs(s)))
        x = np.where(u < 0, a + hw * d, np.where(u > 0, b - hw * d, c))
        w = hw * 0.5 * math.pi * np.cosh(u) / np.cosh(s) ** 2
        return x, w

    total = 0.0
    prev = None
    for k in range(max_levels + 1):
        x, w = nodes(k)
        total += float(np.sum(w * f(x)))
        cur = total * 2.0 ** -k
        if cur == 0.0:
            return cur, True
        if k >= 2 and abs(cur - prev) <= rel * max(abs(cur), floor):
            return cur, True
        prev = cur
    return cur, False


def gauss_legendre(f, a, b, order=30):
    """Non-adaptive Gauss-Legendre rule of the given order on [a, b] (the paper's optional
    "non-adaptive Gauss-scheme"; order 30 per SPEC reading).  numpy.leggauss gives the nodes."""
    if b == a:
        return 0.0, True
    x, w = np.polynomial.legendre.leggauss(order)
    c, hw = 0.5 * (a + b), 0.5 * (b - a)
    return float(hw * np.sum(w * f(c + hw * x))), True


def find_step(integral, breakdown, first, tau_prev, rem, tol_rate, t_total):
    """Largest admissible step per Alg. 1 step 2, P:262, P:332-333,
    Eqs. 18-19; cleaned reading O-6 (C9, C11, C12, C16).

    ``integral(a, b)`` returns int_a^b f.  ok(tau, e) <=> e <= tol_rate tau.
    Returns (tau, e) with e = int_0^tau f <= tol_rate tau (sum of pieces).
    """
    def ok(tau, e):
        return e <= tol_rate * tau

    if breakdown:                                   # O-6.1 (exact subspace)
        return rem, integral(0.0, rem)
    if first:                                       # O-6.2 first restart
        tau = min(T_GUESS, rem)
        e = integral(0.0, tau)
        if ok(tau, e):
            while 2.0 * tau <= rem:
                e2 = integral(0.0, 2.0 * tau)
                if not ok(2.0 * tau, e2):
                    break
                tau, e = 2.0 * tau, e2
    else:                                           # later restarts
        tau = min(SHRINK * tau_prev, rem)
        e = integral(0.0, tau)
    while not ok(tau, e):                           # O-6.3 halve
        tau = tau / 2.0
        if tau < COLLAPSE * t_total:
            raise StepCollapse("step size collapsed below 1e-13 t")
        e = integral(0.0, tau)
    s = tau / N_SUBSTEPS                            # O-6.4 substeps
    while True:
        if tau + s >= rem:
            d = integral(tau, rem)
            if ok(rem, e + d):
                tau, e = rem, e + d
            break
        d = integral(tau, tau + s)
        if ok(tau + s, e + d):
            tau, e = tau + s, e + d
        else:
            break
    return tau, e


def omega(lam, U, tau):
    """omega = exp(-i T tau) e_1 = U (e^{-i lam tau} * U[0, :]) (Eq. 11; C8)."""
    return U @ (np.exp(-1j * lam * tau) * U[0, :])


# ---------------------------------------------------------------------------
# Algorithm 1
# ---------------------------------------------------------------------------

def evolve(rowptr, col, val, v0, t, tol, m, ortho="cgs2", schedule=None,
           max_restarts=1_000_000, samples=None, integrator="tanh-sinh"):
    """v(t) ~= exp(-iHt) v0 with the rigorous bound (Alg. 1).

    ``schedule`` (optional list of step sizes) forces the step sequence
    (parity mode, reading C16): each step's bound is still integrated.
    ``samples`` (ascending times in [0, t]): states at intermediate times from the restart
    whose interval contains them, w_s = V exp(-iT (t_s - t_now)) e_1; returned in
    res["samples"] with per-sample bounds res["sample_bounds"].
    ``integrator``: "tanh-sinh" (default) or "gauss".
    Returns dict(v, bound, restarts, krylov_steps, schedule=[(tau, m_eff, e)],
    warnings, roundoff_step, roundoff_total, breakdowns).
    """
    n = v0.shape[0]
    if tol <= 0 or m < 1 or t < 0 or not math.isfinite(t):
        raise ValueError("bad arguments")
    nv = math.sqrt(np.vdot(v0, v0).real)
    if abs(nv - 1.0) > 1e-8:                       # P:175 / O-1
        raise NotNormalized("initial vector is not normalised")
    w = np.array(v0, dtype=np.complex128)
    res = dict(bound=0.0, restarts=0, krylov_steps=0, schedule=[], warnings=0,
               breakdowns=0)
    samples = [] if samples is None else [float(x) for x in samples]
    res["samples"] = [None] * len(samples)
    res["sample_bounds"] = [0.0] * len(samples)
    si = 0
    while si < len(samples) and samples[si] <= 0.0:       # t_s = 0: the initial state
        res["samples"][si] = w.copy()
        si += 1
    norm1 = one_norm(rowptr, col, val, n)
    r_step = n * norm1 * EPS                       # Eq. 17
    res["roundoff_step"] = r_step
    if t == 0.0:
        res.update(v=w, roundoff_total=0.0)
        return res
    tol_rate = tol / t                             # Eq. 18
    t_now = 0.0
    tau_prev = None

    def matvec(x):
        return spmv(rowptr, col, val, x)

    k = 0
    while t_now < t:
        if k >= max_restarts:
            break
        kr = arnoldi(matvec, w, m, tol_rate, ortho)
        lam, U = small_eig(kr["alpha"], kr["beta"])
        h = kr["h"]
        quad_ok = [True]

        def f(tau):
            return integrand(lam, U, h, tau)

        def integral(a, b):
            if integrator == "gauss":
                v, conv = gauss_legendre(f, a, b)
            else:
                v, conv = tanh_sinh(f, a, b, floor=tol_rate * (b - a))
            if not conv:
                quad_ok[0] = False
            return v

        rem = t - t_now
        if schedule is not None:
            tau = min(float(schedule[k]), rem)
            e = integral(0.0, tau)
        else:
            tau, e = find_step(integral, kr["breakdown"], k == 0, tau_prev, rem, tol_rate, t)
        t_end = t if tau >= rem else t_now + tau
        while si < len(samples) and samples[si] <= t_end:  # sample inside this step
            ds = min(samples[si] - t_now, tau)
            res["samples"][si] = kr["V"] @ omega(lam, U, ds)
            res["sample_bounds"][si] = res["bound"] + integral(0.0, ds)
            si += 1
        om = omega(lam, U, tau)
        w = kr["V"] @ om                           # Eq. 11 / Alg. 1
        t_now = t if tau >= rem else t_now + tau
        tau_prev = tau
        res["bound"] += e
        res["restarts"] += 1
        res["krylov_steps"] += kr["m_eff"]
        res["breakdowns"] += int(kr["breakdown"])
        res["schedule"].append((tau, kr["m_eff"], e))
        if r_step > e:                              # P:334 (per step, C15)
            res["warnings"] |= WARN_ROUNDOFF
        if not quad_ok[0]:
            res["warnings"] |= WARN_QUADRATURE
        k += 1
    res["v"] = w
    res["roundoff_total"] = res["restarts"] * r_step
    return res
