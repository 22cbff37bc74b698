"""Spectrum bounds for the preconditioned solves of SURVEY §8 f2 (input preparation only, like
synth.generator.spectrum_bounds: the interval bounds are INPUTS of lrc_set_preconditioner /
lrc_solve, P:547-569 -- the paper estimates them too; nothing here runs on the solve's data path).

The mean-based preconditioner of P:332-343 is the operator's block at the midpoint of the subset's
parameter range.  For a subset with per-parameter term multipliers E[j, t] (block j = sum_t E[j, t] A_t)
its multipliers are e_mid[t] = (min_j E[j, t] + max_j E[j, t]) / 2.  Two bounds are needed:

* [p_min, p_max] enclosing spec(P_T) (the inner Chebyshev semi-iteration that applies P_T^{-1});
* [lam_min, lam_max] enclosing spec(P_T^{-1} A_j) over the subset (the outer ChebyshevT).

`dense_bounds` computes both exactly (dense symmetric / generalized symmetric eigenvalues; M <= 2000)
and widens them by `margin`; `closed_form_bounds` bounds them for the Kronecker-structured operator of
synth.generator at any size (derivation in its docstring).
"""
from __future__ import annotations

import math
from typing import Tuple

import numpy as np


def legacy_multipliers(rho_f: float, lambda_s: float, d_mu, d_nu):
    """E[j, t] of the six arrays [A0, A1, A2, Jrho, Jmu, Jlam]: (1, mu, rho nu, rho, mu, lam)."""
    d_mu, d_nu = np.asarray(d_mu, np.float64), np.asarray(d_nu, np.float64)
    one = np.ones_like(d_mu)
    return np.stack([one, d_mu, rho_f * d_nu, rho_f * one, d_mu, lambda_s * one], axis=1)


def term_multipliers(coef, diagonals):
    """E[j, t] = sum_g coef[t, g] d_g[j] of a general term list (SURVEY §8 f4 form)."""
    return (np.asarray(coef) @ np.asarray(diagonals)).T


def midpoint(E):
    return 0.5 * (E.min(axis=0) + E.max(axis=0))


def inner_steps(p_min: float, p_max: float, eps: float = 1e-14) -> int:
    """Chebyshev semi-iteration steps q with 2 r^q <= eps, r = (sqrt(k) - 1) / (sqrt(k) + 1)."""
    k = p_max / p_min
    r = (math.sqrt(k) - 1.0) / (math.sqrt(k) + 1.0)
    if r <= 0.0:
        return 1
    return max(1, int(math.ceil(math.log(2.0 / eps) / math.log(1.0 / r))))


def dense_bounds(M, row_ptr, col_idx, vals, E, margin: float = 0.02):
    """Exact bounds (widened by margin) for M <= 2000: eigvalsh(P_T) and the generalized eigenvalues
    of (A_j, P_T) for every parameter j of the subset."""
    import scipy.linalg as sla
    import scipy.sparse as sp

    assert M <= 2000, "dense bounds are for the 16 x 16 grids"

    def dense(mult):
        v = sum(m * a for m, a in zip(mult, vals))
        return sp.csr_matrix((v, col_idx, row_ptr), shape=(M, M)).toarray()

    P = dense(midpoint(E))
    ev = np.linalg.eigvalsh(P)
    p_min, p_max = float(ev[0]), float(ev[-1])
    assert p_min > 0.0, "P_T must be positive definite"
    lo, hi = np.inf, -np.inf
    for mult in E:
        g = sla.eigh(dense(mult), P, eigvals_only=True)
        lo, hi = min(lo, g[0]), max(hi, g[-1])
    return (p_min * (1.0 - margin), p_max * (1.0 + margin), float(lo) * (1.0 - margin), float(hi) * (1.0 + margin))


def closed_form_bounds(g: int, rho_f: float, lambda_s: float, d_mu, d_nu):
    """Bounds for synth.generator's operator A(mu, nu) = K(c(mu, nu)) + J(mu),
    K(c) = L (x) diag(c) + 4 I with field coefficients c = (1 + rho nu, 1 + rho nu, 1, 1 + mu, 1 + mu) and
    J(mu) = rho J_rho + mu J_mu + lam J_lam, ||J(mu)||_2 <= delta(mu) = 1.05 * 0.05 (rho + mu + lam).

    P_T = A(mu_bar, nu_bar).  spec(K(c)) lies in [4 + lmin_L min c, 4 + lmax_L max c] (L SPD), so
    spec(P_T) is in that interval at c_bar, widened by delta(mu_bar) (Weyl).  For the generalized
    problem: K(c) = sum_f c_f (L (x) e_f e_f^T) + 4 I is a sum of PSD forms, so
    x^T K(c) x / x^T K(c_bar) x lies in [r_lo, r_hi] = [min(1, min_f c_f / c_bar_f), max(1, max_f ...)];
    with k = x^T K(c_bar) x / x^T x >= kappa = 4 + lmin_L min c_bar,
    x^T A x / x^T P x >= (r_lo k - delta) / (k + delta_bar) >= (r_lo kappa - delta) / (kappa + delta_bar)
    and <= (r_hi kappa + delta) / (kappa - delta_bar) (both monotone in k)."""
    d_mu, d_nu = np.asarray(d_mu, np.float64), np.asarray(d_nu, np.float64)
    c = math.cos(math.pi / (g + 1))
    lmax_L, lmin_L = 8.0 + 4.0 * c * c, 8.0 - 4.0 * c - 4.0 * c * c

    def coefs(mu, nu):
        return np.array([1.0 + rho_f * nu, 1.0, 1.0 + mu])

    def delta(mu):
        return 1.05 * 0.05 * (rho_f + mu + lambda_s)

    mu_b = 0.5 * (d_mu.min() + d_mu.max())
    nu_b = 0.5 * (d_nu.min() + d_nu.max())
    cb = coefs(mu_b, nu_b)
    db = delta(mu_b)
    kappa = 4.0 + lmin_L * cb.min()
    p_min = kappa - db
    p_max = 4.0 + lmax_L * cb.max() + db
    lo, hi = np.inf, -np.inf
    for mu, nu in zip(d_mu, d_nu):
        r = coefs(mu, nu) / cb
        r_lo, r_hi = min(1.0, r.min()), max(1.0, r.max())
        dj = delta(mu)
        lo = min(lo, (r_lo * kappa - dj) / (kappa + db))
        hi = max(hi, (r_hi * kappa + dj) / (kappa - db))
    assert p_min > 0.0 and lo > 0.0
    return float(p_min), float(p_max), float(lo), float(hi)
