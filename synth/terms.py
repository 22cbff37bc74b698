"""Seeded inputs for the generalized term lists of SURVEY §8 f4 (input construction only; nothing here is
the method's arithmetic -- the oracle builds its own literal term lists from the parameter arrays).

Three operators of the paper on the FE-like grids of synth.generator (same node-block pattern):

* "tiny4" / "small4" -- the four-parameter Newton operator of P:478-482 (`equation_matrix_fourpars1`):
      A0 S + A1 S D_mu- + A2 S D_nurho- + A3 S D_lambda- + Jmu S D_mu + Jlam S D_lambda + Jrho S D_rho,
  D_x- = D_x - x_ref I, parameters (mu_s, nu_f, lambda_s, rho_f) on a little-endian
  m1 x m2 x m3 x m4 grid, D_nurho = diag(nu_f rho_f).  A0 = L(x)I5 + 4I, A1 = L(x)diag(0,0,0,1,1)
  (displacement), A2 = L(x)diag(1,1,0,0,0) (velocity), A3 = L(x)diag(0,0,1,0,0); J* = symmetric N(0,1) on
  the pattern scaled to spectral norm 0.05 (synth.generator's streams).  Reference values x_ref = the
  lower end of each range (so every D_x- >= 0).
* "tinytheta" -- the theta-scheme operator of P:388-396 (`equation_timedep_matrix1`):
      (1/dt) A_t S + theta F(S),  A_t = rho_f A_t^f + rho_s A_t^s  (one assembled mass matrix: identity
  on the node's velocity and displacement fields, 0.5 on the pressure field), F the operator of P:30-36,
  dt = 0.1, theta = 0.5.
* "tinypicard" -- the fixed-point operator of P:647-651 (`equation_picard_matrix1`):
      A0 X + A1 X D_mu- + rho_f A2 X D_nu- + F_mu X D_mu + lambda_s F_lam X + rho_f F_rho X,
  F* drawn like J* (0.05 spectral norm).

For the library each operator is also expressed in its general form (lrc_set_operator_terms):
L(S) = sum_g (sum_t C[t][g] A_t) S diag(d_g), grouping the terms by distinct right diagonal; the group
whose diagonal is the identity carries the Chebyshev step.  tests/test_oracle_pins.py checks that this
form equals the oracle's literal term list.
"""
from __future__ import annotations

import dataclasses
import functools
import math
from typing import List, Tuple

import numpy as np

from synth import generator as gen


@dataclasses.dataclass(frozen=True)
class TermConfig:
    name: str
    kind: str              # "fourparam" | "theta" | "picard"
    g: int
    dims: Tuple[int, ...]  # parameter grid (little endian)
    K: int
    r_B: int
    rank_cap: int
    tol: float
    n_iter: int
    seed: int = 0

    @property
    def M(self) -> int:
        return 5 * self.g * self.g

    @property
    def m(self) -> int:
        return int(np.prod(self.dims))


TERM_CONFIGS = {
    "tiny4": TermConfig("tiny4", "fourparam", 16, (2, 2, 2, 2), 1, 2, 10, 1e-10, 30),
    "small4": TermConfig("small4", "fourparam", 64, (3, 3, 3, 3), 3, 3, 20, 1e-9, 50),
    "tinytheta": TermConfig("tinytheta", "theta", 16, (4, 4), 1, 2, 10, 1e-10, 20),
    "tinypicard": TermConfig("tinypicard", "picard", 16, (4, 4), 1, 2, 10, 1e-10, 30),
}
RANGE = (0.5, 2.0)
THETA, DT, RHO_S = 0.5, 0.1, 1.0


@dataclasses.dataclass
class TermProblem:
    cfg: TermConfig
    M: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: List[np.ndarray]          # the T arrays, in the order of the oracle term list
    rho_f: float
    lambda_s: float
    params: np.ndarray              # m x (#parameters) little-endian grid
    refs: Tuple[float, ...]
    coef: np.ndarray                # T x G  (library general form)
    id_group: int
    subsets: List[Tuple[int, int]]
    lam_min: float
    lam_max: float

    def subset(self, k: int):
        """(params rows of subset k, diagonals G x n for the library, B_U, B_V)."""
        s, e = self.subsets[k]
        P = self.params[s:e]
        n = e - s
        BU = gen.counter_normal(self.cfg.seed, gen.STREAM_BU + 50 + k, np.arange(self.M * self.cfg.r_B, dtype=np.uint64))
        BV = gen.counter_normal(self.cfg.seed, gen.STREAM_BV + 50 + k, np.arange(n * self.cfg.r_B, dtype=np.uint64))
        return P, self.diagonals(P), BU.reshape(self.M, self.cfg.r_B), BV.reshape(n, self.cfg.r_B)

    def diagonals(self, P):
        """Right diagonals of the general form, one row per group (row id_group = ones)."""
        one = np.ones(P.shape[0])
        if self.cfg.kind == "fourparam":       # groups: I, D_mu, D_nurho, D_lambda, D_rho
            mu, nu, lam, rho = P[:, 0], P[:, 1], P[:, 2], P[:, 3]
            return np.stack([one, mu, nu * rho, lam, rho])
        mu, nu = P[:, 0], P[:, 1]              # theta / picard: groups I, D_mu, D_nu
        return np.stack([one, mu, nu])


def _arrays(cfg: TermConfig):
    base = gen.make_operator(gen.Config(cfg.name, cfg.g, 1, 1, RANGE, RANGE, 1, 1, 1, 0.0, 1, seed=cfg.seed))
    rp, ci = base.row_ptr, base.col_idx
    M = base.M
    A0, A1, A2, Jrho, Jmu, Jlam = base.vals
    rows = np.repeat(np.arange(M, dtype=np.int64), np.diff(rp.astype(np.int64)))
    f_row = rows % 5
    lap_f = A0 - 4.0 * (rows == ci)                       # L (x) I5 on the pattern
    A3 = np.where(f_row == 2, lap_f, 0.0)
    diag = (rows == ci).astype(np.float64)
    mass = diag * np.where(f_row == 2, 0.5, 1.0)          # rho_f A_t^f + rho_s A_t^s (rho = 1)
    return base, rp, ci, dict(A0=A0, A1=A1, A2=A2, A3=A3, Jrho=Jrho, Jmu=Jmu, Jlam=Jlam, mass=mass)


def _grid(dims):
    axes = [np.linspace(RANGE[0], RANGE[1], d) for d in dims]
    m = int(np.prod(dims))
    out = np.zeros((m, len(dims)))
    for p in range(m):
        q = p
        for a, d in enumerate(dims):           # little endian: the first index runs fastest
            out[p, a] = axes[a][q % d]
            q //= d
    return out


@functools.lru_cache(maxsize=None)
def make_term_problem(name: str) -> TermProblem:
    cfg = TERM_CONFIGS[name]
    base, rp, ci, A = _arrays(cfg)
    params = _grid(cfg.dims)
    rho_f, lam_s = 1.0, 2.0
    if cfg.kind == "fourparam":
        mu_r, nurho_r, lam_r = RANGE[0], RANGE[0] * RANGE[0], RANGE[0]
        refs = (mu_r, nurho_r, lam_r)
        vals = [A["A0"], A["A1"], A["A2"], A["A3"], A["Jmu"], A["Jlam"], A["Jrho"]]
        # groups I, D_mu, D_nurho, D_lambda, D_rho  (D_x- = D_x - x_ref I folds x_ref into group I)
        coef = np.array([[1, 0, 0, 0, 0], [-mu_r, 1, 0, 0, 0], [-nurho_r, 0, 1, 0, 0], [-lam_r, 0, 0, 1, 0],
                         [0, 1, 0, 0, 0], [0, 0, 0, 1, 0], [0, 0, 0, 0, 1]], dtype=np.float64)
    elif cfg.kind == "theta":
        refs = ()
        vals = [A["mass"], A["A0"], A["A1"], A["A2"], A["Jrho"], A["Jmu"], A["Jlam"]]
        th = THETA
        coef = np.array([[1.0 / DT, 0, 0], [th, 0, 0], [0, th, 0], [0, 0, th * rho_f], [th * rho_f, 0, 0],
                         [0, th, 0], [th * lam_s, 0, 0]], dtype=np.float64)
    else:
        mu_r, nu_r = RANGE[0], RANGE[0]
        refs = (mu_r, nu_r)
        vals = [A["A0"], A["A1"], A["A2"], A["Jmu"], A["Jlam"], A["Jrho"]]      # F_mu, F_lam, F_rho
        coef = np.array([[1, 0, 0], [-mu_r, 1, 0], [-rho_f * nu_r, 0, rho_f], [0, 1, 0], [lam_s, 0, 0],
                         [rho_f, 0, 0]], dtype=np.float64)
    subsets = gen.split_subsets(cfg.m, cfg.K)
    prob = TermProblem(cfg, base.M, rp, ci, vals, rho_f, lam_s, params, refs, coef, 0, subsets, 0.0, 0.0)
    prob.lam_min, prob.lam_max = spectrum_bounds(prob)
    return prob


def _block_values(prob: TermProblem, P_row):
    d = prob.diagonals(P_row[None, :])[:, 0]          # the G diagonal values of this parameter
    e = prob.coef @ d                                  # per-array multiplier
    return sum(e[t] * v for t, v in enumerate(prob.vals))


def spectrum_bounds(prob: TermProblem, margin: float = 0.02):
    """Interval enclosing the spectra of all blocks: exact dense eigenvalues of every block
    for the 16 x 16 grids, else the closed form of synth.generator plus Weyl's inequality."""
    import scipy.sparse as sp
    if prob.M <= 2000:
        lo, hi = np.inf, -np.inf
        for P_row in prob.params:
            Ab = sp.csr_matrix((_block_values(prob, P_row), prob.col_idx, prob.row_ptr), shape=(prob.M, prob.M))
            ev = np.linalg.eigvalsh(Ab.toarray())
            lo, hi = min(lo, ev[0]), max(hi, ev[-1])
        return float(lo) * (1.0 - margin), float(hi) * (1.0 + margin)
    # four-parameter operator: A = L(x)diag(c_f) + 4I + (mu Jmu + lam Jlam + rho Jrho), c_f >= 1
    g = prob.cfg.g
    c = math.cos(math.pi / (g + 1))
    lmax_L, lmin_L = 8.0 + 4.0 * c * c, 8.0 - 4.0 * c - 4.0 * c * c
    P = prob.params
    mu_r, nurho_r, lam_r = prob.refs
    cf = np.stack([1 + P[:, 1] * P[:, 3] - nurho_r, 1 + P[:, 2] - lam_r, 1 + P[:, 0] - mu_r])
    delta = 1.05 * 0.05 * float(np.max(P[:, 0] + P[:, 2] + P[:, 3]))
    return 4.0 + lmin_L * float(cf.min()) - delta, 4.0 + lmax_L * float(cf.max()) + delta
