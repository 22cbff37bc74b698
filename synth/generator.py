"""Deterministic generator for the five BASELINE.json configs.

Recipe (a reading; BASELINE.json fixes the shapes, the paper fixes none of the values):

* 2D g x g node grid, node = iy*g + ix, 5 fields per node (ux, uy, p, dx, dy) so
  M = 5 g^2 (the paper's d = 2 count M = 5N).  DOF = 5*node + f.
* One shared CSR pattern: every row of node n couples to all 5 fields of every
  existing node in the 3x3 neighbourhood of n (Dirichlet truncation).  Columns
  sorted ascending; the 5 rows of a node share one column list.
* L = 9-point graph Laplacian on the nodes: 8 on the diagonal, -1 per existing
  neighbour (integer valued, SPD, spectrum in (0, 12)).
* A0 = L (x) I5 + 4 I, A1 = L (x) diag(0,0,0,1,1), A2 = L (x) diag(1,1,0,0,0),
  stored on the shared pattern with explicit zeros.
* J_rho, J_mu, J_lambda = 0.05 * Jt / est||Jt||_2 with Jt symmetric, Jt_ij ~ N(0,1)
  i.i.d. for i <= j on the pattern (mirrored).  est||.||_2 = fixed-step power
  iteration (nominal norm 0.05; the arrays are shared by both sides so the exact
  value is immaterial).
* rho_f = 1, lambda_s = 2.
* Parameter grid: mu = linspace(lo, hi, m1), nu = linspace(lo, hi, m2), little
  endian order (mu fastest); K contiguous subsets sized by P:157-160.
* B^k = B_U^k B_V^k^T with N(0,1) factors (M x r_B, n x r_B), one stream per subset.
* Random numbers: a counter-based generator (splitmix64 of (seed, stream, index),
  Box-Muller) so that every value is a pure function of its counter.
* Spectrum bounds [lam_min, lam_max] of the block-diagonal Kronecker operator,
  union over all parameters: Tiny -- exact dense eigenvalues of all
  blocks widened by 2%; larger configs -- closed-form spectrum of the J-free part
  plus Weyl's inequality for the J terms (see spectrum_bounds).

Nothing here is the method's arithmetic; this is input construction only.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Tuple

import numpy as np

_U64 = np.uint64
_GOLDEN = _U64(0x9E3779B97F4A7C15)
_M1 = _U64(0xBF58476D1CE4E5B9)
_M2 = _U64(0x94D049BB133111EB)

# random streams (counter-based: stream id selects an independent sequence)
STREAM_J = {"rho": 1, "mu": 2, "lambda": 3}
STREAM_BU = 100  # + k
STREAM_BV = 200  # + k
STREAM_DENSE_S = 300
STREAM_POWER = 400


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + _GOLDEN
        z = (z ^ (z >> _U64(30))) * _M1
        z = (z ^ (z >> _U64(27))) * _M2
        return z ^ (z >> _U64(31))


def _stream_key(seed: int, stream: int) -> np.uint64:
    a = _splitmix64(np.array([seed], dtype=np.uint64))
    with np.errstate(over="ignore"):
        b = _splitmix64(a ^ _splitmix64(np.array([stream], dtype=np.uint64)))
    return b[0]


def counter_normal(seed: int, stream: int, index: np.ndarray, chunk: int = 1 << 22) -> np.ndarray:
    """N(0,1) sample for each uint64 counter in `index` (pure function of (seed, stream, index))."""
    index = np.asarray(index, dtype=np.uint64).ravel()
    key = _stream_key(seed, stream)
    out = np.empty(index.shape[0], dtype=np.float64)
    two = _U64(2)
    for s in range(0, index.shape[0], chunk):
        idx = index[s:s + chunk]
        with np.errstate(over="ignore"):
            h1 = _splitmix64((idx * two) ^ key)
            h2 = _splitmix64((idx * two + _U64(1)) ^ key)
        u1 = ((h1 >> _U64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)
        u2 = (h2 >> _U64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
        out[s:s + chunk] = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
    return out


# ----------------------------------------------------------------------------------------------
# configs (BASELINE.json configs[0..4]; missing details are DESIGN.md readings)
# ----------------------------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    g: int                 # node grid g x g, M = 5 g^2
    m1: int                # number of shear moduli mu_s
    m2: int                # number of fluid viscosities nu_f
    mu_range: Tuple[float, float]
    nu_range: Tuple[float, float]
    K: int                 # subsets
    r_B: int               # rank of B
    rank_cap: int          # R
    tol: float             # truncation tolerance tau
    n_iter: int            # Chebyshev iterations N
    dense_cols: int = 0    # config 5: dense S columns
    reps: int = 0          # config 5: repetitions
    seed: int = 0

    @property
    def M(self) -> int:
        return 5 * self.g * self.g

    @property
    def m(self) -> int:
        return self.m1 * self.m2


CONFIGS: Dict[str, Config] = {
    "tiny": Config("tiny", 16, 4, 4, (0.5, 2.0), (0.5, 2.0), 1, 2, 10, 1e-10, 30),
    "small": Config("small", 64, 10, 10, (0.5, 2.0), (0.5, 2.0), 4, 3, 20, 1e-9, 50),
    "medium": Config("medium", 256, 20, 20, (0.5, 2.0), (0.5, 2.0), 8, 4, 40, 1e-8, 80),
    "large": Config("large", 512, 40, 25, (0.25, 4.0), (0.25, 4.0), 10, 5, 60, 1e-8, 100),
    "fullrank": Config("fullrank", 512, 16, 16, (0.25, 4.0), (0.25, 4.0), 1, 0, 0, 0.0, 0,
                       dense_cols=256, reps=20),
}


def config_by_name(name: str) -> Config:
    return CONFIGS[name.lower()]


# ----------------------------------------------------------------------------------------------
# operator
# ----------------------------------------------------------------------------------------------
@dataclasses.dataclass
class Operator:
    M: int
    row_ptr: np.ndarray            # int32[M+1]
    col_idx: np.ndarray            # int32[nnz]
    vals: List[np.ndarray]         # six fp64[nnz]: A0, A1, A2, J_rho, J_mu, J_lambda
    rho_f: float
    lambda_s: float
    g: int = 0

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])


def _pattern(g: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    """Shared node-block pattern. Returns row_ptr, col_idx, row_node, col_node (per nnz)."""
    nn = g * g
    iy, ix = np.divmod(np.arange(nn, dtype=np.int64), g)
    nbr = np.full((nn, 9), -1, dtype=np.int64)
    k = 0
    for dy in (-1, 0, 1):          # neighbour nodes in increasing node order
        for dx in (-1, 0, 1):
            jy, jx = iy + dy, ix + dx
            ok = (jy >= 0) & (jy < g) & (jx >= 0) & (jx < g)
            nbr[:, k] = np.where(ok, jy * g + jx, -1)
            k += 1
    cnt = (nbr >= 0).sum(axis=1)                  # neighbours per node
    row_len = np.repeat(5 * cnt, 5)               # per DOF row
    M = 5 * nn
    row_ptr = np.zeros(M + 1, dtype=np.int64)
    np.cumsum(row_len, out=row_ptr[1:])
    # per node: sorted valid neighbours, each expanded to 5 field columns
    valid = nbr >= 0
    nb_sorted = np.where(valid, nbr, np.iinfo(np.int64).max)
    nb_sorted.sort(axis=1)
    # node column list (variable length) -> flatten by mask
    cols_node = (nb_sorted[:, :, None] * 5 + np.arange(5)[None, None, :])   # (nn, 9, 5)
    mask_node = np.repeat((nb_sorted < np.iinfo(np.int64).max)[:, :, None], 5, axis=2)
    # each of the 5 rows of a node repeats the node's column list
    cols = np.broadcast_to(cols_node[:, None, :, :], (nn, 5, 9, 5))
    mask = np.broadcast_to(mask_node[:, None, :, :], (nn, 5, 9, 5))
    col_idx = cols[mask]
    nb_node = np.broadcast_to(nb_sorted[:, None, :, None], (nn, 5, 9, 5))[mask]
    row_node = np.broadcast_to(np.arange(nn)[:, None, None, None], (nn, 5, 9, 5))[mask]
    assert col_idx.shape[0] == row_ptr[-1]
    return row_ptr.astype(np.int32), col_idx.astype(np.int32), row_node, nb_node


def _power_norm(row_ptr, col_idx, vals, M, seed, steps=40) -> float:
    import scipy.sparse as sp
    A = sp.csr_matrix((vals, col_idx, row_ptr), shape=(M, M))
    x = counter_normal(seed, STREAM_POWER, np.arange(M, dtype=np.uint64))
    x /= np.linalg.norm(x)
    lam = 0.0
    for _ in range(steps):
        y = A @ x
        lam = float(np.linalg.norm(y))
        if lam == 0.0:
            return 0.0
        x = y / lam
    return lam


def make_operator(cfg: Config, j_norm_steps: int = 40) -> Operator:
    g = cfg.g
    M = cfg.M
    row_ptr, col_idx, row_node, col_node = _pattern(g)
    nnz = col_idx.shape[0]
    rows = np.repeat(np.arange(M, dtype=np.int64), np.diff(row_ptr.astype(np.int64)))
    f_row = rows % 5
    f_col = col_idx.astype(np.int64) % 5
    same_field = f_row == f_col
    lap = np.where(row_node == col_node, 8.0, -1.0)
    lap_f = np.where(same_field, lap, 0.0)
    diag = rows == col_idx
    A0 = lap_f + 4.0 * diag
    A1 = np.where(f_row >= 3, lap_f, 0.0)
    A2 = np.where(f_row <= 1, lap_f, 0.0)
    del lap, lap_f
    lo = np.minimum(rows, col_idx.astype(np.int64)).astype(np.uint64)
    hi = np.maximum(rows, col_idx.astype(np.int64)).astype(np.uint64)
    pair = lo * np.uint64(M) + hi
    del lo, hi, rows
    Js = []
    for name in ("rho", "mu", "lambda"):
        Jt = counter_normal(cfg.seed, STREAM_J[name], pair)
        nrm = _power_norm(row_ptr, col_idx, Jt, M, cfg.seed, steps=j_norm_steps)
        Js.append(Jt * (0.05 / nrm))
    vals = [A0, A1, A2, Js[0], Js[1], Js[2]]
    assert all(v.shape[0] == nnz for v in vals)
    return Operator(M=M, row_ptr=row_ptr, col_idx=col_idx, vals=vals, rho_f=1.0, lambda_s=2.0, g=g)


# ----------------------------------------------------------------------------------------------
# parameter grid and subsets
# ----------------------------------------------------------------------------------------------
def parameter_grid(cfg: Config) -> Tuple[np.ndarray, np.ndarray]:
    """Little-endian ordered (mu, nu) arrays of length m: column p <-> (mu^{(p mod m1)}, nu^{floor(p/m1)})."""
    mu = np.linspace(cfg.mu_range[0], cfg.mu_range[1], cfg.m1)
    nu = np.linspace(cfg.nu_range[0], cfg.nu_range[1], cfg.m2)
    p = np.arange(cfg.m)
    return mu[p % cfg.m1], nu[p // cfg.m1]


def split_subsets(m: int, K: int) -> List[Tuple[int, int]]:
    """Contiguous subsets sized by P:157-160: floor(m/K) for k < K, the rest for the last. Returns [start, stop)."""
    base = m // K
    out = []
    start = 0
    for k in range(K):
        size = base if k < K - 1 else m - (K - 1) * base
        out.append((start, start + size))
        start += size
    return out


def upper_median_index(start: int, stop: int, m1: int) -> Tuple[int, int]:
    """Upper median of the little-endian ordered subset, as a 1-based multi-index (i1, i2)."""
    size = stop - start
    p = start + size // 2          # 0-based ordinal of the upper median
    return (p % m1) + 1, (p // m1) + 1


# ----------------------------------------------------------------------------------------------
# right-hand sides and dense S
# ----------------------------------------------------------------------------------------------
def rhs_factors(cfg: Config, k: int, M: int, n: int) -> Tuple[np.ndarray, np.ndarray]:
    """B^k = B_U B_V^T, N(0,1) factors; B_U is M x r_B, B_V is n x r_B (row-major)."""
    r = cfg.r_B
    BU = counter_normal(cfg.seed, STREAM_BU + k, np.arange(M * r, dtype=np.uint64)).reshape(M, r)
    BV = counter_normal(cfg.seed, STREAM_BV + k, np.arange(n * r, dtype=np.uint64)).reshape(n, r)
    return BU, BV


def dense_factor(cfg: Config, M: int, ncols: int, rows: Optional[np.ndarray] = None) -> np.ndarray:
    """Config 5's dense S (M x ncols, N(0,1)); `rows` selects a subset of rows (same values)."""
    if rows is None:
        idx = np.arange(M * ncols, dtype=np.uint64)
        return counter_normal(cfg.seed, STREAM_DENSE_S, idx).reshape(M, ncols)
    rows = np.asarray(rows, dtype=np.uint64)
    idx = (rows[:, None] * np.uint64(ncols) + np.arange(ncols, dtype=np.uint64)[None, :]).ravel()
    return counter_normal(cfg.seed, STREAM_DENSE_S, idx).reshape(rows.shape[0], ncols)


# ----------------------------------------------------------------------------------------------
# spectrum bounds (the paper's "Est." harness step)
# ----------------------------------------------------------------------------------------------
def _block_csr(op: Operator, mu: float, nu: float):
    import scipy.sparse as sp
    v = op.vals
    vals = v[0] + mu * (v[1] + v[4]) + op.rho_f * nu * v[2] + op.rho_f * v[3] + op.lambda_s * v[5]
    return sp.csr_matrix((vals, op.col_idx, op.row_ptr), shape=(op.M, op.M))


def spectrum_bounds(op: Operator, cfg: Config, margin: float = 0.02) -> Tuple[float, float]:
    """Interval [lam_min, lam_max] enclosing the spectra of all blocks A(mu_j, nu_j).

    M <= 2000 (Tiny): exact dense eigenvalues of every block, widened by `margin`.
    Larger configs: the generator's structure gives the bound in closed form.  Each block is
    A(mu, nu) = L (x) diag(1+rho nu, 1+rho nu, 1, 1+mu, 1+mu) + 4 I + (rho J_rho + mu J_mu + lam J_lam),
    L = 9 I - (I+T) (x) (I+T) with T the path adjacency, so spec(L) = {9 - (1+2cos a)(1+2cos b)},
    a, b in {k pi/(g+1)}: lam_max(L) = 8 + 4 c^2, lam_min(L) = 8 - 4c - 4c^2, c = cos(pi/(g+1)).
    Weyl's inequality adds +-delta, delta = 1.05 * 0.05 * (rho + mu_max + lam) (1.05 covers the
    power-iteration under-estimate of ||J~||_2 used to scale J to nominal norm 0.05).
    """
    mu, nu = parameter_grid(cfg)
    if op.M <= 2000:
        lo, hi = np.inf, -np.inf
        for mu_j, nu_j in zip(mu, nu):
            ev = np.linalg.eigvalsh(_block_csr(op, mu_j, nu_j).toarray())
            lo, hi = min(lo, ev[0]), max(hi, ev[-1])
        return float(lo) * (1.0 - margin), float(hi) * (1.0 + margin)
    c = math.cos(math.pi / (cfg.g + 1))
    lmax_L = 8.0 + 4.0 * c * c
    lmin_L = 8.0 - 4.0 * c - 4.0 * c * c
    delta = 1.05 * 0.05 * (op.rho_f + float(mu.max()) + op.lambda_s)
    coef_max = 1.0 + max(float(mu.max()), op.rho_f * float(nu.max()), 0.0)
    coef_min = 1.0 + min(float(mu.min()), op.rho_f * float(nu.min()), 0.0)
    return 4.0 + lmin_L * coef_min - delta, 4.0 + lmax_L * coef_max + delta


# ----------------------------------------------------------------------------------------------
# a whole problem instance
# ----------------------------------------------------------------------------------------------
@dataclasses.dataclass
class Problem:
    cfg: Config
    op: Operator
    mu: np.ndarray
    nu: np.ndarray
    subsets: List[Tuple[int, int]]
    lam_min: float
    lam_max: float

    def subset(self, k: int):
        """(d_mu, d_nu, B_U, B_V) of subset k."""
        s, e = self.subsets[k]
        n = e - s
        BU, BV = rhs_factors(self.cfg, k, self.op.M, n)
        return self.mu[s:e].copy(), self.nu[s:e].copy(), BU, BV


def make_problem(name: str) -> Problem:
    cfg = config_by_name(name)
    op = make_operator(cfg)
    mu, nu = parameter_grid(cfg)
    subsets = split_subsets(cfg.m, cfg.K)
    b = spectrum_bounds(op, cfg)
    return Problem(cfg, op, mu, nu, subsets, b[0], b[1])
