"""Pins of the CPU oracle against things other than itself (SURVEY.md §8(c) pins P1-P9).

Each test cites what fixes the expected value: a closed form, a textbook/library routine,
brute force, or a number printed in the paper.  No expected value comes from the CUDA path.
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from numpy.polynomial import chebyshev as npcheb

from oracle import chebyshevt as orc
from synth import generator as gen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------------------------------
# helpers (input construction only)
# ------------------------------------------------------------------------------------------
def diagonal_problem(M=40, n=6, rB=2, seed=5, lo=1.0):
    rng = np.random.default_rng(seed)
    a = [lo + rng.random(M) * 3.0] + [rng.random(M) for _ in range(5)]
    mats = [sp.diags(x).tocsr() for x in a]
    d_mu = 0.5 + rng.random(n) * 1.5
    d_nu = 0.5 + rng.random(n) * 1.5
    rho, lam = 1.0, 2.0
    terms = orc.term_list(mats, rho, lam, d_mu, d_nu)
    # eigenvalue lambda_ij of the diagonal operator, written out from P:30-36 entry by entry
    Lam = (a[0][:, None] + d_mu[None, :] * a[1][:, None] + rho * d_nu[None, :] * a[2][:, None]
           + rho * a[3][:, None] + d_mu[None, :] * a[4][:, None] + lam * a[5][:, None])
    BU = rng.standard_normal((M, rB))
    BV = rng.standard_normal((n, rB))
    return terms, Lam, BU, BV


def cheb_T(k, x):
    """T_k(x) via numpy's Chebyshev-series evaluation (library routine)."""
    coef = np.zeros(k + 1)
    coef[k] = 1.0
    return npcheb.chebval(x, coef)


@pytest.fixture(scope="module")
def tiny():
    prob = gen.make_problem("tiny")
    d_mu, d_nu, BU, BV = prob.subset(0)
    mats = orc.csr_matrices(prob.op.M, prob.op.row_ptr, prob.op.col_idx, prob.op.vals)
    terms = orc.term_list(mats, prob.op.rho_f, prob.op.lambda_s, d_mu, d_nu)
    return prob, terms, BU, BV


def block_solve(terms, B):
    """Exact S* by per-column sparse solves of the block-diagonal system."""
    M, n = B.shape
    S = np.zeros_like(B)
    for j in range(n):
        Aj = None
        for c, A, e in terms:
            Aj = c * e[j] * A if Aj is None else Aj + c * e[j] * A
        S[:, j] = spla.spsolve(Aj.tocsc(), B[:, j])
    return S


# ------------------------------------------------------------------------------------------
# P1: exact Chebyshev error polynomial on diagonal operators
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("N", [1, 2, 5, 12])
def test_P1_diagonal_closed_form(N):
    terms, Lam, BU, BV = diagonal_problem()
    lmin, lmax = Lam.min(), Lam.max()
    res = orc.chebyshevt(terms, BU, BV, lmin, lmax, tau=0.0, R=BV.shape[0], N=N)
    X = orc.dense_product(res.U, res.V)
    B = BU @ BV.T
    S_star = B / Lam
    c, d = 0.5 * (lmax - lmin), 0.5 * (lmax + lmin)
    pN = cheb_T(N, (d - Lam) / c) / cheb_T(N, d / c)       # error polynomial
    X_exact = (1.0 - pN) * S_star
    assert np.linalg.norm(X - X_exact) <= 1e-13 * np.linalg.norm(X_exact)


def test_P1_richardson_c0_closed_form():
    """c = 0 (lam_min = lam_max = d): Richardson with gamma = 1/d, error (1 - lambda/d)^N."""
    terms, Lam, BU, BV = diagonal_problem(lo=3.0)
    d = float(Lam.max())
    N = 7
    res = orc.chebyshevt(terms, BU, BV, d, d, tau=0.0, R=BV.shape[0], N=N)
    S_star = (BU @ BV.T) / Lam
    X_exact = (1.0 - (1.0 - Lam / d) ** N) * S_star
    X = orc.dense_product(res.U, res.V)
    assert np.linalg.norm(X - X_exact) <= 1e-13 * np.linalg.norm(X_exact)


# ------------------------------------------------------------------------------------------
# P2 / P4: Chebyshev bound and dense Kronecker solve on Tiny
# ------------------------------------------------------------------------------------------
def test_P4_kronecker_solution_matches_column_solves(tiny):
    prob, terms, BU, BV = tiny
    B = BU @ BV.T
    K = orc.kron_operator(terms)
    s = spla.spsolve(K.tocsc(), orc.vec(B))
    S_kron = orc.unvec(s, prob.op.M)
    S_cols = block_solve(terms, B)
    assert np.linalg.norm(S_kron - S_cols) <= 1e-12 * np.linalg.norm(S_cols)


def test_P2_chebyshev_bound_untruncated(tiny):
    prob, terms, BU, BV = tiny
    n = BV.shape[0]
    N = 30
    res = orc.chebyshevt(terms, BU, BV, prob.lam_min, prob.lam_max, tau=0.0, R=n, N=N)
    S_star = block_solve(terms, BU @ BV.T)
    c, d = 0.5 * (prob.lam_max - prob.lam_min), 0.5 * (prob.lam_max + prob.lam_min)
    bound = np.linalg.norm(S_star) / cheb_T(N, d / c)
    err = np.linalg.norm(orc.dense_product(res.U, res.V) - S_star)
    assert err <= bound * (1 + 1e-6) + 1e-13 * np.linalg.norm(S_star)
    assert err >= 1e-3 * bound   # it really is a Chebyshev rate, not an exact solve


def test_P4_converged_solution_untruncated(tiny):
    prob, terms, BU, BV = tiny
    n = BV.shape[0]
    N = 70
    res = orc.chebyshevt(terms, BU, BV, prob.lam_min, prob.lam_max, tau=1e-15, R=n, N=N,
                         record_iterates=False)
    S_star = block_solve(terms, BU @ BV.T)
    err = np.linalg.norm(orc.dense_product(res.U, res.V) - S_star) / np.linalg.norm(S_star)
    assert err <= 1e-11
    assert res.rel_residual <= 1e-11


def test_P4_truncated_solution_near_best_rank(tiny):
    """BJ's Tiny settings (R = 10, tau = 1e-10, N = 30): error close to the best rank-10 error of S*."""
    prob, terms, BU, BV = tiny
    cfg = prob.cfg
    res = orc.chebyshevt(terms, BU, BV, prob.lam_min, prob.lam_max, tau=cfg.tol, R=cfg.rank_cap,
                         N=cfg.n_iter, record_iterates=False)
    S_star = block_solve(terms, BU @ BV.T)
    s = np.linalg.svd(S_star, compute_uv=False)
    best = np.sqrt(np.sum(s[cfg.rank_cap:] ** 2))
    err = np.linalg.norm(orc.dense_product(res.U, res.V) - S_star)
    assert best <= err <= 1.5 * best
    assert res.U.shape[1] == cfg.rank_cap


# ------------------------------------------------------------------------------------------
# P3: identity operator, c = 0, d = 1
# ------------------------------------------------------------------------------------------
def test_P3_identity_operator_one_step():
    M, n = 30, 5
    rng = np.random.default_rng(3)
    I = sp.identity(M, format="csr")
    Z = sp.csr_matrix((M, M))
    terms = orc.term_list([I, Z, Z, Z, Z, Z], 1.0, 2.0, rng.random(n), rng.random(n))
    BU, BV = rng.standard_normal((M, 2)), rng.standard_normal((n, 2))
    res = orc.chebyshevt(terms, BU, BV, 1.0, 1.0, tau=0.0, R=n, N=4)
    B = BU @ BV.T
    for U, V in res.iterates:
        assert np.linalg.norm(U @ V.T - B) <= 1e-14 * np.linalg.norm(B)
    assert res.rel_residual <= 1e-14


# ------------------------------------------------------------------------------------------
# P5: truncation vs brute-force dense SVD
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("R,tau", [(1, 0.0), (3, 0.0), (5, 1e-3), (12, 1e-10), (20, 0.0)])
def test_P5_truncation_is_best_rank_approx(R, tau):
    rng = np.random.default_rng(11)
    M, n, w = 200, 30, 12
    U = rng.standard_normal((M, w)) * np.logspace(0, -6, w)[None, :]
    V = rng.standard_normal((n, w))
    X = U @ V.T
    Ut, Vt, s = orc.truncate(U, V, tau, R)
    Pd, sd, Qd = np.linalg.svd(X, full_matrices=False)       # brute force on the dense product
    r = min(R, w, int(np.sum(sd > tau * sd[0])))   # rank(X) <= w
    assert Ut.shape[1] == r
    Xr = (Pd[:, :r] * sd[:r]) @ Qd[:r]
    assert np.linalg.norm(Ut @ Vt.T - Xr) <= 1e-12 * np.linalg.norm(X)
    assert np.allclose(s[:min(w, n)], sd[:min(w, n)], rtol=0, atol=1e-12 * sd[0])
    # error equals the tail singular-value norm
    assert abs(np.linalg.norm(X - Ut @ Vt.T) - np.sqrt(np.sum(sd[r:] ** 2))) <= 1e-11 * sd[0]
    # U' has orthonormal columns (reading S12)
    assert np.linalg.norm(Ut.T @ Ut - np.eye(r)) <= 1e-13


def test_P5_truncation_edge_cases():
    rng = np.random.default_rng(2)
    M, n = 50, 8
    # zero factor -> rank 0
    Ut, Vt, _ = orc.truncate(np.zeros((M, 3)), rng.standard_normal((n, 3)), 0.0, 5)
    assert Ut.shape == (M, 0) and Vt.shape == (n, 0)
    # empty factor
    Ut, Vt, s = orc.truncate(np.zeros((M, 0)), np.zeros((n, 0)), 0.0, 5)
    assert Ut.shape[1] == 0 and s.size == 0
    # rank-1 is kept exactly
    a, b = rng.standard_normal((M, 1)), rng.standard_normal((n, 1))
    Ut, Vt, _ = orc.truncate(a, b, 1e-12, 1)
    assert np.linalg.norm(Ut @ Vt.T - a @ b.T) <= 1e-14 * np.linalg.norm(a @ b.T)
    # exactly rank-deficient concatenation (duplicated column blocks, the k = 2 situation)
    U = rng.standard_normal((M, 4))
    Ud = np.hstack([U, U, U[:, :2]])
    Vd = rng.standard_normal((n, 10))
    Ut, Vt, s = orc.truncate(Ud, Vd, 1e-12, 10)
    assert Ut.shape[1] == 4
    assert np.linalg.norm(Ut @ Vt.T - Ud @ Vd.T) <= 1e-13 * np.linalg.norm(Ud @ Vd.T)


# ------------------------------------------------------------------------------------------
# P6: operator -- factored vs Kronecker vector notation vs dense
# ------------------------------------------------------------------------------------------
def test_P6_operator_factored_vs_kronecker(tiny):
    prob, terms, BU, BV = tiny
    rng = np.random.default_rng(7)
    U, V = rng.standard_normal((prob.op.M, 4)), rng.standard_normal((BV.shape[0], 4))
    UL, VL = orc.apply_lowrank(terms, U, V)
    K = orc.kron_operator(terms)
    LX_kron = orc.unvec(K @ orc.vec(U @ V.T), prob.op.M)
    LX_dense = orc.apply_dense(terms, U @ V.T)
    ref = np.linalg.norm(LX_kron)
    assert np.linalg.norm(UL @ VL.T - LX_kron) <= 1e-13 * ref
    assert np.linalg.norm(LX_dense - LX_kron) <= 1e-13 * ref


def test_P6_kronecker_is_block_diagonal(tiny):
    """vec(L(S)) = diago(A(mu_j, nu_j)) vec(S) with A(mu,nu) = A0 + mu A1 + rho nu A2 + rho Jr + mu Jm + lam Jl."""
    prob, terms, BU, BV = tiny
    op = prob.op
    d_mu, d_nu = prob.mu, prob.nu
    mats = orc.csr_matrices(op.M, op.row_ptr, op.col_idx, op.vals)
    blocks = [mats[0] + m * mats[1] + op.rho_f * v * mats[2] + op.rho_f * mats[3] + m * mats[4]
              + op.lambda_s * mats[5] for m, v in zip(d_mu, d_nu)]
    K_blocks = sp.block_diag(blocks, format="csr")
    K = orc.kron_operator(terms)
    assert abs(K - K_blocks).max() <= 1e-14 * abs(K).max()


def test_vec_roundtrip():
    S = np.arange(12.0).reshape(4, 3)
    v = orc.vec(S)
    assert np.array_equal(v[:4], S[:, 0])            # column stacking
    assert np.array_equal(orc.unvec(v, 4), S)


# ------------------------------------------------------------------------------------------
# P7: omega recursion vs closed form 2 sigma T_k(sigma) / T_{k+1}(sigma)
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("lmin,lmax", [(4.0, 40.0), (0.9, 1.1), (1.0, 100.0)])
def test_P7_omega_closed_form(lmin, lmax):
    N = 40
    w = orc.omegas(lmin, lmax, N)
    c, d = 0.5 * (lmax - lmin), 0.5 * (lmax + lmin)
    sig = d / c
    assert w[0] == 1.0
    for k in range(1, N):
        closed = 2.0 * sig * cheb_T(k, sig) / cheb_T(k + 1, sig)
        assert abs(w[k] - closed) <= 1e-13 * closed
    # monotone decreasing from w_2 towards the limit 2 / (1 + sqrt(1 - c^2/d^2))
    assert np.all(np.diff(w[1:]) <= 0) and w[-1] >= 2.0 / (1.0 + np.sqrt(1.0 - (c / d) ** 2)) - 1e-14


def test_P7_omega_c0_is_one():
    assert np.all(orc.omegas(2.0, 2.0, 10) == 1.0)


# ------------------------------------------------------------------------------------------
# P8: structural rank bounds
# ------------------------------------------------------------------------------------------
def test_P8_rank_structure(tiny):
    prob, terms, BU, BV = tiny
    rng = np.random.default_rng(9)
    r = 3
    U, V = rng.standard_normal((prob.op.M, r)), rng.standard_normal((BV.shape[0], r))
    UL, VL = orc.apply_lowrank(terms, U, V)
    s = np.linalg.svd(UL @ VL.T, compute_uv=False)
    # rank(L(X)) <= 3 rank(X): the six terms have only three distinct right diagonals
    assert s[3 * r] <= 1e-12 * s[0]
    cfg = prob.cfg
    res = orc.chebyshevt(terms, BU, BV, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, 8)
    rB = BU.shape[1]
    prev = 0
    for rk in res.ranks:
        assert rk <= min(cfg.rank_cap, BV.shape[0], rB + 4 * prev)
        prev = rk
    assert res.ranks[0] == rB


# ------------------------------------------------------------------------------------------
# P9: asymptotic contraction on a spectrum in [0.9, 1.1]
# ------------------------------------------------------------------------------------------
def test_P9_contraction_rate():
    M, n = 60, 4
    rng = np.random.default_rng(4)
    lam = np.linspace(0.9, 1.1, M)
    Z = sp.csr_matrix((M, M))
    terms = orc.term_list([sp.diags(lam).tocsr(), Z, Z, Z, Z, Z], 1.0, 2.0, np.ones(n), np.ones(n))
    BU, BV = rng.standard_normal((M, 2)), rng.standard_normal((n, 2))
    S_star = (BU @ BV.T) / lam[:, None]
    errs = []
    for N in (4, 8):
        res = orc.chebyshevt(terms, BU, BV, 0.9, 1.1, tau=0.0, R=n, N=N)
        errs.append(np.linalg.norm(res.U @ res.V.T - S_star))
    rate = (errs[1] / errs[0]) ** (1.0 / 4.0)
    expected = 0.1 / (1.0 + np.sqrt(1.0 - 0.01))              # c / (d + sqrt(d^2 - c^2)) = 0.0501
    assert abs(expected - 0.0501) < 1e-4
    assert rate <= expected * 1.05


# ------------------------------------------------------------------------------------------
# residual vs brute force
# ------------------------------------------------------------------------------------------
def test_residual_vs_dense(tiny):
    prob, terms, BU, BV = tiny
    rng = np.random.default_rng(8)
    U, V = rng.standard_normal((prob.op.M, 5)) * 1e-2, rng.standard_normal((BV.shape[0], 5))
    B = BU @ BV.T
    K = orc.kron_operator(terms)
    Rd = B - orc.unvec(K @ orc.vec(U @ V.T), prob.op.M)
    assert abs(orc.residual(terms, BU, BV, U, V) - np.linalg.norm(Rd) / np.linalg.norm(B)) <= 1e-13
    assert orc.residual(terms, BU, BV, np.zeros((prob.op.M, 0)), np.zeros((BV.shape[0], 0))) == 1.0
    assert orc.residual(terms, np.zeros((prob.op.M, 0)), np.zeros((BV.shape[0], 0)), U, V) == 0.0


def test_restart_resets_omega(tiny):
    """Reading S8: after a restart the recurrence starts again with w_1 = 1 (one Richardson step)."""
    prob, terms, BU, BV = tiny
    res = orc.chebyshevt(terms, BU, BV, prob.lam_min, prob.lam_max, 0.0, 16, 8, restart_every=6)
    assert len(res.ranks) == 8 and np.isfinite(res.rel_residual)
    res0 = orc.chebyshevt(terms, BU, BV, prob.lam_min, prob.lam_max, 0.0, 16, 6)
    np.testing.assert_allclose(res.iterates[5][0] @ res.iterates[5][1].T, res0.U @ res0.V.T, atol=1e-13)


# ------------------------------------------------------------------------------------------
# paper examples: clustering and the column <-> parameter map
# ------------------------------------------------------------------------------------------
def test_clustering_example_golden():
    with open(os.path.join(GOLDEN, "clustering_example.json")) as f:
        g = json.load(f)
    m1, m2, K = g["m1"], g["m2"], g["K"]
    subs = gen.split_subsets(m1 * m2, K)
    for (s, e), members, med in zip(subs, g["subsets"], g["upper_median"]):
        got = [[(p % m1) + 1, (p // m1) + 1] for p in range(s, e)]
        assert got == members
        assert list(gen.upper_median_index(s, e, m1)) == med


def test_column_parameter_map():
    cfg = gen.config_by_name("small")
    mu, nu = gen.parameter_grid(cfg)
    mu_ax = np.linspace(*cfg.mu_range, cfg.m1)
    nu_ax = np.linspace(*cfg.nu_range, cfg.m2)
    for p in range(1, cfg.m + 1):                      # 1-based column p
        assert mu[p - 1] == mu_ax[((p - 1) % cfg.m1)]
        assert nu[p - 1] == nu_ax[int(np.ceil(p / cfg.m1)) - 1]


# ------------------------------------------------------------------------------------------
# generator sanity (inputs, not the method)
# ------------------------------------------------------------------------------------------
def test_generator_structure(tiny):
    prob, terms, BU, BV = tiny
    op = prob.op
    g = op.g
    assert op.nnz == 25 * (3 * g - 2) ** 2
    mats = orc.csr_matrices(op.M, op.row_ptr, op.col_idx, op.vals)
    for A in mats:
        assert abs(A - A.T).max() == 0.0
    for A in mats[3:]:
        assert abs(np.linalg.norm(A.toarray(), 2) - 0.05) < 0.005
    # bounds enclose every block spectrum
    for m, v in zip(prob.mu, prob.nu):
        Aj = (mats[0] + m * mats[1] + op.rho_f * v * mats[2] + op.rho_f * mats[3] + m * mats[4]
              + op.lambda_s * mats[5]).toarray()
        ev = np.linalg.eigvalsh(Aj)
        assert prob.lam_min < ev[0] and ev[-1] < prob.lam_max


def test_generator_closed_form_bounds_enclose_small():
    prob = gen.make_problem("small")
    op = prob.op
    from scipy.sparse.linalg import eigsh
    for m in (prob.mu.min(), prob.mu.max()):
        for v in (prob.nu.min(), prob.nu.max()):
            vals = (op.vals[0] + m * (op.vals[1] + op.vals[4]) + op.rho_f * v * op.vals[2]
                    + op.rho_f * op.vals[3] + op.lambda_s * op.vals[5])
            A = sp.csr_matrix((vals, op.col_idx, op.row_ptr), shape=(op.M, op.M))
            hi = eigsh(A, k=1, which="LA", return_eigenvectors=False, tol=1e-8)[0]
            assert hi < prob.lam_max
    assert prob.lam_min < 4.0


def test_counter_rng_is_pure_function():
    a = gen.counter_normal(0, 7, np.arange(1000, dtype=np.uint64))
    b = gen.counter_normal(0, 7, np.arange(500, 1000, dtype=np.uint64))
    assert np.array_equal(a[500:], b)
    assert abs(a.mean()) < 0.15 and abs(a.std() - 1.0) < 0.1


# ------------------------------------------------------------------------------------------
# restart (reading S8, "restarted once after 6 iterations"): after a restart at k0 the error
# of an untruncated solve on a diagonal operator is p_j(Lambda) p_k0(Lambda) e_0 (Chebyshev error
# polynomials composed), entry by entry
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("k0,N", [(3, 7), (6, 12), (1, 4)])
def test_P1_restart_composes_error_polynomials(k0, N):
    terms, Lam, BU, BV = diagonal_problem(seed=9)
    lmin, lmax = Lam.min(), Lam.max()
    res = orc.chebyshevt(terms, BU, BV, lmin, lmax, tau=0.0, R=BV.shape[0], N=N, restart_every=k0)
    c, d = 0.5 * (lmax - lmin), 0.5 * (lmax + lmin)
    S_star = (BU @ BV.T) / Lam
    p = lambda j: cheb_T(j, (d - Lam) / c) / cheb_T(j, d / c)
    for k in range(1, N + 1):
        # k = q k0 + j updates: q completed cycles of k0 steps then j steps of a fresh cycle
        q, j = divmod(k, k0)
        err = p(k0) ** q * (p(j) if j else 1.0) * S_star
        X = orc.dense_product(*res.iterates[k - 1])
        assert np.linalg.norm(X - (S_star - err)) <= 1e-12 * np.linalg.norm(S_star), k


# ------------------------------------------------------------------------------------------
# generalized term lists -- the four-parameter operator, the
# theta-scheme operator and the Picard operator
# ------------------------------------------------------------------------------------------
def _literal_terms(prob, P):
    from synth import terms as st
    mats = orc.csr_matrices(prob.M, prob.row_ptr, prob.col_idx, prob.vals)
    cfg = prob.cfg
    if cfg.kind == "fourparam":
        return orc.term_list_fourparam(mats, P[:, 0], P[:, 1] * P[:, 3], P[:, 2], P[:, 3], *prob.refs)
    if cfg.kind == "theta":
        zero = sp.csr_matrix(mats[0].shape)
        return orc.term_list_theta(mats[1:], prob.rho_f, prob.lambda_s, P[:, 0], P[:, 1], mats[0], zero,
                                   st.RHO_S, st.DT, st.THETA)
    return orc.term_list_picard(mats, prob.rho_f, prob.lambda_s, P[:, 0], P[:, 1], *prob.refs)


@pytest.mark.parametrize("name", ["tiny4", "tinytheta", "tinypicard"])
def test_f4_general_form_equals_the_papers_operator(name):
    """The library's grouped form sum_g (sum_t C[t][g] A_t) S diag(d_g) (synth.terms) applies exactly the
    operator of the paper written term by term (oracle term lists), on a dense S and in Kronecker form."""
    from synth import terms as st
    prob = st.make_term_problem(name)
    P, D, BU, BV = prob.subset(0)
    lit = _literal_terms(prob, P)
    mats = orc.csr_matrices(prob.M, prob.row_ptr, prob.col_idx, prob.vals)
    if prob.cfg.kind == "theta":     # the grouped form's first array is the assembled mass matrix
        pass
    grp = orc.term_list_general(mats, prob.coef, D)
    rng = np.random.default_rng(4)
    S = rng.standard_normal((prob.M, P.shape[0]))
    a, b = orc.apply_dense(lit, S), orc.apply_dense(grp, S)
    assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(a)
    Ka, Kb = orc.kron_operator(lit), orc.kron_operator(grp)
    assert abs(Ka - Kb).max() <= 1e-13 * abs(Ka).max()
    assert np.all(D[prob.id_group] == 1.0)


def test_f4_fourparam_diagonal_closed_form():
    """Chebyshev error polynomial on a diagonal four-parameter operator: the eigenvalue of column j, entry
    i, written out from P:478-482 (A0 + A1 (mu - mu_r) + A2 (nu rho - nurho_r) + A3 (lam - lam_r) + Jmu mu +
    Jlam lam + Jrho rho, diagonal entries)."""
    rng = np.random.default_rng(21)
    M, n = 40, 6
    a = [1.0 + 3.0 * rng.random(M)] + [rng.random(M) for _ in range(6)]
    mats = [sp.diags(x).tocsr() for x in a]
    mu, nu, lam, rho = (0.5 + 1.5 * rng.random(n) for _ in range(4))
    refs = (0.5, 0.25, 0.5)
    terms = orc.term_list_fourparam(mats, mu, nu * rho, lam, rho, *refs)
    Lam = (a[0][:, None] + a[1][:, None] * (mu - refs[0])[None, :] + a[2][:, None] * (nu * rho - refs[1])[None, :]
           + a[3][:, None] * (lam - refs[2])[None, :] + a[4][:, None] * mu[None, :] + a[5][:, None] * lam[None, :]
           + a[6][:, None] * rho[None, :])
    BU, BV = rng.standard_normal((M, 2)), rng.standard_normal((n, 2))
    lmin, lmax = Lam.min(), Lam.max()
    for N in (1, 3, 8):
        res = orc.chebyshevt(terms, BU, BV, lmin, lmax, tau=0.0, R=n, N=N)
        c, d = 0.5 * (lmax - lmin), 0.5 * (lmax + lmin)
        S_star = (BU @ BV.T) / Lam
        pN = cheb_T(N, (d - Lam) / c) / cheb_T(N, d / c)
        X = orc.dense_product(res.U, res.V)
        assert np.linalg.norm(X - (1.0 - pN) * S_star) <= 1e-13 * np.linalg.norm(S_star)


def test_f4_theta_scheme_kronecker():
    """theta-scheme operator = (1/dt) I (x) A_t + theta (Kronecker form of P:30-36), assembled independently."""
    rng = np.random.default_rng(8)
    M, n = 30, 4
    mats = [sp.random(M, M, density=0.2, random_state=np.random.RandomState(i), format="csr") for i in range(6)]
    mass_f, mass_s = sp.diags(rng.random(M)).tocsr(), sp.diags(rng.random(M)).tocsr()
    d_mu, d_nu = rng.random(n), rng.random(n)
    rho, lam, rho_s, dt, th = 1.3, 2.0, 0.7, 0.05, 0.6
    terms = orc.term_list_theta(mats, rho, lam, d_mu, d_nu, mass_f, mass_s, rho_s, dt, th)
    K = orc.kron_operator(terms).toarray()
    I = np.eye(n)
    ref = np.kron(I, (rho * mass_f + rho_s * mass_s).toarray() / dt)
    F = (np.kron(I, mats[0].toarray()) + np.kron(np.diag(d_mu), mats[1].toarray()) + rho * np.kron(np.diag(d_nu), mats[2].toarray())
         + rho * np.kron(I, mats[3].toarray()) + np.kron(np.diag(d_mu), mats[4].toarray()) + lam * np.kron(I, mats[5].toarray()))
    assert np.abs(K - (ref + th * F)).max() <= 1e-13 * np.abs(ref + th * F).max()


def test_f4_term_problems_generate():
    from synth import terms as st
    for name in ("tiny4", "tinytheta", "tinypicard"):
        prob = st.make_term_problem(name)
        assert len(prob.vals) == prob.coef.shape[0] and prob.coef.shape[1] == prob.diagonals(prob.params[:1]).shape[0]
        assert 0 < prob.lam_min < prob.lam_max
        assert max(int(np.count_nonzero(prob.coef[:, g])) for g in range(prob.coef.shape[1])) <= 6


# ------------------------------------------------------------------------------------------
# GMREST (reading R14) against things other than itself
# ------------------------------------------------------------------------------------------
def _small_operator(seed=3, M=24, n=4):
    rng = np.random.default_rng(seed)
    base = sp.random(M, M, density=0.25, random_state=np.random.RandomState(seed), format="csr")
    mats = [(base + base.T) * 0.2 + sp.identity(M, format="csr") * 3.0]
    mats += [sp.random(M, M, density=0.2, random_state=np.random.RandomState(seed + i), format="csr") * 0.3
             for i in range(1, 6)]
    d_mu, d_nu = 0.5 + rng.random(n), 0.5 + rng.random(n)
    terms = orc.term_list(mats, 1.0, 2.0, d_mu, d_nu)
    BU, BV = rng.standard_normal((M, 2)), rng.standard_normal((n, 2))
    return terms, BU, BV


def test_f3_gmrest_untruncated_is_restarted_gmres():
    """tau = 0, R = n (no effective truncation): every cycle equals textbook restarted GMRES(m) on the
    vectorized system vec(L(S)) = vec(B), written here as a plain Arnoldi/least squares."""
    terms, BU, BV = _small_operator()
    M, n = BU.shape[0], BV.shape[0]
    K = orc.kron_operator(terms).toarray()
    b = orc.vec(BU @ BV.T)
    m, cycles = 5, 3
    res = orc.gmrest(terms, BU, BV, 0.0, n, m, cycles, 0.0)
    x = np.zeros(M * n)
    for c in range(cycles):
        r = b - K @ x
        beta = np.linalg.norm(r)
        Q = [r / beta]
        H = np.zeros((m + 1, m))
        for j in range(m):
            w = K @ Q[j]
            for i in range(j + 1):
                H[i, j] = w @ Q[i]
                w = w - H[i, j] * Q[i]
            H[j + 1, j] = np.linalg.norm(w)
            Q.append(w / H[j + 1, j])
        e1 = np.zeros(m + 1)
        e1[0] = beta
        y = np.linalg.lstsq(H, e1, rcond=None)[0]
        x = x + np.array(Q[:m]).T @ y
        rel = np.linalg.norm(b - K @ x) / np.linalg.norm(b)
        assert abs(res.cycle_residuals[c] - rel) <= 1e-9 * max(rel, 1e-12) + 1e-13, (c, res.cycle_residuals[c], rel)
    X = orc.dense_product(res.U, res.V)
    assert np.linalg.norm(orc.vec(X) - x) <= 1e-10 * np.linalg.norm(x)


def test_f3_gmrest_first_cycle_is_krylov_minimal():
    """The first cycle minimises the residual over the Krylov space span{b, Kb, ..., K^{m-1} b}
    (brute force: least squares over the explicit Krylov matrix)."""
    terms, BU, BV = _small_operator(seed=5)
    n = BV.shape[0]
    K = orc.kron_operator(terms).toarray()
    b = orc.vec(BU @ BV.T)
    for m in (1, 2, 4):
        res = orc.gmrest(terms, BU, BV, 0.0, n, m, 1, 0.0)
        Kr = np.array([np.linalg.matrix_power(K, i) @ b for i in range(m)]).T
        y = np.linalg.lstsq(K @ Kr, b, rcond=None)[0]
        best = np.linalg.norm(b - K @ Kr @ y) / np.linalg.norm(b)
        assert abs(res.cycle_residuals[0] - best) <= 1e-9 * best + 1e-14, (m, res.cycle_residuals[0], best)


def test_f3_gmrest_identity_and_zero_rhs():
    rng = np.random.default_rng(1)
    M, n = 20, 3
    I = sp.identity(M, format="csr")
    Z = sp.csr_matrix((M, M))
    terms = orc.term_list([2.0 * I, Z, Z, Z, Z, Z], 1.0, 2.0, rng.random(n), rng.random(n))
    BU, BV = rng.standard_normal((M, 2)), rng.standard_normal((n, 2))
    res = orc.gmrest(terms, BU, BV, 0.0, n, 6, 2, 1e-14)
    assert res.cycles == 1 and res.inner_steps == [1]            # breakdown after one step: exact
    assert np.linalg.norm(orc.dense_product(res.U, res.V) - 0.5 * BU @ BV.T) <= 1e-14 * np.linalg.norm(BU @ BV.T)
    res0 = orc.gmrest(terms, np.zeros((M, 1)), np.zeros((n, 1)), 0.0, n, 6, 2, 1e-12)
    assert res0.cycles == 0 and res0.U.shape[1] == 0


# ------------------------------------------------------------------------------------------
# the mean-based preconditioner, LU-applied
# ------------------------------------------------------------------------------------------
def test_f2_preconditioned_diagonal_closed_form():
    """Diagonal operator, diagonal P_T: the preconditioned operator has eigenvalues Lambda_ij / pi_i, so
    X_N = (1 - p_N(Lambda / Pi)) * S* with p_N the Chebyshev error polynomial of the preconditioned
    interval (P1 on P^{-1} L)."""
    terms, Lam, BU, BV = diagonal_problem(seed=13)
    P = orc.mean_preconditioner(terms)
    pi = P.diagonal()
    # P_T entries written out from P:334-341: every term at the midpoint of its diagonal
    ref = sum(c * 0.5 * (e.min() + e.max()) * A.diagonal() for c, A, e in terms)
    assert np.allclose(pi, ref, rtol=1e-15, atol=0)
    Q = Lam / pi[:, None]
    lmin, lmax = Q.min(), Q.max()
    S_star = (BU @ BV.T) / Lam
    c, d = 0.5 * (lmax - lmin), 0.5 * (lmax + lmin)
    for N in (1, 2, 5):
        res = orc.chebyshevt(terms, BU, BV, lmin, lmax, tau=0.0, R=BV.shape[0], N=N, precond=P)
        pN = cheb_T(N, (d - Q) / c) / cheb_T(N, d / c)
        X = orc.dense_product(res.U, res.V)
        assert np.linalg.norm(X - (1.0 - pN) * S_star) <= 1e-12 * np.linalg.norm(S_star), N


def test_f2_exact_preconditioner_converges_in_one_step():
    """One parameter at the mean: P_T equals the operator, P^{-1} L = I, bounds [1, 1] -> X_1 = S*."""
    prob = gen.make_problem("tiny")
    op = prob.op
    mats = orc.csr_matrices(op.M, op.row_ptr, op.col_idx, op.vals)
    terms = orc.term_list(mats, op.rho_f, op.lambda_s, np.array([1.3]), np.array([0.7]))
    rng = np.random.default_rng(2)
    BU, BV = rng.standard_normal((op.M, 1)), rng.standard_normal((1, 1))
    P = orc.mean_preconditioner(terms)
    res = orc.chebyshevt(terms, BU, BV, 1.0, 1.0, tau=0.0, R=1, N=1, precond=P)
    S = block_solve(terms, BU @ BV.T)
    assert np.linalg.norm(orc.dense_product(res.U, res.V) - S) <= 1e-12 * np.linalg.norm(S)
    assert res.rel_residual <= 1e-12


def test_f2_harness_bounds_enclose_the_spectra():
    """synth.precond (the bounds the f2 tests and bench pass in): its midpoint multipliers rebuild the
    oracle's P_T from the raw arrays, and the closed-form intervals contain the exact spectra of P_T
    and of P_T^{-1} A_j (dense generalized eigenvalues) for the Tiny subset."""
    import scipy.linalg as sla
    from synth import precond as spc
    prob = gen.make_problem("tiny")
    op, cfg = prob.op, prob.cfg
    d_mu, d_nu, _, _ = prob.subset(0)
    mats = orc.csr_matrices(op.M, op.row_ptr, op.col_idx, op.vals)
    terms = orc.term_list(mats, op.rho_f, op.lambda_s, d_mu, d_nu)
    E = spc.legacy_multipliers(op.rho_f, op.lambda_s, d_mu, d_nu)
    P_h = sum(m * A for m, A in zip(spc.midpoint(E), mats)).toarray()
    P_o = orc.mean_preconditioner(terms).toarray()
    assert np.max(np.abs(P_h - P_o)) <= 1e-14 * np.max(np.abs(P_o))
    p_min, p_max, lo, hi = spc.closed_form_bounds(cfg.g, op.rho_f, op.lambda_s, d_mu, d_nu)
    ev = np.linalg.eigvalsh(P_o)
    assert p_min <= ev[0] and ev[-1] <= p_max
    for j in (0, 5, 15):
        A = sum(m * M_ for m, M_ in zip(E[j], mats)).toarray()
        g = sla.eigh(A, P_o, eigvals_only=True)
        assert lo <= g[0] and g[-1] <= hi, (j, g[0], g[-1], lo, hi)
    assert spc.inner_steps(1.0, 1.0) == 1
    r = (np.sqrt(9.0) - 1) / (np.sqrt(9.0) + 1)
    q = spc.inner_steps(1.0, 9.0, 1e-10)
    assert 2 * r ** q <= 1e-10 < 2 * r ** (q - 1)
