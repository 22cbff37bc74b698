"""GPU-vs-oracle parity through the C ABI (BASELINE.json north_star tolerances).

  * K1 operator application (a1): every block within 1e-12 relative (fp64 rounding-order only).
  * truncation (a2-a6): products within 1e-12, ranks equal, sigma within 1e-12 sigma_1.
  * ChebyshevT (whole path): X_k within 1e-8 relative Frobenius for every recorded k, equal ranks
    except near-ties (reading S13), final residual within 1e-9 (reading S14).
"""
import numpy as np
import pytest

from oracle import chebyshevt as orc
from gpu_common import (lowrank_rel_diff, make_ctx, near_tie, oracle_terms, problem, random_csr,
                              require_gpu, torch)

pytestmark = pytest.mark.gpu


def _blocks(W, r, nb):
    return [W[:, t * r:(t + 1) * r] for t in range(nb)]


def _oracle_grouped(terms, U, rho, lam):
    """W0 = (A0 + rho Jrho + lam Jlam)U, W1 = (A1 + Jmu)U, W2 = rho A2 U from the oracle's six terms."""
    A = [t[1] for t in terms]
    return [A[0] @ U + rho * (A[3] @ U) + lam * (A[5] @ U), A[1] @ U + A[4] @ U, rho * (A[2] @ U)]


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# ------------------------------------------------------------------------------------------
# a1: fused SpMM
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name,r", [("tiny", 1), ("tiny", 10), ("small", 20), ("small", 33), ("small", 60),
                                    ("small", 100)])
def test_apply_lowrank_modes(name, r):
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    prob = problem(name)
    op = prob.op
    d_mu, d_nu, _, _ = prob.subset(0)
    ctx = make_ctx(op, d_mu, d_nu)
    rng = np.random.default_rng(r)
    U = rng.standard_normal((op.M, r))
    terms = oracle_terms(op, d_mu, d_nu)
    ref3 = _oracle_grouped(terms, U, op.rho_f, op.lambda_s)
    W = ctx.apply_lowrank(U, lrcheb.LRC_APPLY_PLAIN3)
    for got, ref in zip(_blocks(W, r, 3), ref3):
        assert _rel(got, ref) <= 1e-12
    gamma = 0.037
    W = ctx.apply_lowrank(torch.from_numpy(U).cuda(), lrcheb.LRC_APPLY_S2STEP, gamma).cpu().numpy()
    refs = [U - gamma * ref3[0], ref3[1], ref3[2]]
    for got, ref in zip(_blocks(W, r, 3), refs):
        assert _rel(got, ref) <= 1e-12
    W = ctx.apply_lowrank(U, lrcheb.LRC_APPLY_SIX)
    for t, got in enumerate(_blocks(W, r, 6)):
        c, A, _ = terms[t]
        assert _rel(got, c * (A @ U)) <= 1e-12
    ctx.close()


@pytest.mark.parametrize("diag_only", [False, True])
def test_apply_irregular_pattern(diag_only):
    """Generic CSR: random row lengths, empty rows, ragged M (not a multiple of any tile)."""
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    rng = np.random.default_rng(17)
    M = 1237
    op = random_csr(M, rng, density=0.02, empty_rows=(0, 5, 6, 7, 1000, M - 1), diag_only=diag_only)
    n = 9
    d_mu, d_nu = rng.random(n) + 0.5, rng.random(n) + 0.5
    ctx = make_ctx(op, d_mu, d_nu)
    terms = oracle_terms(op, d_mu, d_nu)
    for r in (3, 40):
        U = rng.standard_normal((M, r))
        W = ctx.apply_lowrank(U, lrcheb.LRC_APPLY_PLAIN3)
        for got, ref in zip(_blocks(W, r, 3), _oracle_grouped(terms, U, op.rho_f, op.lambda_s)):
            assert _rel(got, ref) <= 1e-12
    ctx.close()


@pytest.mark.parametrize("ncols,ld,cfg", [(16, 16, "tiny"), (256, 256, "tiny"), (37, 37, "tiny"),
                                           (100, 100, "small"), (37, 41, "tiny"), (200, 203, "small")])
def test_apply_dense(ncols, ld, cfg):
    """BASELINE config 5 mode: Y = sum_t c_t A_t S D_t (oracle.apply_dense).  Covers one and several
    64-column chunks, a ragged last chunk, odd widths and an odd leading dimension (8-byte copies)."""
    require_gpu()
    prob = problem(cfg)
    op = prob.op
    rng = np.random.default_rng(ncols + ld)
    d_mu, d_nu = 0.25 + 3.75 * rng.random(ncols), 0.25 + 3.75 * rng.random(ncols)
    ctx = make_ctx(op, d_mu, d_nu)
    S_full = rng.standard_normal((op.M, ld))
    S = S_full[:, :ncols]
    if ld != ncols:    # a strided device view keeps the leading dimension
        import torch
        Y = ctx.apply_dense(torch.from_numpy(S_full).cuda()[:, :ncols]).cpu().numpy()
    else:
        Y = ctx.apply_dense(S)
    ref = orc.apply_dense(oracle_terms(op, d_mu, d_nu), S)
    assert _rel(Y, ref) <= 1e-12
    ctx.close()


# ------------------------------------------------------------------------------------------
# a2-a6: truncation
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("w,cap,tau,deficient", [(12, 5, 0.0, False), (40, 10, 1e-8, False),
                                                  (30, 16, 1e-12, True), (7, 7, 0.0, False),
                                                  (100, 20, 1e-10, False)])
def test_truncate(w, cap, tau, deficient):
    require_gpu()
    prob = problem("tiny")
    op = prob.op
    n = 16 if w <= 40 else 40
    rng = np.random.default_rng(w + cap)
    d_mu, d_nu = rng.random(n) + 0.5, rng.random(n) + 0.5
    ctx = make_ctx(op, d_mu, d_nu)
    U = rng.standard_normal((op.M, w)) * np.logspace(0, -9, w)[None, :]
    if deficient:      # duplicated column blocks: exactly rank-deficient concatenation (the k = 2 case)
        U[:, w // 2:] = U[:, : w - w // 2]
    V = rng.standard_normal((n, w))
    Ug, Vg, rg, sg = ctx.truncate(U, V, tau, cap)
    Uo, Vo, so = orc.truncate(U, V, tau, cap)
    assert rg == Uo.shape[1] or near_tie(so, tau, cap, Uo.shape[1])
    assert lowrank_rel_diff(Ug[:, :rg], Vg[:, :rg], Uo, Vo) <= 1e-10
    k = min(len(sg), len(so), cap)
    assert np.all(np.abs(sg[:k] - so[:k]) <= 1e-11 * so[0])
    # columns beyond the rank are zero, U' orthonormal
    assert np.all(Ug[:, rg:] == 0) and np.all(Vg[:, rg:] == 0)
    assert np.linalg.norm(Ug[:, :rg].T @ Ug[:, :rg] - np.eye(rg)) <= 1e-8
    ctx.close()


# ------------------------------------------------------------------------------------------
# whole ChebyshevT path
# ------------------------------------------------------------------------------------------
def _solve_parity(name, subset, N, check_every=1, device_inputs=False, **kw):
    prob = problem(name)
    cfg, op = prob.cfg, prob.op
    d_mu, d_nu, BU, BV = prob.subset(subset)
    ctx = make_ctx(op, d_mu, d_nu, device_inputs=device_inputs)
    tau, cap = kw.pop("tau", cfg.tol), kw.pop("cap", cfg.rank_cap)
    if device_inputs:
        bu, bv = torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda()
    else:
        bu, bv = BU, BV
    U, V, info = ctx.solve(bu, bv, prob.lam_min, prob.lam_max, tau, cap, N, record_iterates=True, **kw)
    terms = oracle_terms(op, d_mu, d_nu)
    ref = orc.chebyshevt(terms, BU, BV, prob.lam_min, prob.lam_max, tau, cap, N,
                         restart_every=kw.get("restart_every") or None)
    worst = 0.0
    for k in range(1, N + 1):
        if k % check_every and k != N:
            continue
        Uk, Vk, rk = ctx.get_iterate(k, cap)
        Uo, Vo = ref.iterates[k - 1]
        assert rk == ref.ranks[k - 1] or near_tie(ref.sigmas[k - 1], tau, cap, ref.ranks[k - 1]), (k, rk, ref.ranks[k - 1])
        err = lowrank_rel_diff(Uk[:, :rk], Vk[:, :rk], Uo, Vo)
        worst = max(worst, err)
        assert err <= 1e-8, (k, err)
    for k in range(1, N + 1):      # the ABI's rank history, every iteration (near-ties exempt, S13)
        rk, ro = info["rank_history"][k - 1], ref.ranks[k - 1]
        assert rk == ro or near_tie(ref.sigmas[k - 1], tau, cap, ro), (k, rk, ro)
    assert abs(info["rel_residual"] - ref.rel_residual) <= 1e-9, (info["rel_residual"], ref.rel_residual)
    if device_inputs:
        U, V = U.cpu().numpy(), V.cpu().numpy()
    r = info["rank"]
    assert lowrank_rel_diff(U[:, :r], V[:, :r], ref.U, ref.V) <= 1e-8
    ctx.close()
    return worst, info, ref


def test_solve_tiny_every_iteration():
    require_gpu()
    _solve_parity("tiny", 0, 30)


def test_solve_tiny_device_inputs_no_graph():
    require_gpu()
    _solve_parity("tiny", 0, 12, device_inputs=True, no_graph=True)


def test_solve_small_subsets():
    require_gpu()
    for k in (0, 3):
        _solve_parity("small", k, 50)


def test_solve_restart_and_tau0():
    require_gpu()
    _solve_parity("tiny", 0, 14, restart_every=6, tau=0.0, cap=16)


def test_solve_small_cold_jacobi_start():
    """Same parity with the core SVD started from W = I every iteration (LRC_NO_WARM_START)."""
    require_gpu()
    _solve_parity("small", 1, 30, warm_start=False)


def test_solve_wide_parameter_block():
    """n = 111 parameters in one subset (the build limit is min(n, w) <= 112): p grows to 111, an odd
    width with the PT = 14 instantiations of the tall-skinny kernels (Y block 111 wide + its zero pad
    column, R1^{-1} 111 x 111) against the oracle."""
    require_gpu()
    prob = problem("tiny")
    op = prob.op
    rng = np.random.default_rng(7)
    n, r_B, tau, cap, N = 111, 3, 1e-12, 40, 8
    # parameter values inside the grid's range keep the tiny spectrum bounds valid (monotone in mu, nu)
    d_mu, d_nu = 0.5 + 1.5 * rng.random(n), 0.5 + 1.5 * rng.random(n)
    BU, BV = rng.standard_normal((op.M, r_B)), rng.standard_normal((n, r_B))
    ctx = make_ctx(op, d_mu, d_nu)
    U, V, info = ctx.solve(BU, BV, prob.lam_min, prob.lam_max, tau, cap, N, record_iterates=True)
    ref = orc.chebyshevt(oracle_terms(op, d_mu, d_nu), BU, BV, prob.lam_min, prob.lam_max, tau, cap, N)
    for k in range(1, N + 1):
        Uk, Vk, rk = ctx.get_iterate(k, cap)
        Uo, Vo = ref.iterates[k - 1]
        assert rk == ref.ranks[k - 1] or near_tie(ref.sigmas[k - 1], tau, cap, ref.ranks[k - 1]), (k, rk)
        assert lowrank_rel_diff(Uk[:, :rk], Vk[:, :rk], Uo, Vo) <= 1e-8, k
    assert max(ref.ranks) == cap                      # the cap binds, so p really reached min(n, w)
    assert abs(info["rel_residual"] - ref.rel_residual) <= 1e-9
    ctx.close()


def test_apply_dense_tall_long_block():
    """A node block of 6 rows sharing a 165-entry column list: its staged size (3 x 6 x pitch(165))
    exceeds the value stage, so it must take the chunked long path."""
    require_gpu()
    import scipy.sparse as sp
    from gpu_common import gen
    rng = np.random.default_rng(11)
    M = 400
    rows, cols = [], []
    for i in range(M):
        if 100 <= i < 106:
            c = np.arange(50, 215)                       # the tall long block
        else:
            c = np.unique(np.concatenate([[i], rng.choice(M, 7, replace=False)]))
        rows += [i] * len(c)
        cols += list(c)
    A = sp.csr_matrix((np.ones(len(rows)), (rows, cols)), shape=(M, M))
    A.sort_indices()
    vals = [rng.standard_normal(A.nnz) for _ in range(6)]
    op = gen.Operator(M=M, row_ptr=A.indptr.astype(np.int32), col_idx=A.indices.astype(np.int32), vals=vals,
                      rho_f=1.3, lambda_s=2.0)
    n = 64
    d_mu, d_nu = rng.random(n) + 0.5, rng.random(n) + 0.5
    ctx = make_ctx(op, d_mu, d_nu)
    S = rng.standard_normal((M, n))
    Y = ctx.apply_dense(S)
    ref = orc.apply_dense(oracle_terms(op, d_mu, d_nu), S)
    assert _rel(Y, ref) <= 1e-12
    W = ctx.apply_lowrank(S[:, :40])
    for got, refb in zip(_blocks(W, 40, 3), _oracle_grouped(oracle_terms(op, d_mu, d_nu), S[:, :40], op.rho_f, op.lambda_s)):
        assert _rel(got, refb) <= 1e-12
    ctx.close()


def test_async_solve_and_caller_workspace():
    """LRC_ASYNC (enqueue, then lrc_solve_wait) and a caller-owned workspace arena
    (lrc_workspace_bytes / lrc_set_workspace) give the same iterate as the default path."""
    require_gpu()
    prob = problem("small")
    cfg, op = prob.cfg, prob.op
    d_mu, d_nu, BU, BV = prob.subset(2)
    ctx = make_ctx(op, d_mu, d_nu)
    bu, bv = torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda()
    U0, V0, info0 = ctx.solve(bu, bv, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, cfg.n_iter)
    nbytes = ctx.workspace_bytes(BU.shape[1], cfg.rank_cap, cfg.n_iter)
    assert nbytes > 8 * op.M * cfg.rank_cap * 7
    arena = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    ctx.set_workspace(arena)
    Uo = torch.full((op.M, cfg.rank_cap), -7.0, dtype=torch.float64, device="cuda")
    Vo = torch.full((len(d_mu), cfg.rank_cap), -7.0, dtype=torch.float64, device="cuda")
    ctx.solve_async(bu, bv, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, cfg.n_iter, out=(Uo, Vo))
    info = ctx.wait()
    assert info["rank"] == info0["rank"] and info["rank_history"] == info0["rank_history"]
    r = info["rank"]
    U0, V0, U1, V1 = (x.cpu().numpy() for x in (U0, V0, Uo, Vo))
    assert lowrank_rel_diff(U1[:, :r], V1[:, :r], U0[:, :r], V0[:, :r]) <= 1e-12
    assert abs(info["rel_residual"] - info0["rel_residual"]) <= 1e-12
    # too small an arena -> LRC_ERR_NOMEM, not a fault
    from paper_2008_10275_b200 import lrcheb
    ctx.set_workspace(torch.empty(1 << 20, dtype=torch.uint8, device="cuda"))
    with pytest.raises(lrcheb.LrcError) as e:
        ctx.solve(bu, bv, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, cfg.n_iter)
    assert e.value.status == lrcheb.LRC_ERR_NOMEM
    ctx.set_workspace(None)
    ctx.solve(bu, bv, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, 3)
    ctx.close()


def test_numeric_error_leaves_outputs_untouched():
    """A non-finite right-hand side makes the core SVD flag a non-finite sigma: lrc_solve returns
    LRC_ERR_NUMERIC and does not write U_out / V_out (include/lrcheb.h error contract)."""
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    prob = problem("tiny")
    cfg, op = prob.cfg, prob.op
    d_mu, d_nu, BU, BV = prob.subset(0)
    ctx = make_ctx(op, d_mu, d_nu)
    BU = BU.copy()
    BU[7, 1] = np.nan
    for device in (False, True):
        if device:
            Uo = torch.full((op.M, cfg.rank_cap), 3.0, dtype=torch.float64, device="cuda")
            Vo = torch.full((len(d_mu), cfg.rank_cap), 3.0, dtype=torch.float64, device="cuda")
            args = (torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda())
        else:
            Uo, Vo = np.full((op.M, cfg.rank_cap), 3.0), np.full((len(d_mu), cfg.rank_cap), 3.0)
            args = (BU, BV)
        with pytest.raises(lrcheb.LrcError) as e:
            ctx.solve(*args, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, 4, out=(Uo, Vo))
        assert e.value.status == lrcheb.LRC_ERR_NUMERIC
        Uh = Uo.cpu().numpy() if device else Uo
        Vh = Vo.cpu().numpy() if device else Vo
        assert np.all(Uh == 3.0) and np.all(Vh == 3.0)
    ctx.close()
