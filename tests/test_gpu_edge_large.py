"""GPU edge cases and full-size (BASELINE config 'large') parity, through the C ABI.

Full size: the oracle cannot run 100 Large iterations inside a test (SURVEY §7 hard part 6); the
whole trajectory is compared with the oracle's goldens in test_gpu_fullsize.py, and here one
steady-state step is checked lock-step against the live oracle: the oracle's step
(oracle.chebyshevt_step, literal six-term + Householder truncation) applied to the GPU's X_{k-1}, X_k
must reproduce the GPU's X_{k+1} (reading S15: lock-step single-step checks).
"""
import numpy as np
import pytest

from oracle import chebyshevt as orc
from gpu_common import lowrank_rel_diff, make_ctx, near_tie, oracle_terms, problem, require_gpu, torch

pytestmark = pytest.mark.gpu


def _tiny_ctx():
    prob = problem("tiny")
    d_mu, d_nu, BU, BV = prob.subset(0)
    return prob, make_ctx(prob.op, d_mu, d_nu), d_mu, d_nu, BU, BV


def test_rank_zero_rhs():
    require_gpu()
    prob, ctx, *_ = _tiny_ctx()
    n = prob.cfg.m
    U, V, info = ctx.solve(np.zeros((prob.op.M, 0)), np.zeros((n, 0)), prob.lam_min, prob.lam_max, 1e-10, 4, 5)
    assert info["rank"] == 0 and info["rel_residual"] == 0.0
    assert np.all(U == 0) and np.all(V == 0)
    ctx.close()


def test_single_iteration_is_truncated_gamma_B():
    """N = 1: X_1 = T(gamma B) (w_1 = 1, X_0 = 0)."""
    require_gpu()
    prob, ctx, d_mu, d_nu, BU, BV = _tiny_ctx()
    gamma = 2.0 / (prob.lam_min + prob.lam_max)
    U, V, info = ctx.solve(BU, BV, prob.lam_min, prob.lam_max, 0.0, 10, 1)
    assert info["rank"] == BU.shape[1]
    assert lowrank_rel_diff(U[:, :info["rank"]], V[:, :info["rank"]], BU, gamma * BV) <= 1e-12
    ctx.close()


def test_cap_one_and_richardson_c0():
    require_gpu()
    prob, ctx, d_mu, d_nu, BU, BV = _tiny_ctx()
    terms = oracle_terms(prob.op, d_mu, d_nu)
    for (lmin, lmax, cap, N) in [(prob.lam_min, prob.lam_max, 1, 6), (prob.lam_max, prob.lam_max, 6, 8)]:
        U, V, info = ctx.solve(BU, BV, lmin, lmax, 1e-12, cap, N)
        ref = orc.chebyshevt(terms, BU, BV, lmin, lmax, 1e-12, cap, N, record_iterates=False)
        r = info["rank"]
        assert r == ref.U.shape[1]
        assert lowrank_rel_diff(U[:, :r], V[:, :r], ref.U, ref.V) <= 1e-8
        assert abs(info["rel_residual"] - ref.rel_residual) <= 1e-9
    ctx.close()


def test_invalid_arguments_are_reported():
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    prob, ctx, d_mu, d_nu, BU, BV = _tiny_ctx()
    with pytest.raises(lrcheb.LrcError) as e:          # lambda_min <= 0
        ctx.solve(BU, BV, 0.0, 1.0, 1e-8, 4, 3)
    assert e.value.status == lrcheb.LRC_ERR_ARG
    with pytest.raises(lrcheb.LrcError) as e:          # rank cap > n
        ctx.solve(BU, BV, 1.0, 2.0, 1e-8, 17, 3)
    assert e.value.status == lrcheb.LRC_ERR_ARG
    bad = prob.op.col_idx.copy()
    bad[1], bad[2] = bad[2], bad[1]                     # unsorted row
    with pytest.raises(lrcheb.LrcError) as e:
        ctx.set_operator(prob.op.row_ptr, bad, prob.op.vals, 1.0, 2.0)
    assert e.value.status == lrcheb.LRC_ERR_ARG
    ctx2 = lrcheb.Context(0)
    with pytest.raises(lrcheb.LrcError) as e:          # solve before set_operator
        ctx2.solve(BU, BV, 1.0, 2.0, 1e-8, 4, 3)
    assert e.value.status == lrcheb.LRC_ERR_STATE
    ctx2.close()
    ctx.close()


@pytest.fixture(scope="module")
def large():
    prob = problem("large")
    d_mu, d_nu, BU, BV = prob.subset(0)
    ctx = make_ctx(prob.op, d_mu, d_nu, device_inputs=True)
    terms = oracle_terms(prob.op, d_mu, d_nu)
    yield prob, ctx, terms, d_mu, d_nu, BU, BV
    ctx.close()


def test_large_steady_state_lockstep_step(large):
    require_gpu()
    prob, ctx, terms, d_mu, d_nu, BU, BV = large
    cfg = prob.cfg
    N = 12
    bu, bv = torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda()
    _, _, info = ctx.solve(bu, bv, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, N, record_iterates=True,
                           skip_residual=True)
    U10, V10, r10 = ctx.get_iterate(N - 2, cfg.rank_cap)
    U11, V11, r11 = ctx.get_iterate(N - 1, cfg.rank_cap)
    U12, V12, r12 = ctx.get_iterate(N, cfg.rank_cap)
    assert r11 == cfg.rank_cap                        # steady state: cap-bound
    c, d = orc.chebyshev_cd(prob.lam_min, prob.lam_max)
    om = orc.omegas(prob.lam_min, prob.lam_max, N)
    Uo, Vo, so = orc.chebyshevt_step(terms, BU, BV, U11[:, :r11], V11[:, :r11], U10[:, :r10], V10[:, :r10],
                                     om[N - 1], 1.0 / d, cfg.tol, cfg.rank_cap)
    assert r12 == Uo.shape[1] or near_tie(so, cfg.tol, cfg.rank_cap, Uo.shape[1])
    assert lowrank_rel_diff(U12[:, :r12], V12[:, :r12], Uo, Vo) <= 1e-8
