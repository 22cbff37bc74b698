"""the mean-based preconditioner (LU-applied) on the GPU:
lrc_set_preconditioner + LRC_PRECONDITIONED against the oracle's preconditioned ChebyshevT
(oracle.chebyshevt(..., precond=oracle.mean_preconditioner(terms)), P^{-1} by SuperLU).

The library applies P_T^{-1} by a Chebyshev semi-iteration on P_T run to 1e-14 (R15), so the
north_star tolerances hold unchanged: X_k within 1e-8 (rel. Frobenius) every iteration, ranks equal
except near-ties, the unpreconditioned final residual within 1e-9."""
import numpy as np
import pytest

from oracle import chebyshevt as orc
from gpu_common import lowrank_rel_diff, make_ctx, near_tie, oracle_terms, problem, require_gpu, torch

pytestmark = pytest.mark.gpu


def _check_run(ctx, info, terms, BU, BV, lo, hi, tol, cap, N):
    worst = [0.0]

    def check(k, Uo, Vo, s):
        Uk, Vk, rk = ctx.get_iterate(k, cap)
        assert rk == Uo.shape[1] or near_tie(s, tol, cap, Uo.shape[1]), (k, rk, Uo.shape[1])
        err = lowrank_rel_diff(Uk[:, :rk], Vk[:, :rk], Uo, Vo)
        worst[0] = max(worst[0], err)
        assert err <= 1e-8, (k, err)

    ref = orc.chebyshevt(terms, BU, BV, lo, hi, tol, cap, N, record_iterates=False, on_iterate=check,
                         precond=orc.mean_preconditioner(terms))
    assert abs(info["rel_residual"] - ref.rel_residual) <= 1e-9, (info["rel_residual"], ref.rel_residual)
    return ref, worst[0]


@pytest.mark.parametrize("bounds", ["dense", "closed"])
def test_precond_legacy_tiny_every_iteration(bounds):
    require_gpu()
    from synth import precond as spc
    prob = problem("tiny")
    cfg, op = prob.cfg, prob.op
    d_mu, d_nu, BU, BV = prob.subset(0)
    if bounds == "dense":
        E = spc.legacy_multipliers(op.rho_f, op.lambda_s, d_mu, d_nu)
        p_min, p_max, lo, hi = spc.dense_bounds(op.M, op.row_ptr, op.col_idx, op.vals, E)
    else:
        p_min, p_max, lo, hi = spc.closed_form_bounds(cfg.g, op.rho_f, op.lambda_s, d_mu, d_nu)
    q = spc.inner_steps(p_min, p_max)
    ctx = make_ctx(op, d_mu, d_nu)
    ctx.set_preconditioner(p_min, p_max, q)
    N, cap, tol = cfg.n_iter, cfg.rank_cap, cfg.tol
    _, _, info = ctx.solve(torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda(), lo, hi, tol, cap, N,
                           record_iterates=True, preconditioned=True)
    ref, worst = _check_run(ctx, info, oracle_terms(op, d_mu, d_nu), BU, BV, lo, hi, tol, cap, N)
    print(f"tiny precond ({bounds}): q={q} kappa(P^-1 A)<={hi / lo:.2f} worst {worst:.2e} "
          f"rho {info['rel_residual']:.3e}")
    ctx.close()


def test_precond_graph_replay_and_invalidation():
    """A second solve replays the captured graph with the same result; new parameters discard the
    preconditioner (LRC_ERR_STATE until it is set again); a solve without the flag is unpreconditioned."""
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    from synth import precond as spc
    prob = problem("tiny")
    cfg, op = prob.cfg, prob.op
    d_mu, d_nu, BU, BV = prob.subset(0)
    p_min, p_max, lo, hi = spc.closed_form_bounds(cfg.g, op.rho_f, op.lambda_s, d_mu, d_nu)
    q = spc.inner_steps(p_min, p_max)
    ctx = make_ctx(op, d_mu, d_nu)
    bu, bv = torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda()
    N, cap, tol = 12, cfg.rank_cap, cfg.tol
    with pytest.raises(lrcheb.LrcError) as e:
        ctx.solve(bu, bv, lo, hi, tol, cap, N, preconditioned=True)
    assert e.value.status == lrcheb.LRC_ERR_STATE
    ctx.set_preconditioner(p_min, p_max, q)
    U1, V1, i1 = ctx.solve(bu, bv, lo, hi, tol, cap, N, preconditioned=True)
    U2, V2, i2 = ctx.solve(bu, bv, lo, hi, tol, cap, N, preconditioned=True)
    assert torch.equal(U1, U2) and torch.equal(V1, V2) and i1["rel_residual"] == i2["rel_residual"]
    U3, V3, i3 = ctx.solve(bu, bv, prob.lam_min, prob.lam_max, tol, cap, N)         # unpreconditioned
    ref = orc.chebyshevt(oracle_terms(op, d_mu, d_nu), BU, BV, prob.lam_min, prob.lam_max, tol, cap, N)
    assert abs(i3["rel_residual"] - ref.rel_residual) <= 1e-9
    ctx.set_params(d_mu, d_nu)
    with pytest.raises(lrcheb.LrcError) as e:
        ctx.solve(bu, bv, lo, hi, tol, cap, N, preconditioned=True)
    assert e.value.status == lrcheb.LRC_ERR_STATE
    with pytest.raises(lrcheb.LrcError):
        ctx.set_preconditioner(-1.0, p_max, q)
    ctx.close()


@pytest.mark.parametrize("name", ["tiny4", "tinypicard"])
def test_precond_general_terms(name):
    """The preconditioner of a general term list (SURVEY §8 f4 form): P_T = sum_t A_t * mean(e_t)."""
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    from synth import precond as spc
    from synth import terms as st
    from test_gpu_terms import _literal_terms
    prob = st.make_term_problem(name)
    cfg = prob.cfg
    P, D, BU, BV = prob.subset(0)
    E = spc.term_multipliers(prob.coef, D)
    p_min, p_max, lo, hi = spc.dense_bounds(prob.M, prob.row_ptr, prob.col_idx, prob.vals, E)
    q = spc.inner_steps(p_min, p_max)
    ctx = lrcheb.Context(0)
    ctx.set_operator_terms(prob.row_ptr, prob.col_idx, prob.vals, prob.coef, prob.id_group)
    ctx.set_diagonals(D)
    ctx.set_preconditioner(p_min, p_max, q)
    N, cap, tol = cfg.n_iter, cfg.rank_cap, cfg.tol
    _, _, info = ctx.solve(torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda(), lo, hi, tol, cap, N,
                           record_iterates=True, preconditioned=True)
    _, worst = _check_run(ctx, info, _literal_terms(prob, P), BU, BV, lo, hi, tol, cap, N)
    print(f"{name} precond: q={q} worst {worst:.2e} rho {info['rel_residual']:.3e}")
    ctx.close()
