"""generalized term lists on the GPU (lrc_set_operator_terms / lrc_set_diagonals):
the four-parameter Newton operator, the theta-scheme operator and the
Picard operator, solved by the same ChebyshevT path and compared with the CPU oracle, whose
term lists are written from the paper term by term (oracle.term_list_fourparam / _theta / _picard).

Tolerances as north_star: X_k within 1e-8 (rel. Frobenius) every iteration, ranks equal except
near-ties, final residual within 1e-9; the operator application within 1e-12 (fp64 rounding order)."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import chebyshevt as orc
from gpu_common import lowrank_rel_diff, near_tie, require_gpu, torch

pytestmark = pytest.mark.gpu


def _problem(name):
    from synth import terms as st
    return st.make_term_problem(name)


def _literal_terms(prob, P):
    from synth import terms as st
    mats = orc.csr_matrices(prob.M, prob.row_ptr, prob.col_idx, prob.vals)
    if prob.cfg.kind == "fourparam":
        return orc.term_list_fourparam(mats, P[:, 0], P[:, 1] * P[:, 3], P[:, 2], P[:, 3], *prob.refs)
    if prob.cfg.kind == "theta":
        zero = sp.csr_matrix(mats[0].shape)
        return orc.term_list_theta(mats[1:], prob.rho_f, prob.lambda_s, P[:, 0], P[:, 1], mats[0], zero,
                                   st.RHO_S, st.DT, st.THETA)
    return orc.term_list_picard(mats, prob.rho_f, prob.lambda_s, P[:, 0], P[:, 1], *prob.refs)


def _ctx(prob, D):
    from paper_2008_10275_b200 import lrcheb
    ctx = lrcheb.Context(0)
    ctx.set_operator_terms(prob.row_ptr, prob.col_idx, prob.vals, prob.coef, prob.id_group)
    ctx.set_diagonals(D)
    return ctx


@pytest.mark.parametrize("name,r", [("tiny4", 10), ("tinytheta", 7), ("tinypicard", 20), ("small4", 33)])
def test_terms_apply_matches_oracle_operator(name, r):
    """sum_g W_g (d_g * V)^T from the grouped GPU application equals the oracle's L(U V^T)."""
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    prob = _problem(name)
    P, D, _, _ = prob.subset(0)
    ctx = _ctx(prob, D)
    rng = np.random.default_rng(r)
    U, V = rng.standard_normal((prob.M, r)), rng.standard_normal((P.shape[0], r))
    W = ctx.apply_lowrank(U, lrcheb.LRC_APPLY_PLAIN3)
    G = prob.coef.shape[1]
    X = sum(W[:, g * r:(g + 1) * r] @ (D[g][:, None] * V).T for g in range(G))
    UL, VL = orc.apply_lowrank(_literal_terms(prob, P), U, V)
    ref = UL @ VL.T
    assert np.linalg.norm(X - ref) <= 1e-12 * np.linalg.norm(ref)
    W6 = ctx.apply_lowrank(U, lrcheb.LRC_APPLY_SIX)         # every array alone: A_t U
    mats = orc.csr_matrices(prob.M, prob.row_ptr, prob.col_idx, prob.vals)
    for t, A in enumerate(mats):
        ref_t = A @ U
        assert np.linalg.norm(W6[:, t * r:(t + 1) * r] - ref_t) <= 1e-12 * max(np.linalg.norm(ref_t), 1e-300)
    ctx.close()


@pytest.mark.parametrize("name,subset,check_every", [("tiny4", 0, 1), ("tinytheta", 0, 1), ("tinypicard", 0, 1),
                                                     ("small4", 1, 5)])
def test_terms_solve_matches_oracle(name, subset, check_every):
    require_gpu()
    prob = _problem(name)
    cfg = prob.cfg
    P, D, BU, BV = prob.subset(subset)
    ctx = _ctx(prob, D)
    N, cap, tol = cfg.n_iter, cfg.rank_cap, cfg.tol
    U, V, info = ctx.solve(torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda(), prob.lam_min, prob.lam_max,
                           tol, cap, N, record_iterates=True)
    ref = orc.chebyshevt(_literal_terms(prob, P), BU, BV, prob.lam_min, prob.lam_max, tol, cap, N)
    for k in range(1, N + 1):
        rk, ro = info["rank_history"][k - 1], ref.ranks[k - 1]
        assert rk == ro or near_tie(ref.sigmas[k - 1], tol, cap, ro), (k, rk, ro)
        if k % check_every and k != N:
            continue
        Uk, Vk, rk2 = ctx.get_iterate(k, cap)
        Uo, Vo = ref.iterates[k - 1]
        assert lowrank_rel_diff(Uk[:, :rk2], Vk[:, :rk2], Uo, Vo) <= 1e-8, k
    assert abs(info["rel_residual"] - ref.rel_residual) <= 1e-9, (info["rel_residual"], ref.rel_residual)
    assert info["rel_residual"] < 1.0
    ctx.close()


def test_terms_rejects_bad_lists():
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    prob = _problem("tiny4")
    P, D, _, _ = prob.subset(0)
    ctx = lrcheb.Context(0)
    with pytest.raises(lrcheb.LrcError) as e:          # identity group without an all-ones diagonal
        ctx.set_operator_terms(prob.row_ptr, prob.col_idx, prob.vals, prob.coef, 1)
        ctx.set_diagonals(D)
    assert e.value.status == lrcheb.LRC_ERR_ARG
    ctx.set_operator_terms(prob.row_ptr, prob.col_idx, prob.vals, prob.coef, 0)
    with pytest.raises(lrcheb.LrcError) as e:          # the legacy parameter call does not apply
        ctx.set_params(P[:, 0], P[:, 1])
    assert e.value.status == lrcheb.LRC_ERR_STATE
    ctx.close()
