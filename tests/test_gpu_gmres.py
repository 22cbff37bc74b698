"""GMREST (truncated restarted GMRES; DESIGN.md
reading R14) through the C ABI, against the CPU oracle's gmrest (literal six-term / four-parameter
term lists, Householder + LAPACK SVD truncation): the honest residual after every restart cycle
within 1e-9, the Arnoldi step counts equal, the final iterate within 1e-8 (rel. Frobenius)."""
import numpy as np
import pytest

from oracle import chebyshevt as orc
from gpu_common import lowrank_rel_diff, make_ctx, oracle_terms, problem, require_gpu, torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,subset,m,cycles,cap,tau", [("tiny", 0, 6, 3, 10, 1e-10), ("small", 2, 6, 2, 20, 1e-9),
                                                          ("tiny", 0, 4, 4, 16, 0.0)])
def test_gmrest_matches_oracle(name, subset, m, cycles, cap, tau):
    require_gpu()
    prob = problem(name)
    op = prob.op
    d_mu, d_nu, BU, BV = prob.subset(subset)
    ctx = make_ctx(op, d_mu, d_nu)
    U, V, info = ctx.solve_gmres(torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda(), tau, 0.0, cap, m, cycles)
    ref = orc.gmrest(oracle_terms(op, d_mu, d_nu), BU, BV, tau, cap, m, cycles, 0.0)
    assert info["cycles"] == ref.cycles and info["inner_steps"] == ref.inner_steps, (info, ref.inner_steps)
    for c, (rg, ro) in enumerate(zip(info["cycle_residuals"], ref.cycle_residuals)):
        assert abs(rg - ro) <= 1e-9, (c, rg, ro)
    r = info["rank"]
    Uh, Vh = U.cpu().numpy(), V.cpu().numpy()
    assert r == ref.U.shape[1]
    assert lowrank_rel_diff(Uh[:, :r], Vh[:, :r], ref.U, ref.V) <= 1e-8
    assert ref.cycle_residuals[-1] < ref.cycle_residuals[0] or ref.cycle_residuals[0] < 1e-12
    ctx.close()


def test_gmrest_four_parameter_operator():
    """GMREST on a general term list (SURVEY §8 f4 x f3): the four-parameter operator of P:478-482."""
    require_gpu()
    from synth import terms as st
    from paper_2008_10275_b200 import lrcheb
    import scipy.sparse as sp
    prob = st.make_term_problem("tiny4")
    P, D, BU, BV = prob.subset(0)
    ctx = lrcheb.Context(0)
    ctx.set_operator_terms(prob.row_ptr, prob.col_idx, prob.vals, prob.coef, prob.id_group)
    ctx.set_diagonals(D)
    U, V, info = ctx.solve_gmres(BU, BV, 1e-10, 0.0, 8, 6, 2)
    mats = orc.csr_matrices(prob.M, prob.row_ptr, prob.col_idx, prob.vals)
    terms = orc.term_list_fourparam(mats, P[:, 0], P[:, 1] * P[:, 3], P[:, 2], P[:, 3], *prob.refs)
    ref = orc.gmrest(terms, BU, BV, 1e-10, 8, 6, 2, 0.0)
    assert info["inner_steps"] == ref.inner_steps
    for rg, ro in zip(info["cycle_residuals"], ref.cycle_residuals):
        assert abs(rg - ro) <= 1e-9
    r = info["rank"]
    assert lowrank_rel_diff(U[:, :r], V[:, :r], ref.U, ref.V) <= 1e-8
    ctx.close()
