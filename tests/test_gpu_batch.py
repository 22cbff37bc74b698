"""batched lockstep solve of several parameter subsets (Algorithm 1's loop over
the subsets; the subsets are independent given the operator): one fused SpMM
pass per iteration reads the operator once for all subsets' U factors.

Parity: every subset of a batched solve equals its own single-subset solve (same kernels per subset,
so equal up to the reduction order of the persistent Gram partials: <= 1e-12) and the CPU oracle
(rel. Frobenius <= 1e-8, |d rho| <= 1e-9, ranks equal except near-ties)."""
import os
import sys

import numpy as np
import pytest

from oracle import chebyshevt as orc
from gpu_common import lowrank_rel_diff, near_tie, oracle_terms, problem, require_gpu, torch

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _contexts(prob, subsets):
    from paper_2008_10275_b200 import lrcheb
    op = prob.op
    dev = torch.device("cuda:0")
    rp, ci = torch.from_numpy(op.row_ptr).to(dev), torch.from_numpy(op.col_idx).to(dev)
    vals = [torch.from_numpy(v).to(dev) for v in op.vals]
    ctxs, ins = [], []
    for k in subsets:
        c = lrcheb.Context(0)
        c.set_operator(rp, ci, vals, op.rho_f, op.lambda_s, borrow=True)
        d_mu, d_nu, BU, BV = prob.subset(k)
        c.set_params(d_mu, d_nu)
        ctxs.append(c)
        ins.append((d_mu, d_nu, BU, BV))
    return ctxs, ins, (rp, ci, vals)


@pytest.mark.parametrize("name,subsets", [("small", (0, 1, 2)), ("tiny", (0, 0)), ("medium", (0, 3))])
def test_batched_solve_matches_single_and_oracle(name, subsets):
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    prob = problem(name)
    cfg, op = prob.cfg, prob.op
    N = cfg.n_iter
    ctxs, ins, keep = _contexts(prob, subsets)
    bus = [torch.from_numpy(x[2]).cuda() for x in ins]
    bvs = [torch.from_numpy(x[3]).cuda() for x in ins]
    for rep in range(2):                 # the second call replays the cached batch graph
        res = lrcheb.solve_batch(ctxs, bus, bvs, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, N)
    torch.cuda.synchronize()
    for q, (U, V, info) in enumerate(res):
        d_mu, d_nu, BU, BV = ins[q]
        # the same subset alone
        Us, Vs, infs = ctxs[q].solve(bus[q], bvs[q], prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, N)
        r, rs = info["rank"], infs["rank"]
        assert info["rank_history"] == infs["rank_history"]
        Uh, Vh, Ush, Vsh = (x.cpu().numpy() for x in (U, V, Us, Vs))
        assert lowrank_rel_diff(Uh[:, :r], Vh[:, :r], Ush[:, :rs], Vsh[:, :rs]) <= 1e-12
        assert abs(info["rel_residual"] - infs["rel_residual"]) <= 1e-12
        if name == "medium":
            # Medium: the oracle's whole solve is in tests/golden/medium_s0.npz (written by
            # tests/golden/make_goldens.py from oracle/ only); the other subset is held to its own
            # single-subset solve above
            if subsets[q] == 0:
                _check_medium_golden(prob, info, Uh, Vh)
            continue
        # the oracle
        ref = orc.chebyshevt(oracle_terms(op, d_mu, d_nu), BU, BV, prob.lam_min, prob.lam_max, cfg.tol,
                             cfg.rank_cap, N, record_iterates=False)
        for k in range(N):
            rk, ro = info["rank_history"][k], ref.ranks[k]
            assert rk == ro or near_tie(ref.sigmas[k], cfg.tol, cfg.rank_cap, ro), (k, rk, ro)
        assert lowrank_rel_diff(Uh[:, :r], Vh[:, :r], ref.U, ref.V) <= 1e-8
        assert abs(info["rel_residual"] - ref.rel_residual) <= 1e-9
    for c in ctxs:
        c.close()


def _check_medium_golden(prob, info, U, V):
    sys.path.insert(0, GOLDEN)
    import make_goldens
    g = np.load(os.path.join(GOLDEN, "medium_s0.npz"))
    d_mu, d_nu, BU, BV = prob.subset(0)
    assert make_goldens.same_inputs(g["signature"], make_goldens.signature(prob.op, d_mu, d_nu, BU, BV,
                                                                          prob.lam_min, prob.lam_max))
    cfg = prob.cfg
    for k, (rk, ro) in enumerate(zip(info["rank_history"], g["ranks"])):
        assert rk == ro or near_tie(g["sigmas"][k], cfg.tol, cfg.rank_cap, int(ro)), (k + 1, rk, int(ro))
    rows, rg = g["rows"], int(g["ranks"][-1])
    Xg = g["U_ck"][-1][:, :rg] @ g["V_ck"][-1][:, :rg].T
    r = info["rank"]
    X = U[rows][:, :r] @ V[:, :r].T
    assert np.linalg.norm(X - Xg) / np.linalg.norm(Xg) <= 1e-8
    assert abs(info["rel_residual"] - float(g["rel_residual"])) <= 1e-9


def test_batched_solve_rejects_unshared_operator():
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    prob = problem("tiny")
    op = prob.op
    ctxs, ins, keep = _contexts(prob, (0,))
    other = lrcheb.Context(0)
    other.set_operator(op.row_ptr, op.col_idx, op.vals, op.rho_f, op.lambda_s)      # its own copy
    other.set_params(ins[0][0], ins[0][1])
    bu = torch.from_numpy(ins[0][2]).cuda()
    bv = torch.from_numpy(ins[0][3]).cuda()
    with pytest.raises(lrcheb.LrcError) as e:
        lrcheb.solve_batch([ctxs[0], other], [bu, bu], [bv, bv], prob.lam_min, prob.lam_max, 1e-8, 4, 3)
    assert e.value.status == lrcheb.LRC_ERR_ARG
    other.close()
    ctxs[0].close()
