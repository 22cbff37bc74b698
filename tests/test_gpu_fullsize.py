"""Full-size parity on the configurations the bench measures (BASELINE.json north_star: "GPU
ChebyshevT results match the oracle within the stated tolerances on all five configs"; operator
PAPER.md P:30-36, truncation P:544).

* Large (configs[3]), subsets 0 and 1, all N = 100 iterations through the C ABI, against goldens written by
  tests/golden/make_goldens.py (oracle/ + synth/ only): every rank (near-tie exemption S13), every
  core singular-value vector, X_k on 512 seeded rows at k = 10, 20, ..., 100 (rel. Frobenius <= 1e-8),
  and the final residual (|d rho| <= 1e-9).
* Large in the exact bench launch configuration: 3 contexts on 3 streams / host threads, borrowed
  operator, 3 reserved SMs, subsets 0, 1, 2 concurrently -> X_N rows and rho of each subset.
* Medium (configs[2]) subset 0: all 80 iterations, every X_k on 256 sampled rows against the golden
  (tests/golden/medium_s0.npz; the live oracle when the file is absent).
* Config 5 (configs[4]): the dense M x 256 application on the Large operator, compared with the
  oracle's apply_dense on a seeded block of rows (the oracle restricted to rows R computes
  sum_t c_t A_t[R, :] S diag(e_t) -- the same formula, fewer rows).
"""
import os
import sys
import threading

import numpy as np
import pytest

from oracle import chebyshevt as orc
from gpu_common import lowrank_rel_diff, make_ctx, near_tie, oracle_terms, problem, require_gpu, torch

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
sys.path.insert(0, GOLDEN)
import make_goldens  # noqa: E402  (input signature / row sampling of the golden files)


def _golden(name, subset):
    path = os.path.join(GOLDEN, f"{name}_s{subset}.npz")
    assert os.path.exists(path), f"missing golden {path}: run tests/golden/make_goldens.py {name} {subset}"
    g = np.load(path)
    prob = problem(name)
    d_mu, d_nu, BU, BV = prob.subset(subset)
    sig = make_goldens.signature(prob.op, d_mu, d_nu, BU, BV, prob.lam_min, prob.lam_max)
    assert make_goldens.same_inputs(g["signature"], sig), "golden was written for different inputs (synth/ changed?)"
    return g


def _rows_rel(U, V, r, Ug, Vg, rg, rows):
    """||X[rows] - X_golden[rows]||_F / ||X_golden[rows]||_F."""
    Xg = Ug[:, :rg] @ Vg[:, :rg].T
    X = U[rows][:, :r] @ V[:, :r].T
    return np.linalg.norm(X - Xg) / np.linalg.norm(Xg)


def _check_ranks(ranks, g, tol, cap):
    for k, (rk, ro) in enumerate(zip(ranks, g["ranks"])):
        assert rk == ro or near_tie(g["sigmas"][k], tol, cap, int(ro)), (k + 1, rk, int(ro))


@pytest.fixture(scope="module")
def large_dev():
    prob = problem("large")
    op = prob.op
    dev = torch.device("cuda:0")
    rp, ci = torch.from_numpy(op.row_ptr).to(dev), torch.from_numpy(op.col_idx).to(dev)
    vals = [torch.from_numpy(v).to(dev) for v in op.vals]
    yield prob, rp, ci, vals
    del rp, ci, vals
    torch.cuda.empty_cache()


@pytest.mark.parametrize("subset", [0, 1])
def test_large_all_iterations_vs_golden(large_dev, subset):
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    prob, rp, ci, vals = large_dev
    cfg, op = prob.cfg, prob.op
    g = _golden("large", subset)
    d_mu, d_nu, BU, BV = prob.subset(subset)
    ctx = lrcheb.Context(0)
    ctx.set_operator(rp, ci, vals, op.rho_f, op.lambda_s, borrow=True)
    ctx.set_params(d_mu, d_nu)
    bu, bv = torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda()
    N, cap, tol = cfg.n_iter, cfg.rank_cap, cfg.tol
    U, V, info = ctx.solve(bu, bv, prob.lam_min, prob.lam_max, tol, cap, N, record_iterates=True)
    _check_ranks(info["rank_history"], g, tol, cap)
    # core singular values of every truncation (GPU: shift-compensated CholeskyQR2 + Jacobi; oracle:
    # Householder + LAPACK SVD) -- within 1e-10 sigma_1 (R8 derives 1e-11 for one truncation;
    # 10x margin for the 100-step trajectory)
    S = info["sigma_history"]
    for k in range(N):
        so = g["sigmas"][k]
        m = int(min(np.count_nonzero(so), np.count_nonzero(S[k]), 100))
        assert np.max(np.abs(S[k][:m] - so[:m])) <= 1e-10 * so[0], k + 1
    rows = g["rows"]
    worst = 0.0
    for c, k in enumerate(g["ck"]):
        Uk, Vk, rk = ctx.get_iterate(int(k), cap)
        err = _rows_rel(Uk, Vk, rk, g["U_ck"][c], g["V_ck"][c], int(g["ranks"][k - 1]), rows)
        worst = max(worst, err)
        assert err <= 1e-8, (int(k), err)
    assert abs(info["rel_residual"] - float(g["rel_residual"])) <= 1e-9, (info["rel_residual"], float(g["rel_residual"]))
    Uh, Vh = U.cpu().numpy(), V.cpu().numpy()
    assert _rows_rel(Uh, Vh, info["rank"], g["U_ck"][-1], g["V_ck"][-1], int(g["ranks"][-1]), rows) <= 1e-8
    print(f"large s{subset}: worst checkpoint rel err {worst:.2e}, rho {info['rel_residual']:.6e} "
          f"(oracle {float(g['rel_residual']):.6e})")
    ctx.close()


def test_large_bench_configuration_concurrent(large_dev):
    """The bench's launch configuration (bench.py main): S = 3 contexts, each with its own CUDA
    stream and host thread, all borrowing one device copy of the operator, 3 SMs reserved."""
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    prob, rp, ci, vals = large_dev
    cfg, op = prob.cfg, prob.op
    subsets = [k for k in (0, 1, 2) if os.path.exists(os.path.join(GOLDEN, f"large_s{k}.npz"))]
    assert 0 in subsets
    S = 3
    ctxs, outs, ins = [], [], []
    for i in range(S):
        c = lrcheb.Context(0)
        c.set_reserved_sms(3)
        c.set_operator(rp, ci, vals, op.rho_f, op.lambda_s, borrow=True)
        ctxs.append(c)
        k = (0, 1, 2)[i]
        d_mu, d_nu, BU, BV = prob.subset(k)
        ins.append((k, d_mu, d_nu, torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda()))
        outs.append((torch.empty((op.M, cfg.rank_cap), dtype=torch.float64, device="cuda"),
                     torch.empty((len(d_mu), cfg.rank_cap), dtype=torch.float64, device="cuda")))
    infos = [None] * S
    errs = []

    def worker(i):
        try:
            k, d_mu, d_nu, bu, bv = ins[i]
            ctxs[i].set_params(d_mu, d_nu)
            for _ in range(2):      # twice: the second solve replays the captured CUDA graph
                infos[i] = ctxs[i].solve(bu, bv, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, cfg.n_iter,
                                         out=outs[i])[2]
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ths = [threading.Thread(target=worker, args=(i,)) for i in range(S)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    torch.cuda.synchronize()
    checked = 0
    for i in range(S):
        k = ins[i][0]
        if k not in subsets:
            continue
        g = _golden("large", k)
        info = infos[i]
        _check_ranks(info["rank_history"], g, cfg.tol, cfg.rank_cap)
        U, V = outs[i][0].cpu().numpy(), outs[i][1].cpu().numpy()
        err = _rows_rel(U, V, info["rank"], g["U_ck"][-1], g["V_ck"][-1], int(g["ranks"][-1]), g["rows"])
        assert err <= 1e-8, (k, err)
        assert abs(info["rel_residual"] - float(g["rel_residual"])) <= 1e-9, (k, info["rel_residual"])
        checked += 1
    assert checked >= 1
    for c in ctxs:
        c.close()


def test_medium_every_iteration():
    """Medium subset 0, all N = 80 iterations: every X_k on the golden's 256 sampled rows, every rank and
    core singular-value vector (tests/golden/medium_s0.npz, written by the oracle); without the golden
    file the same comparison runs against the live oracle (~11 min)."""
    require_gpu()
    prob = problem("medium")
    cfg, op = prob.cfg, prob.op
    d_mu, d_nu, BU, BV = prob.subset(0)
    ctx = make_ctx(op, d_mu, d_nu)
    N, cap, tol = cfg.n_iter, cfg.rank_cap, cfg.tol
    _, _, info = ctx.solve(torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda(), prob.lam_min, prob.lam_max,
                           tol, cap, N, record_iterates=True)
    if os.path.exists(os.path.join(GOLDEN, "medium_s0.npz")):
        g = _golden("medium", 0)
        assert list(g["ck"]) == list(range(1, N + 1))
        _check_ranks(info["rank_history"], g, tol, cap)
        S = info["sigma_history"]
        worst = 0.0
        for k in range(1, N + 1):
            so = g["sigmas"][k - 1]
            m = int(min(np.count_nonzero(so), np.count_nonzero(S[k - 1]), 100))
            assert np.max(np.abs(S[k - 1][:m] - so[:m])) <= 1e-10 * so[0], k
            Uk, Vk, rk = ctx.get_iterate(k, cap)
            err = _rows_rel(Uk, Vk, rk, g["U_ck"][k - 1], g["V_ck"][k - 1], int(g["ranks"][k - 1]), g["rows"])
            worst = max(worst, err)
            assert err <= 1e-8, (k, err)
        assert abs(info["rel_residual"] - float(g["rel_residual"])) <= 1e-9
        print(f"medium s0 (golden): worst iterate rel err on sampled rows {worst:.2e}")
        ctx.close()
        return
    terms = oracle_terms(op, d_mu, d_nu)
    Uk_prev = {}

    def check(k, Uo, Vo, s):
        Uk, Vk, rk = ctx.get_iterate(k, cap)
        assert rk == Uo.shape[1] or near_tie(s, tol, cap, Uo.shape[1]), (k, rk, Uo.shape[1])
        assert info["rank_history"][k - 1] == rk
        err = lowrank_rel_diff(Uk[:, :rk], Vk[:, :rk], Uo, Vo)
        Uk_prev["worst"] = max(Uk_prev.get("worst", 0.0), err)
        assert err <= 1e-8, (k, err)

    ref = orc.chebyshevt(terms, BU, BV, prob.lam_min, prob.lam_max, tol, cap, N, record_iterates=False,
                         on_iterate=check)
    assert abs(info["rel_residual"] - ref.rel_residual) <= 1e-9, (info["rel_residual"], ref.rel_residual)
    print(f"medium s0: worst iterate rel err {Uk_prev['worst']:.2e}")
    ctx.close()


def test_config5_dense_on_large_operator(large_dev):
    """BASELINE configs[4]: Y = sum_t c_t A_t S D_t with S = M x 256 N(0,1) (synth dense_factor),
    D_mu / D_nu from the 16 x 16 parameter grid, at the full Large size in the bench's call."""
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    from synth import generator as gen
    prob, rp, ci, vals = large_dev
    op = prob.op
    cfg5 = gen.config_by_name("fullrank")
    mu5, nu5 = gen.parameter_grid(cfg5)
    ncols = cfg5.dense_cols
    S = gen.dense_factor(cfg5, op.M, ncols)
    ctx = lrcheb.Context(0)
    ctx.set_operator(rp, ci, vals, op.rho_f, op.lambda_s, borrow=True)
    ctx.set_params(mu5, nu5)
    Sd = torch.from_numpy(S).cuda()
    Y = ctx.apply_dense(Sd).cpu().numpy()
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([np.arange(0, 4096), np.arange(op.M - 2048, op.M),
                                     rng.choice(op.M, 2048, replace=False)]))
    terms = oracle_terms(op, mu5, nu5)
    sub = [(c, A[rows], e) for (c, A, e) in terms]
    ref = orc.apply_dense(sub, S)
    err = np.linalg.norm(Y[rows] - ref) / np.linalg.norm(ref)
    assert err <= 1e-12, err
    ctx.close()


def test_large_lockstep_groups_concurrent(large_dev):
    """f1 in the bench's group form (bench.py --batch 3 --groups 2): two lockstep groups of three
    subsets (lrc_solve_batch, one batched SpMM per iteration each) on their own host threads, contexts
    and streams, 3 SMs reserved -> every subset's X_N rows and rho against the oracle goldens."""
    require_gpu()
    from paper_2008_10275_b200 import lrcheb
    prob, rp, ci, vals = large_dev
    cfg, op = prob.cfg, prob.op
    groups = [(0, 1, 2), (2, 1, 0)]
    ctxs, ins, outs = [], [], []
    for grp in groups:
        cg, ig, og = [], [], []
        for k in grp:
            c = lrcheb.Context(0)
            c.set_reserved_sms(3)
            c.set_operator(rp, ci, vals, op.rho_f, op.lambda_s, borrow=True)
            d_mu, d_nu, BU, BV = prob.subset(k)
            c.set_params(d_mu, d_nu)
            cg.append(c)
            ig.append((k, torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda()))
            og.append((torch.empty((op.M, cfg.rank_cap), dtype=torch.float64, device="cuda"),
                       torch.empty((len(d_mu), cfg.rank_cap), dtype=torch.float64, device="cuda")))
        ctxs.append(cg); ins.append(ig); outs.append(og)
    results = [None, None]
    errs = []

    def worker(gi):
        try:
            for _ in range(2):      # the second call replays the captured batch graph
                results[gi] = lrcheb.solve_batch(ctxs[gi], [x[1] for x in ins[gi]], [x[2] for x in ins[gi]],
                                                 prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, cfg.n_iter,
                                                 outs=outs[gi])
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ths = [threading.Thread(target=worker, args=(gi,)) for gi in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    torch.cuda.synchronize()
    checked = 0
    for gi in range(2):
        for j, (k, _, _) in enumerate(ins[gi]):
            if not os.path.exists(os.path.join(GOLDEN, f"large_s{k}.npz")):
                continue
            g = _golden("large", k)
            U, V, info = results[gi][j]
            _check_ranks(info["rank_history"], g, cfg.tol, cfg.rank_cap)
            err = _rows_rel(U.cpu().numpy(), V.cpu().numpy(), info["rank"], g["U_ck"][-1], g["V_ck"][-1],
                            int(g["ranks"][-1]), g["rows"])
            assert err <= 1e-8, (gi, k, err)
            assert abs(info["rel_residual"] - float(g["rel_residual"])) <= 1e-9, (gi, k, info["rel_residual"])
            checked += 1
    assert checked >= 2
    for cg in ctxs:
        for c in cg:
            c.close()
