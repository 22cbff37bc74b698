"""Debug probe for the rank-deficient truncation case (test_truncate[30-16-1e-12-True])."""
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2008_10275_b200 import lrcheb  # noqa
from synth import generator as gen  # noqa
from oracle import chebyshevt as orc  # noqa

prob = gen.make_problem("tiny")
op = prob.op
for (w, cap, tau, defic) in [(30, 16, 1e-12, True), (40, 10, 1e-8, False), (100, 20, 1e-10, False)]:
    n = 16 if w <= 40 else 40
    rng = np.random.default_rng(w + cap)
    d_mu, d_nu = rng.random(n) + 0.5, rng.random(n) + 0.5
    ctx = lrcheb.Context(0)
    ctx.set_operator(op.row_ptr, op.col_idx, op.vals, op.rho_f, op.lambda_s)
    ctx.set_params(d_mu, d_nu)
    U = rng.standard_normal((op.M, w)) * np.logspace(0, -9, w)[None, :]
    if defic:
        U[:, w // 2:] = U[:, : w - w // 2]
    V = rng.standard_normal((n, w))
    Ug, Vg, rg, sg = ctx.truncate(U, V, tau, cap)
    Uo, Vo, so = orc.truncate(U, V, tau, cap)
    print(f"w={w} cap={cap} tau={tau} def={defic}: rank gpu {rg} oracle {Uo.shape[1]}")
    print("  sigma gpu/oracle rel:", np.array2string(sg[:min(len(sg), len(so))] / so[0], precision=3, max_line_width=200))
    print("  oracle             :", np.array2string(so / so[0], precision=3, max_line_width=200))
    G = Ug[:, :rg].T @ Ug[:, :rg]
    print("  diag(U^T U):", np.array2string(np.diag(G), precision=4, max_line_width=200))
    print("  ||UtU-I||", np.linalg.norm(G - np.eye(rg)))
    ctx.close()
