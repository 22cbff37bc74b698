"""Print the steady-state core singular-value profile of a config (developer probe)."""
import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2008_10275_b200 import lrcheb  # noqa
from synth import generator as gen  # noqa
name = sys.argv[1] if len(sys.argv) > 1 else "large"
prob = gen.make_problem(name)
cfg, op = prob.cfg, prob.op
d_mu, d_nu, BU, BV = prob.subset(0)
ctx = lrcheb.Context(0)
ctx.set_operator(op.row_ptr, op.col_idx, op.vals, op.rho_f, op.lambda_s)
ctx.set_params(d_mu, d_nu)
_, _, info = ctx.solve(BU, BV, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, cfg.n_iter)
S = info["sigma_history"]
for k in (5, 20, cfg.n_iter - 1):
    s = S[k]
    s = s[s > 0] / s[0]
    print(name, "iter", k + 1, "p_nonzero", len(s), "sigma/sigma1 at", [(i, f"{s[i]:.1e}") for i in range(0, len(s), 10)],
          "last", f"{s[-1]:.1e}")
print("ranks", info["rank_history"][:8], "...", info["rank_history"][-1], "sweeps/it", info["jacobi_sweeps"] / cfg.n_iter)
