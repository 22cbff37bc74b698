"""Developer probe: one solve of a config (subset 0, N iterations) with timing, for hang/perf triage."""
import os
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2008_10275_b200 import lrcheb  # noqa: E402
from synth import generator as gen  # noqa: E402

name, N = sys.argv[1], int(sys.argv[2])
prob = gen.make_problem(name)
cfg, op = prob.cfg, prob.op
d_mu, d_nu, BU, BV = prob.subset(0)
ctx = lrcheb.Context(0)
ctx.set_operator(op.row_ptr, op.col_idx, op.vals, op.rho_f, op.lambda_s)
ctx.set_params(d_mu, d_nu)
t = time.time()
_, _, info = ctx.solve(torch.from_numpy(BU).cuda(), torch.from_numpy(BV).cuda(), prob.lam_min, prob.lam_max, cfg.tol,
                       cfg.rank_cap, N, no_graph=("nograph" in sys.argv))
print(os.path.basename(os.environ.get("LRCHEB_LIB", "liblrcheb.so")), name, N, info["rank_history"], info["rel_residual"],
      f"{time.time() - t:.2f}s", flush=True)
