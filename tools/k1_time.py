"""Developer probe: median device time of the fused SpMM (S2STEP, r = cap) on a config's operator,
for the library selected by LRCHEB_LIB (experimental variants) or the default build."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2008_10275_b200 import lrcheb  # noqa: E402
from synth import generator as gen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
prob = gen.make_problem(name)
op, cfg = prob.op, prob.cfg
dev = torch.device("cuda:0")
ctx = lrcheb.Context(0)
ctx.set_operator(torch.from_numpy(op.row_ptr).to(dev), torch.from_numpy(op.col_idx).to(dev),
                 [torch.from_numpy(v).to(dev) for v in op.vals], op.rho_f, op.lambda_s)
d_mu, d_nu, _, _ = prob.subset(0)
ctx.set_params(d_mu, d_nu)
r = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.rank_cap
U = torch.randn(op.M, r, dtype=torch.float64, device=dev)
for _ in range(3):
    ctx.apply_lowrank(U, lrcheb.LRC_APPLY_S2STEP, 0.1)
ms = []
for _ in range(10):
    ctx.apply_lowrank(U, lrcheb.LRC_APPLY_S2STEP, 0.1)
    ms.append(ctx.last_kernel_ms())
byts = 52 * op.nnz + 4 * (op.M + 1) + 32 * op.M * r
t = float(np.median(ms))
print(f"{os.path.basename(os.environ.get('LRCHEB_LIB', 'liblrcheb.so'))}: K1 {name} r={r}: {t:.3f} ms "
      f"{byts / t / 1e6:.0f} GB/s", flush=True)
