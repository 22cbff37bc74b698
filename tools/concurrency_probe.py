"""Probe: throughput of S concurrent subset solves (S contexts / streams / host threads)."""
import sys
import threading
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2008_10275_b200 import lrcheb  # noqa
from synth import generator as gen  # noqa

prob = gen.make_problem(sys.argv[1] if len(sys.argv) > 1 else "large")
cfg, op = prob.cfg, prob.op
dev = torch.device("cuda:0")
rp, ci = torch.from_numpy(op.row_ptr).to(dev), torch.from_numpy(op.col_idx).to(dev)
vals = [torch.from_numpy(v).to(dev) for v in op.vals]
subs = []
for k in range(cfg.K):
    d_mu, d_nu, BU, BV = prob.subset(k)
    subs.append((d_mu, d_nu, torch.from_numpy(BU).to(dev), torch.from_numpy(BV).to(dev)))
N = cfg.n_iter
for S, reserve in [(1, 0), (2, 0), (2, 2), (2, 4), (3, 3)]:
    ctxs = []
    for i in range(S):
        c = lrcheb.Context(0)
        c.set_reserved_sms(reserve)
        c.set_operator(rp, ci, vals, op.rho_f, op.lambda_s, borrow=True)
        ctxs.append(c)
    torch.cuda.synchronize()

    def run(i, nsolve):
        c = ctxs[i]
        for j in range(nsolve):
            d_mu, d_nu, bu, bv = subs[(i + j * S) % cfg.K]
            c.set_params(d_mu, d_nu)
            c.solve(bu, bv, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, N, skip_residual=True)

    ths = [threading.Thread(target=run, args=(i, 1)) for i in range(S)]   # warm-up (graph capture)
    [t.start() for t in ths]; [t.join() for t in ths]
    torch.cuda.synchronize()
    per = 4
    t0 = time.perf_counter()
    ths = [threading.Thread(target=run, args=(i, per)) for i in range(S)]
    [t.start() for t in ths]; [t.join() for t in ths]
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"S={S} reserve={reserve}: {S * per * N / dt:.1f} it/s ({dt / (S * per) * 1e3:.0f} ms per solve)", flush=True)
    for c in ctxs:
        c.close()
