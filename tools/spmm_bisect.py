"""Developer probe: K1 S2STEP time on one config with phases of the SpMM switched off
(LRCHEB_SPMM_DBG bits: 1 no DMMA, 2 no U staging, 4 no value loads, 8 no stores; 32 = warp-specialised
kernel, 64 = persistent 2-CTA kernel, 128 = deep-prefetch kernel).
Each setting runs in its own process (the switch is read once per process).

    python tools/spmm_bisect.py large 0 15 9      # settings to compare
    python tools/spmm_bisect.py once large        # one measurement in this process (e.g. under ncu)
"""
import os
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])


def measure(cfg):
    import numpy as np
    import torch
    from paper_2008_10275_b200 import lrcheb
    from synth import generator as gen
    prob = gen.make_problem(cfg)
    op = prob.op
    d_mu, d_nu, BU, BV = prob.subset(0)
    dev = torch.device("cuda:0")
    ctx = lrcheb.Context(0)
    ctx.set_operator(torch.from_numpy(op.row_ptr).to(dev), torch.from_numpy(op.col_idx).to(dev),
                     [torch.from_numpy(v).to(dev) for v in op.vals], op.rho_f, op.lambda_s)
    ctx.set_params(d_mu, d_nu)
    r = prob.cfg.rank_cap
    U = torch.randn(op.M, r, dtype=torch.float64, device=dev)
    for _ in range(3):
        ctx.apply_lowrank(U, lrcheb.LRC_APPLY_S2STEP, 0.1)
    ms = []
    for _ in range(7):
        ctx.apply_lowrank(U, lrcheb.LRC_APPLY_S2STEP, 0.1)
        ms.append(ctx.last_kernel_ms())
    byts = 52 * op.nnz + 4 * (op.M + 1) + 32 * op.M * r
    t = float(np.median(ms))
    print(f"{t:.3f} ms {byts / t / 1e6:.0f} GB/s", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "once":
        measure(sys.argv[2])
        sys.exit(0)
    cfg = sys.argv[1] if len(sys.argv) > 1 else "large"
    settings = [int(x) for x in sys.argv[2:]] or [0, 1, 8, 9, 2, 4, 6, 14, 15, 32]
    for dbg in settings:
        env = dict(os.environ, LRCHEB_SPMM_DBG=str(dbg & 31))
        if dbg & 32:
            env["LRCHEB_SPMM_TMA"] = "1"
        if dbg & 64:
            env["LRCHEB_SPMM_PERSIST"] = "1"
        if dbg & 128:
            env["LRCHEB_SPMM_DEEP"] = "1"
        out = subprocess.run([sys.executable, __file__, "once", cfg], env=env, capture_output=True, text=True)
        print(f"dbg={dbg:3d}: {out.stdout.strip() or out.stderr.strip()[-300:]}", flush=True)
