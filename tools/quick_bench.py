"""Developer timing probe (not the contract bench): per-kernel-class timings on one config."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2008_10275_b200 import lrcheb  # noqa: E402
from synth import generator as gen  # noqa: E402


def main(name="large", N=20):
    t0 = time.time()
    prob = gen.make_problem(name)
    print(f"generate {name}: {time.time() - t0:.1f}s  M={prob.op.M} nnz={prob.op.nnz} "
          f"bounds=[{prob.lam_min:.4f},{prob.lam_max:.4f}]", flush=True)
    cfg, op = prob.cfg, prob.op
    d_mu, d_nu, BU, BV = prob.subset(0)
    dev = torch.device("cuda:0")
    ctx = lrcheb.Context(0)
    ctx.set_operator(torch.from_numpy(op.row_ptr).to(dev), torch.from_numpy(op.col_idx).to(dev),
                     [torch.from_numpy(v).to(dev) for v in op.vals], op.rho_f, op.lambda_s)
    ctx.set_params(d_mu, d_nu)
    r = cfg.rank_cap
    U = torch.randn(op.M, r, dtype=torch.float64, device=dev)
    for _ in range(3):
        ctx.apply_lowrank(U, lrcheb.LRC_APPLY_S2STEP, 0.1)
    ms = []
    for _ in range(5):
        ctx.apply_lowrank(U, lrcheb.LRC_APPLY_S2STEP, 0.1)
        ms.append(ctx.last_kernel_ms())
    byts = 52 * op.nnz + 4 * (op.M + 1) + 32 * op.M * r
    t = float(np.median(ms))
    print(f"K1 S2STEP r={r}: {t:.3f} ms  {byts / t / 1e6:.0f} GB/s  ({byts / 1e9:.3f} GB)", flush=True)
    bu, bv = torch.from_numpy(BU).to(dev), torch.from_numpy(BV).to(dev)
    for it in range(3):
        Uo, Vo, info = ctx.solve(bu, bv, prob.lam_min, prob.lam_max, cfg.tol, r, N, skip_residual=(it < 2))
        print(f"solve N={N}: iters {info['ms_iterations']:.2f} ms ({info['ms_iterations'] / N:.3f} ms/it) "
              f"total {info['ms_total']:.2f} ms ranks {info['rank_history'][:6]}..{info['rank_history'][-1]} "
              f"rho={info['rel_residual']:.3e} esc={info['shift_escalations']}", flush=True)




def profile(name="large", N=20, warm=True):
    prob = gen.make_problem(name)
    cfg, op = prob.cfg, prob.op
    d_mu, d_nu, BU, BV = prob.subset(0)
    dev = torch.device("cuda:0")
    ctx = lrcheb.Context(0)
    ctx.set_operator(torch.from_numpy(op.row_ptr).to(dev), torch.from_numpy(op.col_idx).to(dev),
                     [torch.from_numpy(v).to(dev) for v in op.vals], op.rho_f, op.lambda_s)
    ctx.set_params(d_mu, d_nu)
    bu, bv = torch.from_numpy(BU).to(dev), torch.from_numpy(BV).to(dev)
    ctx.solve(bu, bv, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, N, warm_start=warm)
    _, _, info = ctx.solve(bu, bv, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, N, warm_start=warm)
    print(f"[{name} warm={warm}] graph solve N={N}: {info['ms_iterations'] / N:.3f} ms/it, sweeps/it "
          f"{info['jacobi_sweeps'] / N:.1f}, rho={info['rel_residual']:.3e} chol2 cycles/it (chol+R, jacobi, out) "
          f"{[round(c / N) for c in info['chol2_cycles']]}", flush=True)
    ctx.set_profiling(True)
    ctx.solve(bu, bv, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, N, warm_start=warm)
    prof = ctx.profile()
    ctx.set_profiling(False)
    for k, (ms, cnt) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        if cnt:
            print(f"   {k:12s} {ms:9.2f} ms total  {cnt:5d} launches  {ms / cnt:8.4f} ms avg", flush=True)


def dense(reps=10):
    """Config 5: the dense M x 256 application on the Large operator (CUDA-event kernel time)."""
    prob = gen.make_problem("large")
    op = prob.op
    dev = torch.device("cuda:0")
    cfg5 = gen.config_by_name("fullrank")
    mu5, nu5 = gen.parameter_grid(cfg5)
    ctx = lrcheb.Context(0)
    ctx.set_operator(torch.from_numpy(op.row_ptr).to(dev), torch.from_numpy(op.col_idx).to(dev),
                     [torch.from_numpy(v).to(dev) for v in op.vals], op.rho_f, op.lambda_s)
    ctx.set_params(mu5, nu5)
    S5 = torch.randn((op.M, cfg5.dense_cols), dtype=torch.float64, device=dev)
    for _ in range(3):
        ctx.apply_dense(S5)
    ms = []
    for _ in range(reps):
        ctx.apply_dense(S5)
        ms.append(ctx.last_kernel_ms())
    t = float(np.median(ms))
    fl = 6.0 * op.nnz * cfg5.dense_cols
    print(f"config5 dense: {t:.3f} ms  {fl / t / 1e9:.2f} TFLOP/s", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "dense":
        dense()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "profile":
        for nm in sys.argv[2:] or ["large"]:
            for warm in (True, False):
                profile(nm, {"tiny": 30, "small": 50, "medium": 80, "large": 100}[nm], warm)
    else:
        main(sys.argv[1] if len(sys.argv) > 1 else "large", int(sys.argv[2]) if len(sys.argv) > 2 else 20)
