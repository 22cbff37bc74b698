"""Developer probe: per-kernel times of one Large solve (profiled, no graph) with phases of the
tall-skinny kernels switched off (LRCHEB_TS_DBG bits: 1 no copies, 2 no Gram / store epilogue,
4 no phase-A DMMA).  Results are garbage when bits are set; only the timings matter.  Each setting
runs in its own process."""
import os
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])


def measure(cfg, N):
    import torch
    from paper_2008_10275_b200 import lrcheb
    from synth import generator as gen
    prob = gen.make_problem(cfg)
    op, c = prob.op, prob.cfg
    d_mu, d_nu, BU, BV = prob.subset(0)
    dev = torch.device("cuda:0")
    ctx = lrcheb.Context(0)
    ctx.set_operator(torch.from_numpy(op.row_ptr).to(dev), torch.from_numpy(op.col_idx).to(dev),
                     [torch.from_numpy(v).to(dev) for v in op.vals], op.rho_f, op.lambda_s)
    ctx.set_params(d_mu, d_nu)
    bu, bv = torch.from_numpy(BU).to(dev), torch.from_numpy(BV).to(dev)
    # reference ranks: a clean solve first (the truncation of a garbage run would pick other ranks)
    ctx.solve(bu, bv, prob.lam_min, prob.lam_max, c.tol, c.rank_cap, N)
    ctx.set_profiling(True)
    ctx.solve(bu, bv, prob.lam_min, prob.lam_max, c.tol, c.rank_cap, N, no_graph=True)
    prof = ctx.profile()
    print("  ".join(f"{k} {ms / cnt:.3f}" for k, (ms, cnt) in sorted(prof.items()) if cnt and k.startswith("ts_")),
          flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "once":
        measure(sys.argv[2], int(sys.argv[3]))
        sys.exit(0)
    cfg = sys.argv[1] if len(sys.argv) > 1 else "large"
    for dbg in [int(x) for x in sys.argv[2:]] or [0, 1, 2, 4, 6, 3, 5, 7]:
        env = dict(os.environ, LRCHEB_TS_DBG=str(dbg))
        out = subprocess.run([sys.executable, __file__, "once", cfg, "20"], env=env, capture_output=True, text=True)
        print(f"dbg={dbg}: {out.stdout.strip() or out.stderr.strip()[-300:]}", flush=True)
