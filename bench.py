"""bench.py -- ChebyshevT iterations/s + fused-SpMM HBM GB/s on B200 (BASELINE.json `metric`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config large]

A "step" is one whole ChebyshevT solve of one parameter subset (all SURVEY §8(a) rows: N fused
SpMM + truncation iterations and the final residual) on the config's synthetic operator
(BASELINE.json configs[3] "Large" by default, the largest single-GPU
config).  value = (solved subsets x N iterations, all ranks) / max-over-ranks device seconds.
Multi-GPU: subsets are independent, sharded round-robin over ranks with no data-path
collective ("scaling": "weak"); torch.distributed is used for the barrier and the max-reduction
of the timing only.

--impl reference times the CPU oracle (oracle/, the deliberately slow fp64 NumPy/SciPy program)
on a bounded, row-sampled piece of the same workload (see cpu_sample()).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_DMMA_PEAK_TFLOPS = 37.1    # measured: tools/microbench/fp64_peaks.cu -> profiles/r01_phase0_fp64_peaks.jsonl
L2_BYTES = 132644864


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="large")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--streams", type=int, default=3, help="concurrent subset solves per GPU")
    ap.add_argument("--no-dense", dest="dense", action="store_false", help="skip the config-5 measurement")
    ap.add_argument("--reserve-sms", type=int, default=3, help="SMs the persistent kernels leave free")
    return ap.parse_args()


def shard_subsets(K: int, rank: int, world: int):
    """Subsets of this rank: round-robin over ranks (subsets are independent given the
    operator), at least one per rank so every rank does a step of work."""
    return [k for k in range(K) if k % world == rank] or [rank % K]


def max_over_ranks(ms: float, dist, device=None) -> float:
    """Max-over-ranks of a device time (the contract's timing rule); identity at world size 1."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return ms
    import torch
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline and --impl reference)
# ----------------------------------------------------------------------------------------------
def cpu_sample(prob, rows, rng_seed=1):
    """One steady-state ChebyshevT-S2 iteration of the oracle (literal six-term SpMM + Householder
    QR + LAPACK SVD truncation) restricted to the first `rows` rows of the operator: the six
    A_t[rows, :] U_k products, the concatenation's row block and its truncation.  Every oracle cost
    is linear in the number of rows, so iterations/s = (rows / M) / seconds."""
    import scipy.sparse as sp
    from oracle import chebyshevt as orc
    cfg, op = prob.cfg, prob.op
    d_mu, d_nu, BU, BV = prob.subset(0)
    r = cfg.rank_cap
    rng = np.random.default_rng(rng_seed)
    Uk = rng.standard_normal((op.M, r))
    Vk, Vkm1 = rng.standard_normal((len(d_mu), r)), rng.standard_normal((len(d_mu), r))
    Ukm1 = rng.standard_normal((rows, r))
    nnz_r = int(op.row_ptr[rows])
    mats = [sp.csr_matrix((v[:nnz_r], op.col_idx[:nnz_r], op.row_ptr[:rows + 1]), shape=(rows, op.M))
            for v in op.vals]
    terms = orc.term_list(mats, op.rho_f, op.lambda_s, d_mu, d_nu)
    c, d = orc.chebyshev_cd(prob.lam_min, prob.lam_max)
    gamma, omega = 1.0 / d, 1.3
    t0 = time.perf_counter()
    UL, VL = orc.apply_lowrank(terms, Uk, Vk)
    Ucat = np.hstack([BU[:rows], Uk[:rows], UL, Ukm1])
    Vcat = np.hstack([omega * gamma * BV, omega * Vk, -omega * gamma * VL, (1 - omega) * Vkm1])
    orc.truncate(Ucat, Vcat, cfg.tol, r)
    return time.perf_counter() - t0


def cpu_calibrate(prob, seconds):
    rows0 = min(prob.op.M, 32768)
    t0 = cpu_sample(prob, rows0)
    rows = int(min(prob.op.M, max(rows0, rows0 * seconds / max(t0, 1e-3))))
    rows -= rows % 5
    return rows


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------------------------
def main():
    args = parse()
    rank, world, local = dist_env()
    from synth import generator as gen

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2008_10275_b200 import lrcheb

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    prob = gen.make_problem(args.config)
    cfg, op = prob.cfg, prob.op
    N = cfg.n_iter
    # S concurrent subset solves (subsets are independent): one lrc context,
    # CUDA stream and host thread each, all sharing the borrowed operator.  The persistent M-level
    # kernels leave `reserve` SMs free so one solve's single-CTA core steps overlap the other's
    # M-level work.  Steps are dealt round-robin to the streams.
    S = max(1, args.streams)
    reserve = args.reserve_sms if S > 1 else 0
    rp_d, ci_d = torch.from_numpy(op.row_ptr).to(dev), torch.from_numpy(op.col_idx).to(dev)
    vals_d = [torch.from_numpy(v).to(dev) for v in op.vals]
    ctxs = []
    for _ in range(S):
        c = lrcheb.Context(local)
        c.set_reserved_sms(reserve)
        c.set_operator(rp_d, ci_d, vals_d, op.rho_f, op.lambda_s, borrow=True)
        ctxs.append(c)
    ctx = ctxs[0]
    my_subsets = shard_subsets(cfg.K, rank, world)
    inputs = []
    for k in my_subsets:
        d_mu, d_nu, BU, BV = prob.subset(k)
        inputs.append((d_mu, d_nu, torch.from_numpy(BU).to(dev), torch.from_numpy(BV).to(dev),
                       torch.from_numpy(BU).pin_memory(), torch.from_numpy(BV).pin_memory()))
    n = len(inputs[0][0])
    outs = [(torch.empty((op.M, cfg.rank_cap), dtype=torch.float64, device=dev),
             torch.empty((n, cfg.rank_cap), dtype=torch.float64, device=dev),
             torch.empty((op.M, cfg.rank_cap), dtype=torch.float64).pin_memory(),
             torch.empty((n, cfg.rank_cap), dtype=torch.float64).pin_memory()) for _ in range(S)]

    def step(i, host=False, c=None):
        si = (i % S) if c is None else c
        cx = ctxs[si]
        Uo, Vo, Uh, Vh = outs[si]
        d_mu, d_nu, bu, bv, bu_h, bv_h = inputs[i % len(inputs)]
        cx.set_params(d_mu, d_nu)
        if host:
            return cx.solve(bu_h, bv_h, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, N, out=(Uh, Vh))[2]
        return cx.solve(bu, bv, prob.lam_min, prob.lam_max, cfg.tol, cfg.rank_cap, N, out=(Uo, Vo))[2]

    def run_steps(nsteps, host):
        """nsteps solves dealt round-robin to the S streams, one host thread per stream."""
        infos = [None] * nsteps
        def worker(si):
            for i in range(si, nsteps, S):
                infos[i] = step(i, host, si)
        ths = [threading.Thread(target=worker, args=(si,)) for si in range(S)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return infos

    run_steps(max(args.warmup, S), False)           # >= 1 warm-up per stream (graph capture)
    main_s = torch.cuda.Stream(device=dev)

    def timed(host):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches0 = sum(c.kernel_launches() for c in ctxs)
        e0.record(main_s)
        for c in ctxs:
            c.stream.wait_event(e0)
        infos = run_steps(args.steps, host)
        for c in ctxs:
            ev = torch.cuda.Event()
            ev.record(c.stream)
            main_s.wait_event(ev)
        e1.record(main_s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        launches = sum(c.kernel_launches() for c in ctxs) - launches0
        ms = max_over_ranks(ms, dist if world > 1 else None, dev)
        if world > 1:
            dist.barrier()
        return ms, infos, launches

    clk = ClockSampler(local)
    clk.start()
    ms, infos, launches = timed(False)
    clocks = clk.stop()
    ms_e2e, _, _ = timed(True)
    iters = args.steps * N * world
    value = iters / (ms / 1e3)
    e2e_value = iters / (ms_e2e / 1e3)
    h2d = sum(inputs[i % len(inputs)][4].numel() * 8 + inputs[i % len(inputs)][5].numel() * 8
              for i in range(args.steps)) / args.steps
    d2h = (outs[0][2].numel() + outs[0][3].numel()) * 8 + 64

    # ---- roofline pass: per-kernel CUDA events on the launching streams (same workload, no graph)
    ctx.set_profiling(True)
    step(0, c=0)
    prof = ctx.profile()
    ctx.set_profiling(False)
    g1, g2 = prof.get("ts_gram", (0.0, 0)), prof.get("ts_gram2", (0.0, 0))
    gram_split = {"pass1_avg_ms": g1[0] / max(g1[1], 1), "pass2_avg_ms": g2[0] / max(g2[1], 1)}
    step_ms = sum(v[0] for v in prof.values())
    M, nnz, r, rB = op.M, op.nnz, cfg.rank_cap, cfg.r_B
    w = rB + 4 * r
    p = min(n, w)
    # algorithmic (structurally necessary) work per launch at steady state:
    #   pass 1  Y = Ucat R_V^T (R_V^T lower trapezoidal) + G1 = Y^T Y (symmetric)
    #   pass 2  Q1 = Y R1^{-1} (upper triangular) + G2 = Q1^T Q1
    #   basis   U' = Y W_r Sigma_r^{-1}
    flops = {"spmm": 6.0 * nnz * r,
             "ts_gram": 2.0 * M * (w * p - p * (p - 1) / 2.0) + 1.0 * M * p * (p + 1),
             "ts_gram2": 1.0 * M * p * (p + 1) + 1.0 * M * p * (p + 1),
             "ts_store": 2.0 * M * p * r}
    byts = {"spmm": 52.0 * nnz + 4.0 * (M + 1) + 32.0 * M * r,
            "ts_gram": 8.0 * M * w + 8.0 * M * p, "ts_gram2": 8.0 * M * p, "ts_store": 8.0 * M * p + 8.0 * M * r}
    bytes_spmm = byts["spmm"]

    def kernel_entry(name):
        ms_tot, cnt = prof[name]
        avg = ms_tot / max(cnt, 1)
        if name == "spmm":
            ach = bytes_spmm / (avg / 1e3) / 1e9
            return {"bound": "hbm", "achieved": ach, "peak": hbm_peak(), "unit": "GB/s",
                    "frac": ach / hbm_peak(), "avg_ms": avg, "launches": cnt, "share": ms_tot / step_ms}
        ach = flops[name] / (avg / 1e3) / 1e12
        return {"bound": "tensor", "achieved": ach, "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": ach / FP64_DMMA_PEAK_TFLOPS, "avg_ms": avg, "launches": cnt, "share": ms_tot / step_ms}
    cand = {k: v for k, v in prof.items() if k in flops}
    dom = max(cand.items(), key=lambda kv: kv[1][0])
    roof = kernel_entry(dom[0])
    roof["kernel"] = dom[0]
    roof["traffic"] = ncu_traffic(dom[0])
    roof["peak_source"] = ("MEASURED_PEAKS.json hbm_gbs" if roof["unit"] == "GB/s" else
                           "measured DMMA m8n8k4 fp64 (profiles/r01_phase0_fp64_peaks.jsonl)")
    kernels = {k: kernel_entry(k) for k in cand}

    # ---- BASELINE config 5 (full-rank direct approach): fused six-term operator on a dense M x 256 S,
    #      D_mu / D_nu from a 16 x 16 parameter grid, 20 repetitions, HBM GB/s vs the same roofline
    dense = None
    if args.dense and rank == 0:
        cfg5 = gen.config_by_name("fullrank")
        mu5, nu5 = gen.parameter_grid(cfg5)
        ctx5 = lrcheb.Context(local)
        ctx5.set_operator(rp_d, ci_d, vals_d, op.rho_f, op.lambda_s, borrow=True)
        ctx5.set_params(mu5, nu5)
        g = torch.Generator(device=dev).manual_seed(cfg5.seed)
        S5 = torch.randn((op.M, cfg5.dense_cols), dtype=torch.float64, device=dev, generator=g)
        for _ in range(3):
            Y5 = ctx5.apply_dense(S5)
        kms = []
        for _ in range(cfg5.reps):
            Y5 = ctx5.apply_dense(S5)
            kms.append(ctx5.last_kernel_ms())
        avg = float(np.mean(kms))
        byts5 = 52.0 * nnz + 4.0 * (M + 1) + 16.0 * M * cfg5.dense_cols
        dense = {"workload": f"config 5: M={M} dense S M x {cfg5.dense_cols}, {cfg5.reps} repetitions",
                 "avg_ms": avg, "achieved": byts5 / (avg / 1e3) / 1e9, "unit": "GB/s", "peak": hbm_peak(),
                 "frac": byts5 / (avg / 1e3) / 1e9 / hbm_peak(),
                 "tflops": 6.0 * nnz * cfg5.dense_cols / (avg / 1e3) / 1e12,
                 "tensor_frac": 6.0 * nnz * cfg5.dense_cols / (avg / 1e3) / 1e12 / FP64_DMMA_PEAK_TFLOPS,
                 "bound": "tensor (6 nnz ncols fp64 flops at the DMMA peak outlast the bytes at the HBM peak)"}
        del S5, Y5
        ctx5.close()

    # ---- the whole iteration against its roofline: per kernel max(flops / fp64 peak, bytes / HBM peak),
    #      summed over the M-level kernels of one steady-state iteration
    it_parts = {k: (flops[k], byts[k]) for k in flops}
    t_roof = sum(max(f / (FP64_DMMA_PEAK_TFLOPS * 1e12), b / (hbm_peak() * 1e9)) for f, b in it_parts.values())
    t_meas = 1.0 / value
    iteration_roofline = {"flops": sum(f for f, _ in it_parts.values()), "bytes": sum(b for _, b in it_parts.values()),
                          "roofline_ms": t_roof * 1e3, "measured_ms_per_iteration": t_meas * 1e3,
                          "frac": t_roof / t_meas,
                          "per_kernel_ms": {k: max(f / (FP64_DMMA_PEAK_TFLOPS * 1e9), b / (hbm_peak() * 1e6))
                                            for k, (f, b) in it_parts.items()},
                          "bound": "fp64 tensor (the Gram / basis passes); the SpMM alone is HBM-bound"}

    result = {
        "metric": "ChebyshevT iterations/sec (fused-SpMM HBM GB/s in roofline_spmm)",
        "value": value, "unit": "iterations/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded FE-like operator, DESIGN.md input recipe)",
        "config": {"workload": workload_str(cfg, op, n),
                   "step": "one full ChebyshevT solve of one parameter subset (N iterations + final residual)",
                   "subsets_per_rank": len(my_subsets), "parallelism": f"subsets round-robin over {world} GPU(s)",
                   "concurrent_subsets_per_gpu": S, "reserved_sms": reserve,
                   "l2": "inputs larger than L2 (operator 3.06 GB >> 126 MB)"},
        "e2e": {"value": e2e_value, "unit": "iterations/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": roof,
        "roofline_spmm": kernel_entry("spmm"),
        "roofline_kernels": kernels,
        "iteration_roofline": iteration_roofline,
        "config5_dense_spmm": dense,
        "kernel_ms_per_step": {k: v[0] for k, v in prof.items()},
        "ts_gram_passes": gram_split,
        "final_rel_residual": infos[-1]["rel_residual"],
        "ranks_final": infos[-1]["rank"],
    }
    if rank == 0 and not args.no_cpu_baseline:
        rows = cpu_calibrate(prob, args.cpu_seconds)
        t = cpu_sample(prob, rows)
        result["cpu_baseline"] = {"value": (rows / M) / t, "unit": "iterations/s", "cores": cpu_cores(),
                                  "kind": "oracle",
                                  "sample": f"one steady-state oracle iteration (six-term scipy SpMM, single-"
                                            f"threaded; Householder QR + SVD truncation, BLAS threads = cores) on "
                                            f"rows [0,{rows}) of {M}; {t:.1f}s, scaled by rows/M"}
    if rank == 0:
        print(json.dumps(result))
    if world > 1:
        dist.destroy_process_group()


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0   # B200_PROFILING.md fallback


def ncu_traffic(kernel):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary, else None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


def workload_str(cfg, op, n):
    """The workload named in both arms' `config` (same string, so the driver compares like with like)."""
    return (f"{cfg.name}: M={op.M} nnz/matrix={op.nnz} n={n} r_B={cfg.r_B} cap={cfg.rank_cap} tol={cfg.tol} "
            f"N={cfg.n_iter} iterations per subset solve")


def run_reference(args, rank, world):
    """The oracle as it stands, timed on host cores on a row-sampled piece of our config's workload."""
    from synth import generator as gen
    if rank != 0:
        return
    prob = gen.make_problem(args.config)
    cfg, op = prob.cfg, prob.op
    budget = max(2.0, min(30.0, 150.0 / max(1, args.steps + args.warmup)))
    rows = cpu_calibrate(prob, budget)
    for _ in range(args.warmup):
        cpu_sample(prob, rows)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_sample(prob, rows)
    t = time.perf_counter() - t0
    value = args.steps * (rows / op.M) / t
    sample = (f"per step: one steady-state oracle iteration on rows [0,{rows}) of M={op.M} "
              f"({cfg.name}); iterations/s scaled by rows/M")
    print(json.dumps({
        "impl": "reference", "metric": "ChebyshevT iterations/sec (fused-SpMM HBM GB/s in roofline_spmm)",
        "value": value, "unit": "iterations/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_str(cfg, op, len(prob.subset(0)[0])),
                   "sampling": "each step times one steady-state oracle iteration on a row block; see sample"},
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": cpu_cores(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


if __name__ == "__main__":
    main()
