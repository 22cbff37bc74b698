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
    ap.add_argument("--steps", type=int, default=9)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="large")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--streams", type=int, default=3, help="concurrent subset solves per GPU")
    ap.add_argument("--no-dense", dest="dense", action="store_false", help="skip the config-5 measurement")
    ap.add_argument("--reserve-sms", type=int, default=3, help="SMs the persistent kernels leave free")
    ap.add_argument("--groups", type=int, default=1,
                    help="with --batch S: this many lockstep groups of S subsets run concurrently (own host "
                         "threads, contexts and streams; SMs reserved as for --streams)")
    ap.add_argument("--batch", type=int, default=0,
                    help="f1: solve this many subsets in lockstep per call (one batched SpMM per iteration) "
                         "instead of independent concurrent streams")
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
# launch: `--gpus N` without a torchrun environment re-executes this file under torchrun
# ----------------------------------------------------------------------------------------------
def free_port():
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def relaunch_under_torchrun(args):
    """One process per GPU (the contract's launch): python -m torch.distributed.run ... bench.py."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ----------------------------------------------------------------------------------------------
# the distributed skeleton (backend-agnostic: NCCL on the GPU box, gloo in tests/test_multirank.py)
# ----------------------------------------------------------------------------------------------
def run_distributed(args, leg, rank, world, dist=None, device=None, emit=print):
    """Shard the subsets over the ranks (no data-path collective), run W untimed warm-up
    steps, time exactly K steps between barriers (device time from the leg), take the max over
    ranks, and have rank 0 emit the JSON line.  `leg` does the work: prepare(subsets), steps(n, host)
    -> (device ms, infos, launches), extras(value) -> dict of extra keys."""
    cfg = leg.cfg
    mine = shard_subsets(cfg.K, rank, world)
    leg.prepare(mine)
    leg.warmup(args.warmup)

    def timed(host):
        if dist is not None and world > 1:
            dist.barrier()
        ms, infos, launches = leg.steps(args.steps, host)
        ms = max_over_ranks(ms, dist if world > 1 else None, device)
        if dist is not None and world > 1:
            dist.barrier()
        return ms, infos, launches

    leg.clock_start()
    ms, infos, launches = timed(False)
    clocks = leg.clock_stop()
    ms_e2e, _, _ = timed(True)
    iters = args.steps * cfg.n_iter * world
    value = iters / (ms / 1e3)
    e2e_value = iters / (ms_e2e / 1e3)
    result = {
        "metric": "ChebyshevT iterations/sec (fused-SpMM HBM GB/s in roofline_spmm)",
        "value": value, "unit": "iterations/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded FE-like operator, DESIGN.md input recipe)",
        "config": dict(leg.config(), subsets_per_rank=len(mine),
                       parallelism=f"subsets round-robin over {world} GPU(s), no data-path collective"),
        "e2e": {"value": e2e_value, "unit": "iterations/s", "h2d_bytes_per_step": int(leg.h2d_bytes()),
                "d2h_bytes_per_step": int(leg.d2h_bytes())},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    result.update(leg.extras(value, rank, world))
    if infos and infos[-1] is not None:
        result["final_rel_residual"] = infos[-1]["rel_residual"]
        result["ranks_final"] = infos[-1]["rank"]
    if rank == 0:
        emit(json.dumps(result))
    return result


class GpuLeg:
    """The product path: S concurrent subset solves per GPU (one lrc context, CUDA stream and host
    thread each, all borrowing one device copy of the operator)."""

    def __init__(self, args, local):
        import torch
        from paper_2008_10275_b200 import lrcheb
        from synth import generator as gen
        self.args, self.local, self.torch, self.lrcheb, self.gen = args, local, torch, lrcheb, gen
        self.dev = torch.device("cuda", local)
        from synth import terms as st
        self.terms = args.config in st.TERM_CONFIGS      # a general term list
        if self.terms:
            self.prob = st.make_term_problem(args.config)
            self.cfg, self.op = self.prob.cfg, self.prob     # (M, row_ptr, col_idx, vals)
            self.op.nnz = int(self.prob.col_idx.shape[0])
        else:
            self.prob = gen.make_problem(args.config)
            self.cfg, self.op = self.prob.cfg, self.prob.op
        self.G = max(1, args.groups) if args.batch > 1 else 1     # concurrent lockstep groups (f1)
        self.B = args.batch if args.batch > 1 else 1                # subsets per lockstep group
        self.S = max(1, self.B * self.G if args.batch > 1 else args.streams)
        self.reserve = args.reserve_sms if (self.S > 1 and (args.batch <= 1 or self.G > 1)) else 0
        op, dev = self.op, self.dev
        self.rp_d, self.ci_d = torch.from_numpy(op.row_ptr).to(dev), torch.from_numpy(op.col_idx).to(dev)
        self.vals_d = [torch.from_numpy(v).to(dev) for v in op.vals]
        self.ctxs = []
        for _ in range(self.S):
            c = lrcheb.Context(local)
            c.set_reserved_sms(self.reserve)
            if self.terms:
                c.set_operator_terms(self.rp_d, self.ci_d, self.vals_d, self.prob.coef, self.prob.id_group, borrow=True)
            else:
                c.set_operator(self.rp_d, self.ci_d, self.vals_d, op.rho_f, op.lambda_s, borrow=True)
            self.ctxs.append(c)
        self.main_s = torch.cuda.Stream(device=dev)
        self.clk = ClockSampler(local)

    def prepare(self, subsets):
        torch, cfg, op, dev = self.torch, self.cfg, self.op, self.dev
        self.subsets = subsets
        self.inputs = []
        for k in subsets:
            d_mu, d_nu, BU, BV = self.prob.subset(k)
            self.inputs.append((d_mu, d_nu, torch.from_numpy(BU).to(dev), torch.from_numpy(BV).to(dev),
                                torch.from_numpy(BU).pin_memory(), torch.from_numpy(BV).pin_memory()))
        self.n = len(self.inputs[0][0])
        self.outs = [(torch.empty((op.M, cfg.rank_cap), dtype=torch.float64, device=dev),
                      torch.empty((self.n, cfg.rank_cap), dtype=torch.float64, device=dev),
                      torch.empty((op.M, cfg.rank_cap), dtype=torch.float64).pin_memory(),
                      torch.empty((self.n, cfg.rank_cap), dtype=torch.float64).pin_memory())
                     for _ in range(self.S)]

    def step(self, i, host=False, c=None):
        si = (i % self.S) if c is None else c
        cx = self.ctxs[si]
        Uo, Vo, Uh, Vh = self.outs[si]
        d_mu, d_nu, bu, bv, bu_h, bv_h = self.inputs[i % len(self.inputs)]
        self.set_subset(cx, d_mu, d_nu)
        p, cfg = self.prob, self.cfg
        if host:
            return cx.solve(bu_h, bv_h, p.lam_min, p.lam_max, cfg.tol, cfg.rank_cap, cfg.n_iter, out=(Uh, Vh))[2]
        return cx.solve(bu, bv, p.lam_min, p.lam_max, cfg.tol, cfg.rank_cap, cfg.n_iter, out=(Uo, Vo))[2]

    def set_subset(self, cx, x, y):
        """The subset's right diagonals: set_params(d_mu, d_nu), or set_diagonals(D) for a term list."""
        if self.terms:
            cx.set_diagonals(y)
        else:
            cx.set_params(x, y)

    def run_batched(self, nsteps, host):
        """nsteps subset solves in lockstep groups of B subsets (lrc_solve_batch); with G > 1
        groups, G host threads each run their share of the groups on their own B contexts concurrently."""
        if self.G > 1:
            infos = [None] * nsteps
            errs = []
            per = self.B * self.G

            def worker(gi):
                try:
                    for g0 in range(gi * self.B, nsteps, per):
                        n = min(self.B, nsteps - g0)
                        res = self._run_group(g0, n, gi * self.B, host)
                        for j in range(n):
                            infos[g0 + j] = res[j]
                except Exception as e:  # surfaced below
                    errs.append(e)
            ths = [threading.Thread(target=worker, args=(gi,)) for gi in range(self.G)]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            if errs:
                raise errs[0]
            if host:
                self.torch.cuda.synchronize()
            return infos
        infos = [None] * nsteps
        for g0 in range(0, nsteps, self.B):
            n = min(self.B, nsteps - g0)
            res = self._run_group(g0, n, 0, host)
            for j in range(n):
                infos[g0 + j] = res[j]
        if host:
            self.torch.cuda.current_stream().synchronize()
        return infos

    def _run_group(self, g0, n, c0, host):
        """Subsets g0 .. g0+n-1 in lockstep on contexts c0 .. c0+n-1 (one lrc_solve_batch call).
        host=True: the B factors are copied from pinned host memory and the outputs back (e2e leg)."""
        lrcheb, torch, p, cfg = self.lrcheb, self.torch, self.prob, self.cfg
        infos = [None] * n
        idx = list(range(g0, g0 + n))
        cx = self.ctxs[c0:c0 + n]
        bus, bvs = [], []
        for c, i in zip(cx, idx):
            d_mu, d_nu, bu, bv, bu_h, bv_h = self.inputs[i % len(self.inputs)]
            self.set_subset(c, d_mu, d_nu)
            if host:
                bu = bu_h.to(self.dev, non_blocking=True)
                bv = bv_h.to(self.dev, non_blocking=True)
            bus.append(bu)
            bvs.append(bv)
        outs = [(o[0], o[1]) for o in self.outs[c0:c0 + n]]
        res = lrcheb.solve_batch(cx, bus, bvs, p.lam_min, p.lam_max, cfg.tol, cfg.rank_cap, cfg.n_iter,
                                 outs=outs)
        for j in range(n):
            infos[j] = res[j][2]
            if host:
                self.outs[c0 + j][2].copy_(res[j][0], non_blocking=True)
                self.outs[c0 + j][3].copy_(res[j][1], non_blocking=True)
        return infos

    def run_steps(self, nsteps, host):
        """nsteps solves dealt round-robin to the S streams, one host thread per stream."""
        if self.args.batch > 1:
            return self.run_batched(nsteps, host)
        infos = [None] * nsteps
        errs = []

        def worker(si):
            try:
                for i in range(si, nsteps, self.S):
                    infos[i] = self.step(i, host, si)
            except Exception as e:   # surfaced below: a failing solve must fail the bench
                errs.append(e)
        ths = [threading.Thread(target=worker, args=(si,)) for si in range(self.S)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        if errs:
            raise errs[0]
        return infos

    def warmup(self, w):
        self.run_steps(max(w, self.S), False)           # >= 1 warm-up per stream (graph capture)
        self.run_steps(self.S, True)                    # and the host-buffer (e2e) path once per stream

    def steps(self, nsteps, host):
        torch = self.torch
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches0 = sum(c.kernel_launches() for c in self.ctxs)
        e0.record(self.main_s)
        for c in self.ctxs:
            c.stream.wait_event(e0)
        infos = self.run_steps(nsteps, host)
        for c in self.ctxs:
            ev = torch.cuda.Event()
            ev.record(c.stream)
            self.main_s.wait_event(ev)
        e1.record(self.main_s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), infos, sum(c.kernel_launches() for c in self.ctxs) - launches0

    def clock_start(self):
        self.clk.start()

    def clock_stop(self):
        return self.clk.stop()

    def h2d_bytes(self):
        a = self.args
        return sum(self.inputs[i % len(self.inputs)][4].numel() * 8 + self.inputs[i % len(self.inputs)][5].numel() * 8
                   for i in range(a.steps)) / a.steps

    def d2h_bytes(self):
        return (self.outs[0][2].numel() + self.outs[0][3].numel()) * 8 + 64

    def config(self):
        return {"workload": workload_str(self.cfg, self.op, self.n),
                "step": "one full ChebyshevT solve of one parameter subset (N iterations + final residual)",
                "concurrent_subsets_per_gpu": self.S, "reserved_sms": self.reserve,
                "subset_schedule": (f"f1 batched lockstep: {self.B} subsets per lrc_solve_batch call (one fused SpMM "
                                    f"pass per iteration for all of them), {self.G} such group(s) concurrently")
                                   if self.args.batch > 1 else
                                   f"{self.S} independent solves on concurrent streams",
                "l2": f"inputs larger than L2 (operator {operator_bytes(self.op) / 1e9:.2f} GB vs 126 MB)"
                      if operator_bytes(self.op) > L2_BYTES else "operator fits in L2 (latency-bound config)"}

    def single_stream(self, steps=2):
        """Per-subset latency: the same solve on one context alone (graph replay)."""
        torch = self.torch
        self.step(0, c=0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s = self.ctxs[0].stream
        e0.record(s)
        for i in range(steps):
            self.step(i * self.S, c=0)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        return {"value": steps * self.cfg.n_iter / (ms / 1e3), "unit": "iterations/s",
                "ms_per_iteration": ms / (steps * self.cfg.n_iter), "steps": steps,
                "note": "one subset at a time on one stream (latency view); reserved SMs as in the headline"}

    def batched_f1(self, calls=2):
        """SURVEY §8 f1 measured beside the headline: groups of S subsets solved in lockstep by
        lrc_solve_batch (one batched SpMM pass per iteration), S = the headline's concurrent streams."""
        torch = self.torch
        S = min(len(self.ctxs), 4)
        if S < 2 or self.args.batch > 1:
            return None
        saved = self.args.batch, self.B, self.G
        self.args.batch, self.B, self.G = S, S, 1
        try:
            self.run_batched(S, False)                       # capture the batch graph
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            self.run_batched(S * calls, False)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        finally:
            self.args.batch, self.B, self.G = saved
        return {"value": S * calls * self.cfg.n_iter / (ms / 1e3), "unit": "iterations/s", "subsets_per_call": S,
                "calls": calls, "note": "f1 lockstep: one fused SpMM pass per iteration for all S subsets' U, their "
                                        "truncations on S streams; the headline's independent concurrent streams "
                                        "measure faster (the lockstep aligns every subset's single-CTA core steps)"}

    def extras(self, value, rank, world):
        args, cfg, op = self.args, self.cfg, self.op
        out = {"single_stream": self.single_stream(), "f1_batched": self.batched_f1()}
        ctx = self.ctxs[0]
        # ---- roofline pass: per-kernel CUDA events on the launching streams (same workload, no graph)
        ctx.set_profiling(True)
        self.step(0, c=0)
        prof = ctx.profile()
        ctx.set_profiling(False)
        g1, g2 = prof.get("ts_gram", (0.0, 0)), prof.get("ts_gram2", (0.0, 0))
        step_ms = sum(v[0] for v in prof.values())
        M, nnz, r, rB, n = op.M, op.nnz, cfg.rank_cap, cfg.r_B, self.n
        w = rB + 4 * r
        p = min(n, w)
        T, G = (len(op.vals), self.prob.coef.shape[1]) if self.terms else (6, 3)
        flops, byts = algorithmic_work(M, nnz, r, rB, n, T, G)

        def kernel_entry(name):
            ms_tot, cnt = prof[name]
            avg = ms_tot / max(cnt, 1)
            if name == "spmm":
                ach = byts["spmm"] / (avg / 1e3) / 1e9
                return {"bound": "hbm", "achieved": ach, "peak": hbm_peak(), "unit": "GB/s",
                        "frac": ach / hbm_peak(), "avg_ms": avg, "launches": cnt, "share": ms_tot / step_ms,
                        "traffic": ncu_traffic(name, args.config)}
            ach = flops[name] / (avg / 1e3) / 1e12
            return {"bound": "tensor", "achieved": ach, "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": ach / FP64_DMMA_PEAK_TFLOPS, "avg_ms": avg, "launches": cnt, "share": ms_tot / step_ms,
                    "traffic": ncu_traffic(name, args.config)}
        cand = {k: v for k, v in prof.items() if k in flops}
        dom = max(cand.items(), key=lambda kv: kv[1][0])
        roof = kernel_entry(dom[0])
        roof["kernel"] = dom[0]
        roof["peak_source"] = ("MEASURED_PEAKS.json hbm_gbs" if roof["unit"] == "GB/s" else
                               "measured DMMA m8n8k4 fp64 (profiles/r01_phase0_fp64_peaks.jsonl); "
                               "MEASURED_PEAKS.json has no fp64 entry")
        kernels = {k: kernel_entry(k) for k in cand}
        out.update({"roofline": roof, "roofline_spmm": kernel_entry("spmm"), "roofline_kernels": kernels,
                    "kernel_ms_per_step": {k: v[0] for k, v in prof.items()},
                    "ts_gram_passes": {"pass1_avg_ms": g1[0] / max(g1[1], 1), "pass2_avg_ms": g2[0] / max(g2[1], 1)}})
        # ---- the whole iteration against its roofline: per kernel max(flops / fp64 peak, bytes / HBM
        #      peak), summed over the M-level kernels of one steady-state iteration
        it_parts = {k: (flops[k], byts[k]) for k in flops}
        t_roof = sum(max(f / (FP64_DMMA_PEAK_TFLOPS * 1e12), b / (hbm_peak() * 1e9)) for f, b in it_parts.values())
        t_meas = world / value                       # one GPU's time per iteration
        out["iteration_roofline"] = {
            "flops": sum(f for f, _ in it_parts.values()), "bytes": sum(b for _, b in it_parts.values()),
            "roofline_ms": t_roof * 1e3, "measured_ms_per_iteration": t_meas * 1e3, "frac": t_roof / t_meas,
            "hbm_only_ms": sum(b for _, b in it_parts.values()) / (hbm_peak() * 1e9) * 1e3,
            "per_kernel_ms": {k: max(f / (FP64_DMMA_PEAK_TFLOPS * 1e9), b / (hbm_peak() * 1e6))
                              for k, (f, b) in it_parts.items()},
            "bound": "fp64 tensor (the Gram / basis passes); the SpMM alone is HBM-bound"}
        if args.dense and rank == 0 and args.config == "large":
            out["config5_dense_spmm"] = self.dense_config5()
        if rank == 0 and not args.no_cpu_baseline and not self.terms:
            rows = cpu_calibrate(self.prob, args.cpu_seconds)
            t = cpu_sample(self.prob, rows)
            out["cpu_baseline"] = {"value": (rows / M) / t, "unit": "iterations/s", "cores": cpu_cores(),
                                   "kind": "oracle",
                                   "sample": f"one steady-state oracle iteration (six-term scipy SpMM, single-"
                                             f"threaded; Householder QR + SVD truncation, BLAS threads = cores) on "
                                             f"rows [0,{rows}) of {M}; {t:.1f}s, scaled by rows/M"}
        return out

    def dense_config5(self):
        """BASELINE config 5 (full-rank direct approach): fused six-term operator on a dense M x 256 S,
        D_mu / D_nu from a 16 x 16 parameter grid, 20 repetitions, HBM GB/s vs the same roofline."""
        torch, gen, op, nnz, M = self.torch, self.gen, self.op, self.op.nnz, self.op.M
        cfg5 = gen.config_by_name("fullrank")
        mu5, nu5 = gen.parameter_grid(cfg5)
        ctx5 = self.lrcheb.Context(self.local)
        ctx5.set_operator(self.rp_d, self.ci_d, self.vals_d, op.rho_f, op.lambda_s, borrow=True)
        ctx5.set_params(mu5, nu5)
        g = torch.Generator(device=self.dev).manual_seed(cfg5.seed)
        S5 = torch.randn((M, cfg5.dense_cols), dtype=torch.float64, device=self.dev, generator=g)
        for _ in range(3):
            Y5 = ctx5.apply_dense(S5)
        kms = []
        for _ in range(cfg5.reps):
            Y5 = ctx5.apply_dense(S5)
            kms.append(ctx5.last_kernel_ms())
        avg = float(np.mean(kms))
        byts5 = 52.0 * nnz + 4.0 * (M + 1) + 16.0 * M * cfg5.dense_cols
        fl5 = 6.0 * nnz * cfg5.dense_cols
        del S5, Y5
        ctx5.close()
        return {"workload": f"config 5: M={M} dense S M x {cfg5.dense_cols}, {cfg5.reps} repetitions",
                "avg_ms": avg, "achieved": byts5 / (avg / 1e3) / 1e9, "unit": "GB/s", "peak": hbm_peak(),
                "frac": byts5 / (avg / 1e3) / 1e9 / hbm_peak(),
                "tflops": fl5 / (avg / 1e3) / 1e12, "tensor_frac": fl5 / (avg / 1e3) / 1e12 / FP64_DMMA_PEAK_TFLOPS,
                "bound": "tensor (6 nnz ncols fp64 flops at the DMMA peak outlast the bytes at the HBM peak)",
                "traffic": ncu_traffic("dense", "large")}


def algorithmic_work(M, nnz, r, rB, n, T=6, G=3):
    """Structurally necessary flops / bytes per launch at steady state (DESIGN.md §2 table): the SpMM reads
    T value arrays + the column indices, U once and writes G grouped outputs (2 G nnz r flops); pass 1
    Y = Ucat R_V^T (R_V^T lower trapezoidal) + G1 = Y^T Y (symmetric); pass 2 Q1 = Y R1^{-1} (upper
    triangular) + G2 = Q1^T Q1;  basis  U' = Y W_r Sigma_r^{-1}.  w = r_B + (G + 1) r."""
    w = rB + (G + 1) * r
    p = min(n, w)
    flops = {"spmm": 2.0 * G * nnz * r,
             "ts_gram": 2.0 * M * (w * p - p * (p - 1) / 2.0) + 1.0 * M * p * (p + 1),
             "ts_gram2": 1.0 * M * p * (p + 1) + 1.0 * M * p * (p + 1),
             "ts_store": 2.0 * M * p * r}
    byts = {"spmm": (8.0 * T + 4.0) * nnz + 4.0 * (M + 1) + 8.0 * (1 + G) * M * r,
            "ts_gram": 8.0 * M * w + 8.0 * M * p, "ts_gram2": 8.0 * M * p, "ts_store": 8.0 * M * p + 8.0 * M * r}
    return flops, byts


def operator_bytes(op):
    return (8 * len(op.vals) + 4) * op.nnz + 4 * (op.M + 1)


def main():
    args = parse()
    if args.impl == "reference":
        rank, world, _ = dist_env()
        return run_reference(args, rank, world)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    rank, world, local = dist_env()
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    leg = GpuLeg(args, local)
    run_distributed(args, leg, rank, world, dist if world > 1 else None, dev)
    if world > 1:
        dist.destroy_process_group()


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0   # B200_PROFILING.md fallback


def ncu_traffic(kernel, config="large"):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary (profiles/
    ncu_traffic.json, keyed by config), else None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        d = d.get(config, d if config == "large" else {})
        return d.get(kernel)
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
