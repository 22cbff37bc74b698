"""Write the full-size parity goldens of the GPU tests (TEST INFRASTRUCTURE; calls only oracle/ and
the input generators of synth/ -- no value here comes from the CUDA path).

    python tests/golden/make_goldens.py large 0 1 2        # ~1 h per Large subset on 8 host cores
    python tests/golden/make_goldens.py medium 0           # every iterate X_1..X_80 on 256 rows

For each (config, subset) it runs the oracle's whole ChebyshevT solve (oracle.chebyshevt: literal
six-term concatenation, Householder QR + LAPACK SVD truncation; PAPER.md P:30-36 operator, P:544
truncation, readings S1-S19) on the BASELINE config's seeded inputs and stores, in
tests/golden/<config>_s<subset>.npz:

  ranks[N]            rank of X_1..X_N
  sigmas[N, 128]      core singular values of every truncation (descending, zero padded)
  rel_residual        ||B - L(X_N)||_F / ||B||_F (untruncated, reading S14)
  rows[R]             a seeded sample of R row indices of the M rows
  ck[C]               checkpoint iterations k
  U_ck[C, R, cap]     U_k[rows, :] (zero padded past rank)
  V_ck[C, n, cap]     V_k (zero padded past rank)
  signature           numeric signature of the inputs (a changed generator invalidates the file loudly)

X_k restricted to the sampled rows is U_ck[c] @ V_ck[c].T; the GPU tests compare their own X_k on
the same rows within the BASELINE tolerance (1e-8 relative Frobenius) and rho within 1e-9.
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import chebyshevt as orc  # noqa: E402
from synth import generator as gen    # noqa: E402

ROW_SEED = 20081027
N_ROWS = 512


def signature(op, d_mu, d_nu, BU, BV, lam_min, lam_max) -> np.ndarray:
    """Numeric signature of the inputs: per array (sum |x|, ||x||_2, sum x cos(i/1000)) on a strided sample.
    The synthetic inputs are reproducible only up to the last bits across hosts (NumPy's vectorised
    log/cos in the Box-Muller generator differ by an ulp between CPU instruction sets), so the GPU
    tests compare signatures within 1e-10 of each array's sum |x| instead of hashing bytes."""
    parts = [op.row_ptr.astype(np.float64), op.col_idx[:100000].astype(np.float64)]
    parts += [np.asarray(v[::997], np.float64) for v in op.vals]
    parts += [np.ravel(a).astype(np.float64) for a in (d_mu, d_nu, BU[::101], BV)]
    parts.append(np.array([lam_min, lam_max, op.rho_f, op.lambda_s]))
    sig = []
    for x in parts:
        w = np.cos(np.arange(x.size, dtype=np.float64) * 0.001)
        sig += [np.sum(np.abs(x)), np.sqrt(np.sum(x * x)), np.sum(x * w)]
    return np.array(sig)


def same_inputs(sig_a, sig_b, rtol: float = 1e-10) -> bool:
    a, b = np.asarray(sig_a).reshape(-1, 3), np.asarray(sig_b).reshape(-1, 3)
    if a.shape != b.shape:
        return False
    scale = np.maximum(a[:, :1], 1e-300)          # a perturbation dx moves each component by <= ||dx||_1
    return bool(np.all(np.abs(a - b) <= rtol * scale))


def sample_rows(M: int, R: int = N_ROWS) -> np.ndarray:
    rng = np.random.default_rng(ROW_SEED)
    return np.sort(rng.choice(M, size=min(R, M), replace=False)).astype(np.int64)


def checkpoints(N: int, full: bool, every: bool = False):
    if every:
        return list(range(1, N + 1))
    return list(range(10, N + 1, 10)) if full else [N]


def make(prob, subset: int, full_checkpoints: bool, every: bool = False, n_rows: int = N_ROWS):
    cfg, op = prob.cfg, prob.op
    d_mu, d_nu, BU, BV = prob.subset(subset)
    n, N, cap = len(d_mu), cfg.n_iter, cfg.rank_cap
    mats = orc.csr_matrices(op.M, op.row_ptr, op.col_idx, op.vals)
    terms = orc.term_list(mats, op.rho_f, op.lambda_s, d_mu, d_nu)
    rows = sample_rows(op.M, n_rows)
    cks = checkpoints(N, full_checkpoints, every)
    U_ck = np.zeros((len(cks), len(rows), cap))
    V_ck = np.zeros((len(cks), n, cap))
    t0 = [time.time()]

    def on_iterate(k, U, V, s):
        r = U.shape[1]
        if k in cks:
            c = cks.index(k)
            U_ck[c, :, :r] = U[rows]
            V_ck[c, :, :r] = V
        dt = time.time() - t0[0]
        t0[0] = time.time()
        print(f"  {cfg.name} s{subset} k={k} rank={r} sigma1={s[0]:.6e} ({dt:.1f}s)", flush=True)

    res = orc.chebyshevt(terms, BU, BV, prob.lam_min, prob.lam_max, cfg.tol, cap, N,
                         record_iterates=False, on_iterate=on_iterate)
    sig = np.zeros((N, 128))
    for k, s in enumerate(res.sigmas):
        sig[k, :min(128, len(s))] = s[:128]
    out = os.path.join(HERE, f"{cfg.name}_s{subset}.npz")
    np.savez_compressed(out, ranks=np.array(res.ranks, dtype=np.int64), sigmas=sig,
                        rel_residual=np.float64(res.rel_residual), rows=rows, ck=np.array(cks, dtype=np.int64),
                        U_ck=U_ck, V_ck=V_ck,
                        signature=signature(op, d_mu, d_nu, BU, BV, prob.lam_min, prob.lam_max),
                        config=cfg.name, subset=np.int64(subset), N=np.int64(N), tol=np.float64(cfg.tol),
                        cap=np.int64(cap))
    print(f"wrote {out}: rho={res.rel_residual:.12e} ranks[-5:]={res.ranks[-5:]}", flush=True)


def add_signature(name: str, subset: int):
    """Add the input signature to a golden written by an earlier version of this script (computed here
    from synth/ only, on the host that wrote the golden)."""
    path = os.path.join(HERE, f"{name}_s{subset}.npz")
    g = dict(np.load(path))
    prob = gen.make_problem(name)
    d_mu, d_nu, BU, BV = prob.subset(subset)
    g.pop("fingerprint", None)
    g["signature"] = signature(prob.op, d_mu, d_nu, BU, BV, prob.lam_min, prob.lam_max)
    np.savez_compressed(path, **g)
    print(f"signed {path}")


def main():
    if sys.argv[1] == "--sign":
        for k in sys.argv[3:]:
            add_signature(sys.argv[2], int(k))
        return
    name = sys.argv[1]
    subsets = [int(x) for x in sys.argv[2:]] or [0]
    t = time.time()
    prob = gen.make_problem(name)
    print(f"problem {name}: M={prob.op.M} nnz={prob.op.nnz} ({time.time() - t:.0f}s)", flush=True)
    for i, k in enumerate(subsets):
        if name == "medium":        # every iterate of subset 0 (the GPU test compares all 80)
            make(prob, k, full_checkpoints=True, every=(i == 0), n_rows=256)
        else:
            make(prob, k, full_checkpoints=(i == 0))


if __name__ == "__main__":
    main()
