"""Write the full-size parity goldens of the GPU tests (TEST INFRASTRUCTURE; calls only oracle/ and
the input generators of synth/ -- no value here comes from the CUDA path).

    python tests/golden/make_goldens.py large 0 1 2        # ~1 h per Large subset on 8 host cores

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
  fingerprint         hashes of the inputs (so a changed generator invalidates the file loudly)

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


def fingerprint(op, d_mu, d_nu, BU, BV, lam_min, lam_max) -> str:
    h = hashlib.sha256()
    h.update(op.row_ptr.tobytes())
    h.update(op.col_idx[:100000].tobytes())
    for v in op.vals:
        h.update(np.ascontiguousarray(v[::997]).tobytes())
    for a in (d_mu, d_nu, BU[::101], BV):
        h.update(np.ascontiguousarray(a).tobytes())
    h.update(np.array([lam_min, lam_max, op.rho_f, op.lambda_s]).tobytes())
    return h.hexdigest()


def sample_rows(M: int, R: int = N_ROWS) -> np.ndarray:
    rng = np.random.default_rng(ROW_SEED)
    return np.sort(rng.choice(M, size=min(R, M), replace=False)).astype(np.int64)


def checkpoints(N: int, full: bool):
    return list(range(10, N + 1, 10)) if full else [N]


def make(prob, subset: int, full_checkpoints: bool):
    cfg, op = prob.cfg, prob.op
    d_mu, d_nu, BU, BV = prob.subset(subset)
    n, N, cap = len(d_mu), cfg.n_iter, cfg.rank_cap
    mats = orc.csr_matrices(op.M, op.row_ptr, op.col_idx, op.vals)
    terms = orc.term_list(mats, op.rho_f, op.lambda_s, d_mu, d_nu)
    rows = sample_rows(op.M)
    cks = checkpoints(N, full_checkpoints)
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
                        fingerprint=fingerprint(op, d_mu, d_nu, BU, BV, prob.lam_min, prob.lam_max),
                        config=cfg.name, subset=np.int64(subset), N=np.int64(N), tol=np.float64(cfg.tol),
                        cap=np.int64(cap))
    print(f"wrote {out}: rho={res.rel_residual:.12e} ranks[-5:]={res.ranks[-5:]}", flush=True)


def main():
    name = sys.argv[1]
    subsets = [int(x) for x in sys.argv[2:]] or [0]
    t = time.time()
    prob = gen.make_problem(name)
    print(f"problem {name}: M={prob.op.M} nnz={prob.op.nnz} ({time.time() - t:.0f}s)", flush=True)
    for i, k in enumerate(subsets):
        make(prob, k, full_checkpoints=(i == 0))


if __name__ == "__main__":
    main()
