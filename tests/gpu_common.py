"""Shared helpers of the GPU parity tests: seeded inputs (synth/), the oracle (oracle/), and the
C-ABI binding.  Input construction and comparison only -- no arithmetic of the method here."""
import functools

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import chebyshevt as orc
from synth import generator as gen

torch = pytest.importorskip("torch")


def require_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@functools.lru_cache(maxsize=None)
def problem(name):
    return gen.make_problem(name)


def oracle_terms(op, d_mu, d_nu):
    mats = orc.csr_matrices(op.M, op.row_ptr, op.col_idx, op.vals)
    return orc.term_list(mats, op.rho_f, op.lambda_s, d_mu, d_nu)


def make_ctx(op, d_mu, d_nu, device_inputs=False):
    from paper_2008_10275_b200 import lrcheb
    ctx = lrcheb.Context(0)
    if device_inputs:
        dev = torch.device("cuda:0")
        ctx.set_operator(torch.from_numpy(op.row_ptr).to(dev), torch.from_numpy(op.col_idx).to(dev),
                         [torch.from_numpy(v).to(dev) for v in op.vals], op.rho_f, op.lambda_s)
    else:
        ctx.set_operator(op.row_ptr, op.col_idx, op.vals, op.rho_f, op.lambda_s)
    ctx.set_params(d_mu, d_nu)
    return ctx


def lowrank_rel_diff(U1, V1, U2, V2):
    """||U1 V1^T - U2 V2^T||_F / ||U2 V2^T||_F via a thin QR of the stacked factors (no densify)."""
    U = np.hstack([U1, U2])
    V = np.hstack([V1, -V2])
    _, Ru = np.linalg.qr(U)
    num = np.linalg.norm(Ru @ V.T)
    _, R2 = np.linalg.qr(U2)
    den = np.linalg.norm(R2 @ V2.T)
    return num / den if den > 0 else num


def near_tie(sig, tau, cap, rank_o, eps=1e-12):
    """Reading S13: rank parity is exempt when a core singular value lies within eps*sigma_1 of
    the threshold tau*sigma_1, or the cap cut is a near-tie."""
    s = np.asarray(sig)
    if s.size == 0 or s[0] == 0:
        return False
    thr = tau * s[0]
    if np.any(np.abs(s - thr) <= eps * s[0]):
        return True
    if rank_o == cap and s.size > cap and abs(s[cap - 1] - s[cap]) <= eps * s[0]:
        return True
    return False


def random_csr(M, rng, density=0.01, empty_rows=(), diag_only=False):
    """Irregular CSR (sorted, no duplicates) with some empty rows, six value arrays."""
    if diag_only:
        A = sp.identity(M, format="csr")
    else:
        A = sp.random(M, M, density=density, random_state=np.random.RandomState(int(rng.integers(1 << 31))),
                      format="csr")
        A = (A + sp.identity(M, format="csr")).tocsr()
        A = A.tolil()
        for r in empty_rows:
            A.rows[r] = []
            A.data[r] = []
        A = A.tocsr()
    A.sort_indices()
    rp = A.indptr.astype(np.int32)
    ci = A.indices.astype(np.int32)
    vals = [rng.standard_normal(ci.shape[0]) for _ in range(6)]
    return gen.Operator(M=M, row_ptr=rp, col_idx=ci, vals=vals, rho_f=1.3, lambda_s=2.0)
