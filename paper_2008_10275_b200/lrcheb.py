"""Thin ctypes binding of liblrcheb (include/lrcheb.h) -- argument marshalling only.

Every step of the ChebyshevT path runs in the CUDA kernels of ``liblrcheb.so``; this module only
turns torch tensors / numpy arrays into (pointer, leading dimension, lrc_mem) triples and back.
There is no CPU fallback: if the shared library is missing or fails to load, importing this module
raises.  PyTorch is used for device memory and streams only.

Names follow the C ABI (lrc_set_operator -> Context.set_operator, ...).  Dense factors are
row-major fp64; torch CUDA tensors are passed as LRC_MEM_DEVICE, CPU tensors / numpy arrays as
LRC_MEM_HOST.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblrcheb.so")

LRC_OK, LRC_ERR_ARG, LRC_ERR_SHAPE, LRC_ERR_STATE, LRC_ERR_NOMEM, LRC_ERR_CUDA, LRC_ERR_NUMERIC = range(7)
LRC_MEM_HOST, LRC_MEM_DEVICE, LRC_MEM_DEVICE_BORROW = 0, 1, 2
LRC_RECORD_ITERATES, LRC_SKIP_FINAL_RESIDUAL, LRC_NO_GRAPH, LRC_NO_WARM_START, LRC_ASYNC = 1, 2, 4, 8, 16
LRC_PRECONDITIONED = 32
LRC_APPLY_PLAIN3, LRC_APPLY_SIX, LRC_APPLY_S2STEP = 0, 1, 2
SIGMA_STRIDE = 128

# every entry point declared in include/lrcheb.h
EXPORTS = (
    "lrc_create", "lrc_destroy", "lrc_last_error", "lrc_version", "lrc_set_operator",
    "lrc_set_params", "lrc_solve", "lrc_apply_lowrank", "lrc_apply_dense", "lrc_truncate",
    "lrc_get_iterate", "lrc_last_kernel_ms", "lrc_kernel_launches", "lrc_set_profiling", "lrc_get_profile",
    "lrc_set_reserved_sms", "lrc_solve_wait", "lrc_workspace_bytes", "lrc_set_workspace", "lrc_solve_batch",
    "lrc_set_operator_terms", "lrc_set_diagonals", "lrc_solve_gmres", "lrc_set_preconditioner",
)


class LrcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"lrcheb status {status}: {msg}")
        self.status = status


class SolveOpts(ctypes.Structure):
    _fields_ = [("lambda_min", ctypes.c_double), ("lambda_max", ctypes.c_double),
                ("tol", ctypes.c_double), ("rank_cap", ctypes.c_int64), ("n_iter", ctypes.c_int64),
                ("restart_every", ctypes.c_int64), ("flags", ctypes.c_uint32)]


class GmresOpts(ctypes.Structure):
    _fields_ = [("trunc_tol", ctypes.c_double), ("tol", ctypes.c_double), ("rank_cap", ctypes.c_int64),
                ("restart", ctypes.c_int64), ("max_cycles", ctypes.c_int64)]


class GmresInfo(ctypes.Structure):
    _fields_ = [("cycles", ctypes.c_int64), ("rank", ctypes.c_int64), ("rel_residual", ctypes.c_double),
                ("b_norm", ctypes.c_double), ("inner_steps", ctypes.POINTER(ctypes.c_int64)),
                ("cycle_residuals", ctypes.POINTER(ctypes.c_double))]


class SolveInfo(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int64), ("rel_residual", ctypes.c_double), ("b_norm", ctypes.c_double),
                ("diverged", ctypes.c_int32), ("shift_escalations", ctypes.c_int32),
                ("ms_iterations", ctypes.c_float), ("ms_total", ctypes.c_float),
                ("rank_history", ctypes.POINTER(ctypes.c_int64)),
                ("sigma_history", ctypes.POINTER(ctypes.c_double)), ("jacobi_sweeps", ctypes.c_int64),
                ("chol2_cycles", ctypes.c_double * 3)]


def load_library(path: str = None) -> ctypes.CDLL:
    path = path or os.environ.get("LRCHEB_LIB") or LIB_PATH   # LRCHEB_LIB: an alternative in-tree build
    if not os.path.exists(path):
        raise ImportError(f"liblrcheb.so not built at {path}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, I64, D, U32, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_uint32, ctypes.c_int
    lib.lrc_create.argtypes = [ctypes.POINTER(P), I32, P]
    lib.lrc_destroy.argtypes = [P]
    lib.lrc_destroy.restype = None
    lib.lrc_last_error.argtypes = [P]
    lib.lrc_last_error.restype = ctypes.c_char_p
    lib.lrc_version.restype = ctypes.c_char_p
    lib.lrc_set_operator.argtypes = [P, I64, I64, P, P, ctypes.POINTER(P), D, D, I32]
    lib.lrc_set_params.argtypes = [P, I64, P, P, I32]
    lib.lrc_set_operator_terms.argtypes = [P, I64, I64, P, P, I32, ctypes.POINTER(P), I32, P, I32, I32]
    lib.lrc_set_diagonals.argtypes = [P, I64, I32, P, I32]
    lib.lrc_set_preconditioner.argtypes = [P, D, D, I64]
    lib.lrc_solve_gmres.argtypes = [P, P, I64, P, I64, I64, ctypes.POINTER(GmresOpts), P, I64, P, I64, I32,
                                    ctypes.POINTER(GmresInfo)]
    lib.lrc_solve.argtypes = [P, P, I64, P, I64, I64, ctypes.POINTER(SolveOpts), P, I64, P, I64, I32,
                              ctypes.POINTER(SolveInfo)]
    lib.lrc_apply_lowrank.argtypes = [P, P, I64, I64, P, I64, U32, D, I32]
    lib.lrc_apply_dense.argtypes = [P, P, I64, I64, P, I64, I32]
    lib.lrc_truncate.argtypes = [P, P, I64, P, I64, I64, D, I64, P, P, ctypes.POINTER(I64), P, I32]
    lib.lrc_get_iterate.argtypes = [P, I64, P, P, ctypes.POINTER(I64), I32]
    lib.lrc_last_kernel_ms.argtypes = [P]
    lib.lrc_last_kernel_ms.restype = ctypes.c_float
    lib.lrc_solve_wait.argtypes = [P, ctypes.POINTER(SolveInfo)]
    PP = ctypes.POINTER(P)
    PI = ctypes.POINTER(I64)
    lib.lrc_solve_batch.argtypes = [PP, I32, PP, PI, PP, PI, I64, ctypes.POINTER(SolveOpts), PP, PI, PP, PI, I32,
                                    ctypes.POINTER(SolveInfo)]
    lib.lrc_workspace_bytes.argtypes = [P, I64, I64, I64, U32, ctypes.POINTER(ctypes.c_size_t)]
    lib.lrc_set_workspace.argtypes = [P, P, ctypes.c_size_t]
    lib.lrc_set_reserved_sms.argtypes = [P, I32]
    lib.lrc_set_reserved_sms.restype = I32
    lib.lrc_kernel_launches.argtypes = [P]
    lib.lrc_kernel_launches.restype = I64
    lib.lrc_set_profiling.argtypes = [P, I32]
    lib.lrc_set_profiling.restype = None
    lib.lrc_get_profile.argtypes = [P, I32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(D), ctypes.POINTER(I64)]
    lib.lrc_get_profile.restype = I32
    for name in ("lrc_create", "lrc_set_operator", "lrc_set_params", "lrc_solve", "lrc_apply_lowrank",
                 "lrc_apply_dense", "lrc_truncate", "lrc_get_iterate", "lrc_solve_wait", "lrc_workspace_bytes",
                 "lrc_set_workspace", "lrc_solve_batch", "lrc_set_operator_terms", "lrc_set_diagonals",
                 "lrc_solve_gmres", "lrc_set_preconditioner"):
        getattr(lib, name).restype = I32
    return lib


_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _mat(x, rows: int = None, cols: int = None):
    """(pointer, ld, where, keepalive) of a 2-D row-major fp64 array (torch or numpy)."""
    if _is_torch(x):
        import torch
        if x.dtype != torch.float64:
            raise TypeError(f"fp64 tensor required, got {x.dtype}")
        if x.dim() == 1:
            x = x.reshape(-1, 1)
        assert x.stride(1) == 1 or x.shape[1] <= 1, "rows must be contiguous (row-major)"
        ld = x.stride(0) if x.shape[0] > 1 else max(x.shape[1], 1)
        return x.data_ptr(), max(int(ld), int(x.shape[1])), (LRC_MEM_DEVICE if x.is_cuda else LRC_MEM_HOST), x
    a = np.ascontiguousarray(x, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return a.ctypes.data, a.shape[1], LRC_MEM_HOST, a


def _vec(x, dtype):
    """(pointer, where, keepalive) of a 1-D array of `dtype` (np.int32 or np.float64)."""
    if _is_torch(x):
        import torch
        want = torch.int32 if np.dtype(dtype) == np.int32 else torch.float64
        if x.dtype != want:
            raise TypeError(f"{want} tensor required, got {x.dtype}")
        x = x.contiguous()
        return x.data_ptr(), (LRC_MEM_DEVICE if x.is_cuda else LRC_MEM_HOST), x
    a = np.ascontiguousarray(x, dtype=dtype)
    return a.ctypes.data, LRC_MEM_HOST, a


class Context:
    """One lrc_ctx on one CUDA device, ordered on a torch-owned CUDA stream."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        self._lib = lib()
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.Stream(device=device)
        h = ctypes.c_void_p()
        st = self._lib.lrc_create(ctypes.byref(h), device, ctypes.c_void_p(self.stream.cuda_stream))
        if st != LRC_OK:
            raise LrcError(st, "lrc_create failed: " + self._lib.lrc_last_error(None).decode())
        self._h = h
        self._keep = []
        self.M = self.n = 0

    def close(self):
        if getattr(self, "_h", None):
            self._lib.lrc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != LRC_OK:
            raise LrcError(st, self._lib.lrc_last_error(self._h).decode())

    def _order(self, *xs):
        """Make the ctx stream wait for torch's current stream if device tensors are involved."""
        import torch
        if any(_is_torch(x) and x.is_cuda for x in xs if x is not None):
            self.stream.wait_stream(torch.cuda.current_stream(self.device))

    def _settle(self, *xs):
        """set_operator / set_params read device inputs with blocking copies outside any torch
        stream: let the producing (current) torch stream finish first."""
        import torch
        if any(_is_torch(x) and x.is_cuda for x in xs if x is not None):
            torch.cuda.current_stream(self.device).synchronize()

    # ------------------------------------------------------------------------------------
    def set_operator(self, row_ptr, col_idx, vals: Sequence, rho_f: float, lambda_s: float,
                     borrow: bool = False):
        rp, w1, k1 = _vec(row_ptr, np.int32)
        ci, w2, k2 = _vec(col_idx, np.int32)
        vs = [_vec(v, np.float64) for v in vals]
        assert len(vs) == 6
        wheres = {w1, w2} | {v[1] for v in vs}
        assert len(wheres) == 1, "all operator arrays must live in the same memory space"
        where = wheres.pop()
        if borrow:
            assert where == LRC_MEM_DEVICE
            where = LRC_MEM_DEVICE_BORROW
        self._settle(*([k1, k2] + [v[2] for v in vs]))
        M = (k1.shape[0] if hasattr(k1, "shape") else len(k1)) - 1
        nnz = k2.shape[0]
        arr = (ctypes.c_void_p * 6)(*[v[0] for v in vs])
        self._check(self._lib.lrc_set_operator(self._h, M, nnz, rp, ci, arr, float(rho_f), float(lambda_s), where))
        self._keep = [k1, k2] + [v[2] for v in vs] if borrow else []
        self.M = M
        self.G, self.T = 3, 6

    def set_operator_terms(self, row_ptr, col_idx, vals: Sequence, coef, id_group: int, borrow: bool = False):
        """General term list: L(S) = sum_g (sum_t coef[t, g] A_t) S diag(d_g); coef is T x G."""
        rp, w1, k1 = _vec(row_ptr, np.int32)
        ci, w2, k2 = _vec(col_idx, np.int32)
        vs = [_vec(v, np.float64) for v in vals]
        wheres = {w1, w2} | {v[1] for v in vs}
        assert len(wheres) == 1, "all operator arrays must live in the same memory space"
        where = wheres.pop()
        if borrow:
            assert where == LRC_MEM_DEVICE
            where = LRC_MEM_DEVICE_BORROW
        self._settle(*([k1, k2] + [v[2] for v in vs]))
        C = np.ascontiguousarray(coef, dtype=np.float64)
        T, G = C.shape
        assert T == len(vs)
        M = (k1.shape[0] if hasattr(k1, "shape") else len(k1)) - 1
        arr = (ctypes.c_void_p * T)(*[v[0] for v in vs])
        self._check(self._lib.lrc_set_operator_terms(self._h, M, k2.shape[0], rp, ci, T, arr, G, C.ctypes.data,
                                                     int(id_group), where))
        self._keep = [k1, k2] + [v[2] for v in vs] if borrow else []
        self.M = M
        self.G, self.T = G, T

    def set_diagonals(self, diags):
        """The G right diagonals (G x n) of a general term list."""
        D = np.ascontiguousarray(diags, dtype=np.float64)
        G, n = D.shape
        self._check(self._lib.lrc_set_diagonals(self._h, n, G, D.ctypes.data, LRC_MEM_HOST))
        self.n = n

    def set_preconditioner(self, p_min: float, p_max: float, inner_steps: int):
        """Mean-based preconditioner P_T for solves with ``preconditioned=True``;
        [p_min, p_max] bounds the spectrum of P_T, inner_steps Chebyshev steps apply P_T^{-1}."""
        self._check(self._lib.lrc_set_preconditioner(self._h, float(p_min), float(p_max), int(inner_steps)))

    def set_params(self, d_mu, d_nu):
        pm, w1, k1 = _vec(d_mu, np.float64)
        pn, w2, k2 = _vec(d_nu, np.float64)
        assert w1 == w2
        self._settle(k1, k2)
        n = k1.shape[0]
        self._check(self._lib.lrc_set_params(self._h, n, pm, pn, w1))
        self.n = n

    # ------------------------------------------------------------------------------------
    def solve(self, B_U, B_V, lambda_min: float, lambda_max: float, tol: float, rank_cap: int,
              n_iter: int, restart_every: int = 0, record_iterates: bool = False,
              skip_residual: bool = False, no_graph: bool = False, warm_start: bool = True, out=None,
              preconditioned: bool = False):
        """Returns (U, V, info).  Outputs live where the inputs live (torch CUDA tensors for device
        inputs, numpy for host inputs) unless ``out=(U_out, V_out)`` is given."""
        pu, ldbu, w1, ku = _mat(B_U)
        pv, ldbv, w2, kv = _mat(B_V)
        assert w1 == w2
        r_B = ku.shape[1]
        self._order(ku, kv)
        if out is None:
            if w1 == LRC_MEM_DEVICE:
                import torch
                Uo = torch.empty((self.M, rank_cap), dtype=torch.float64, device=ku.device)
                Vo = torch.empty((self.n, rank_cap), dtype=torch.float64, device=ku.device)
            else:
                Uo = np.empty((self.M, rank_cap))
                Vo = np.empty((self.n, rank_cap))
        else:
            Uo, Vo = out
        pUo, lduo, w3, _ = _mat(Uo)
        pVo, ldvo, w4, _ = _mat(Vo)
        assert w3 == w1 and w4 == w1
        flags = ((LRC_RECORD_ITERATES if record_iterates else 0) | (LRC_SKIP_FINAL_RESIDUAL if skip_residual else 0)
                 | (LRC_NO_GRAPH if no_graph else 0) | (0 if warm_start else LRC_NO_WARM_START)
                 | (LRC_PRECONDITIONED if preconditioned else 0))
        opts = SolveOpts(float(lambda_min), float(lambda_max), float(tol), int(rank_cap), int(n_iter),
                         int(restart_every), flags)
        rh = (ctypes.c_int64 * n_iter)()
        sh = (ctypes.c_double * (n_iter * SIGMA_STRIDE))()
        info = SolveInfo()
        info.rank_history = ctypes.cast(rh, ctypes.POINTER(ctypes.c_int64))
        info.sigma_history = ctypes.cast(sh, ctypes.POINTER(ctypes.c_double))
        self._check(self._lib.lrc_solve(self._h, pu, ldbu, pv, ldbv, r_B, ctypes.byref(opts), pUo, lduo, pVo,
                                        ldvo, w1, ctypes.byref(info)))
        res = dict(rank=info.rank, rel_residual=info.rel_residual, b_norm=info.b_norm, diverged=bool(info.diverged),
                   shift_escalations=info.shift_escalations, ms_iterations=info.ms_iterations,
                   ms_total=info.ms_total, rank_history=list(rh), jacobi_sweeps=info.jacobi_sweeps, chol2_cycles=list(info.chol2_cycles),
                   sigma_history=np.frombuffer(sh, dtype=np.float64).reshape(n_iter, SIGMA_STRIDE).copy())
        return Uo, Vo, res

    def solve_gmres(self, B_U, B_V, trunc_tol: float, tol: float, rank_cap: int, restart: int = 6,
                    max_cycles: int = 10, out=None):
        """GMREST (lrc_solve_gmres): truncated restarted GMRES.  Returns (U, V, info)."""
        pu, ldbu, w1, ku = _mat(B_U)
        pv, ldbv, w2, kv = _mat(B_V)
        assert w1 == w2
        self._order(ku, kv)
        if out is None:
            if w1 == LRC_MEM_DEVICE:
                import torch
                Uo = torch.empty((self.M, rank_cap), dtype=torch.float64, device=ku.device)
                Vo = torch.empty((self.n, rank_cap), dtype=torch.float64, device=ku.device)
            else:
                Uo, Vo = np.empty((self.M, rank_cap)), np.empty((self.n, rank_cap))
        else:
            Uo, Vo = out
        pUo, lduo, _, _ = _mat(Uo)
        pVo, ldvo, _, _ = _mat(Vo)
        opts = GmresOpts(float(trunc_tol), float(tol), int(rank_cap), int(restart), int(max_cycles))
        steps = (ctypes.c_int64 * max_cycles)()
        cres = (ctypes.c_double * max_cycles)()
        info = GmresInfo()
        info.inner_steps = ctypes.cast(steps, ctypes.POINTER(ctypes.c_int64))
        info.cycle_residuals = ctypes.cast(cres, ctypes.POINTER(ctypes.c_double))
        self._check(self._lib.lrc_solve_gmres(self._h, pu, ldbu, pv, ldbv, ku.shape[1], ctypes.byref(opts), pUo, lduo,
                                              pVo, ldvo, w1, ctypes.byref(info)))
        c = int(info.cycles)
        return Uo, Vo, dict(cycles=c, rank=info.rank, rel_residual=info.rel_residual, b_norm=info.b_norm,
                            inner_steps=list(steps)[:c], cycle_residuals=list(cres)[:c])

    def solve_async(self, B_U, B_V, lambda_min: float, lambda_max: float, tol: float, rank_cap: int,
                    n_iter: int, out, restart_every: int = 0, warm_start: bool = True):
        """LRC_ASYNC solve (device tensors only): enqueues the whole solve on the context stream and
        returns; wait() completes it and returns the info dict."""
        pu, ldbu, w1, ku = _mat(B_U)
        pv, ldbv, w2, kv = _mat(B_V)
        Uo, Vo = out
        pUo, lduo, w3, _ = _mat(Uo)
        pVo, ldvo, w4, _ = _mat(Vo)
        assert w1 == w2 == w3 == w4 == LRC_MEM_DEVICE
        self._order(ku, kv)
        flags = LRC_ASYNC | (0 if warm_start else LRC_NO_WARM_START)
        opts = SolveOpts(float(lambda_min), float(lambda_max), float(tol), int(rank_cap), int(n_iter),
                         int(restart_every), flags)
        self._pending = (ku, kv, Uo, Vo, int(n_iter))
        self._check(self._lib.lrc_solve(self._h, pu, ldbu, pv, ldbv, ku.shape[1], ctypes.byref(opts), pUo, lduo,
                                        pVo, ldvo, LRC_MEM_DEVICE, None))

    def wait(self):
        n_iter = self._pending[4] if getattr(self, "_pending", None) else 1
        rh = (ctypes.c_int64 * n_iter)()
        info = SolveInfo()
        info.rank_history = ctypes.cast(rh, ctypes.POINTER(ctypes.c_int64))
        st = self._lib.lrc_solve_wait(self._h, ctypes.byref(info))
        self._pending = None
        self._check(st)
        return dict(rank=info.rank, rel_residual=info.rel_residual, b_norm=info.b_norm, diverged=bool(info.diverged),
                    ms_iterations=info.ms_iterations, ms_total=info.ms_total, rank_history=list(rh))

    def workspace_bytes(self, r_B: int, rank_cap: int, n_iter: int, record_iterates: bool = False) -> int:
        b = ctypes.c_size_t()
        self._check(self._lib.lrc_workspace_bytes(self._h, int(r_B), int(rank_cap), int(n_iter),
                                                  LRC_RECORD_ITERATES if record_iterates else 0, ctypes.byref(b)))
        return int(b.value)

    def set_workspace(self, buf):
        """Hand the context a caller-owned device buffer (e.g. a torch uint8 CUDA tensor) to carve its
        workspace from; None returns to library-owned memory."""
        if buf is None:
            self._check(self._lib.lrc_set_workspace(self._h, None, 0))
            self._ws_keep = None
            return
        self._check(self._lib.lrc_set_workspace(self._h, ctypes.c_void_p(buf.data_ptr()),
                                                buf.numel() * buf.element_size()))
        self._ws_keep = buf

    def apply_lowrank(self, U, mode: int = LRC_APPLY_PLAIN3, gamma: float = 0.0):
        pu, ldu, w, ku = _mat(U)
        r = ku.shape[1]
        nout = getattr(self, "T", 6) if mode == LRC_APPLY_SIX else getattr(self, "G", 3)
        self._order(ku)
        if w == LRC_MEM_DEVICE:
            import torch
            W = torch.empty((self.M, nout * r), dtype=torch.float64, device=ku.device)
        else:
            W = np.empty((self.M, nout * r))
        pw, ldw, _, _ = _mat(W)
        self._check(self._lib.lrc_apply_lowrank(self._h, pu, ldu, r, pw, ldw, mode, float(gamma), w))
        return W

    def apply_dense(self, S):
        ps, lds, w, ks = _mat(S)
        nc = ks.shape[1]
        self._order(ks)
        if w == LRC_MEM_DEVICE:
            import torch
            Y = torch.empty((self.M, nc), dtype=torch.float64, device=ks.device)
        else:
            Y = np.empty((self.M, nc))
        py, ldy, _, _ = _mat(Y)
        self._check(self._lib.lrc_apply_dense(self._h, ps, lds, nc, py, ldy, w))
        return Y

    def truncate(self, U, V, tol: float, cap: int):
        pu, ldu, w1, ku = _mat(U)
        pv, ldv, w2, kv = _mat(V)
        assert w1 == w2
        wdt = ku.shape[1]
        self._order(ku, kv)
        if w1 == LRC_MEM_DEVICE:
            import torch
            Uo = torch.empty((self.M, cap), dtype=torch.float64, device=ku.device)
            Vo = torch.empty((self.n, cap), dtype=torch.float64, device=ku.device)
        else:
            Uo, Vo = np.empty((self.M, cap)), np.empty((self.n, cap))
        pUo, _, _, _ = _mat(Uo)
        pVo, _, _, _ = _mat(Vo)
        rank = ctypes.c_int64()
        sig = np.zeros(SIGMA_STRIDE)
        self._check(self._lib.lrc_truncate(self._h, pu, ldu, pv, ldv, wdt, float(tol), int(cap), pUo, pVo,
                                           ctypes.byref(rank), sig.ctypes.data, w1))
        return Uo, Vo, rank.value, sig[:min(self.n, wdt)].copy()

    def get_iterate(self, k: int, rank_cap: int):
        """X_k of the last solve run with record_iterates=True, as host arrays (U, V, rank)."""
        U = np.empty((self.M, rank_cap))
        V = np.empty((self.n, rank_cap))
        r = self.get_iterate_into(k, U, V)
        return U, V, r

    def get_iterate_into(self, k: int, U, V):
        pu, _, w1, _ = _mat(U)
        pv, _, w2, _ = _mat(V)
        assert w1 == w2
        rank = ctypes.c_int64()
        self._check(self._lib.lrc_get_iterate(self._h, int(k), pu, pv, ctypes.byref(rank), w1))
        return rank.value

    def last_kernel_ms(self) -> float:
        return float(self._lib.lrc_last_kernel_ms(self._h))

    def set_reserved_sms(self, n: int):
        self._check(self._lib.lrc_set_reserved_sms(self._h, int(n)))

    def kernel_launches(self) -> int:
        return int(self._lib.lrc_kernel_launches(self._h))

    def set_profiling(self, on: bool):
        self._lib.lrc_set_profiling(self._h, 1 if on else 0)

    def profile(self) -> dict:
        """{class: (total device ms, launches)} accumulated since set_profiling(True)."""
        out = {}
        ncls = self._lib.lrc_get_profile(self._h, -1, None, None, None)
        for c in range(ncls):
            name, ms, cnt = ctypes.c_char_p(), ctypes.c_double(), ctypes.c_int64()
            self._lib.lrc_get_profile(self._h, c, ctypes.byref(name), ctypes.byref(ms), ctypes.byref(cnt))
            out[name.value.decode()] = (ms.value, cnt.value)
        return out


def solve_batch(ctxs, B_Us, B_Vs, lambda_min: float, lambda_max: float, tol: float, rank_cap: int, n_iter: int,
                outs=None, warm_start: bool = True, skip_residual: bool = False):
    """lrc_solve_batch: S contexts (sharing one borrowed operator, each with its subset's params) solved
    in lockstep with one batched SpMM per iteration.  Device tensors in and out; returns
    [(U, V, info)] per subset."""
    import torch
    S = len(ctxs)
    lib_ = ctxs[0]._lib
    P = ctypes.c_void_p
    mats_u = [_mat(b) for b in B_Us]
    mats_v = [_mat(b) for b in B_Vs]
    assert all(m[2] == LRC_MEM_DEVICE for m in mats_u + mats_v)
    r_B = mats_u[0][3].shape[1]
    for c, mu, mv in zip(ctxs, mats_u, mats_v):
        c._order(mu[3], mv[3])
    # every context stream must also see the operator / params of the first one
    for c in ctxs[1:]:
        c.stream.wait_stream(ctxs[0].stream)
        ctxs[0].stream.wait_stream(c.stream)
    if outs is None:
        outs = [(torch.empty((c.M, rank_cap), dtype=torch.float64, device=mats_u[0][3].device),
                 torch.empty((c.n, rank_cap), dtype=torch.float64, device=mats_u[0][3].device)) for c in ctxs]
    mo_u = [_mat(o[0]) for o in outs]
    mo_v = [_mat(o[1]) for o in outs]
    flags = (0 if warm_start else LRC_NO_WARM_START) | (LRC_SKIP_FINAL_RESIDUAL if skip_residual else 0)
    opts = SolveOpts(float(lambda_min), float(lambda_max), float(tol), int(rank_cap), int(n_iter), 0, flags)
    hs = (P * S)(*[c._h for c in ctxs])
    bu = (P * S)(*[m[0] for m in mats_u]); ldbu = (ctypes.c_int64 * S)(*[m[1] for m in mats_u])
    bv = (P * S)(*[m[0] for m in mats_v]); ldbv = (ctypes.c_int64 * S)(*[m[1] for m in mats_v])
    uo = (P * S)(*[m[0] for m in mo_u]); ldu = (ctypes.c_int64 * S)(*[m[1] for m in mo_u])
    vo = (P * S)(*[m[0] for m in mo_v]); ldv = (ctypes.c_int64 * S)(*[m[1] for m in mo_v])
    infos = (SolveInfo * S)()
    hists = [(ctypes.c_int64 * n_iter)() for _ in range(S)]
    for q in range(S):
        infos[q].rank_history = ctypes.cast(hists[q], ctypes.POINTER(ctypes.c_int64))
    st = lib_.lrc_solve_batch(hs, S, bu, ldbu, bv, ldbv, r_B, ctypes.byref(opts), uo, ldu, vo, ldv, LRC_MEM_DEVICE,
                              infos)
    if st != LRC_OK:
        raise LrcError(st, lib_.lrc_last_error(ctxs[0]._h).decode())
    res = []
    for q in range(S):
        inf = infos[q]
        res.append((outs[q][0], outs[q][1], dict(rank=inf.rank, rel_residual=inf.rel_residual, b_norm=inf.b_norm,
                                                 diverged=bool(inf.diverged), ms_iterations=inf.ms_iterations,
                                                 ms_total=inf.ms_total, rank_history=list(hists[q]))))
    return res


def version() -> str:
    return lib().lrc_version().decode()
