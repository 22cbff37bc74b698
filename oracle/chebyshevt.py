"""ORACLE -- plain, slow, obviously-correct CPU fp64 implementation of the truncated low-rank
ChebyshevT solve (arxiv 2008.10275).  TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
legs may import, call or execute anything under `oracle/`.  The product path
(`paper_2008_10275_b200`) never does; it shares no code, header, table or helper with
this file.  Inputs come from `synth/` (input construction only).

Citations: "P:n" = /root/reference/PAPER.md line n; "S:n" = SPEC.md line n;
readings S1..S19 = SURVEY.md §8(c) / DESIGN.md "Readings".

What is computed:
  operator (`equation_intro_mat1`):
      L(S) = A0 S + A1 S Dmu + rho_f A2 S Dnu + rho_f Jrho S + Jmu S Dmu + lambda_s Jlam S
  written as six terms  sum_t c_t A_t S diag(e_t)  with
      (c_t, e_t) = (1, 1), (1, d_mu), (rho_f, d_nu), (rho_f, 1), (1, d_mu), (lambda_s, 1).
  Chebyshev semi-iteration for a spectrum in [d - c, d + c] (P:547-569 names c, d; the
  algorithm text is in the cited [WeiBR20_ZAMM, Alg. 3], absent from the paper: reading S1):
      X_{k+1} = T( w_{k+1} [X_k + gamma (B - L(X_k))] + (1 - w_{k+1}) X_{k-1} ),
      gamma = 1/d, w_1 = 1, w_2 = 1/(1 - c^2/(2 d^2)), w_{k+1} = 1/(1 - w_k c^2/(4 d^2)).
  truncation T ("truncation operator T(.)", htucker):
      Householder QR of the left factor, SVD of the small core, keep
      r' = min(R, #{sigma_i > tau sigma_1}) (reading S5), U' = Q P_r, V' = Y_r Sigma_r.
  The concatenation is the LITERAL six-term one (8r + r_B columns); the GPU path groups
  terms by right diagonal -- both give the same X_{k+1} in exact arithmetic.

Every pin of this file is in tests/test_oracle_pins.py (closed forms, Kronecker solves,
brute-force SVD, paper examples).  The cap-bound truncated trajectory itself has no
closed form: "parity unpinned" beyond GPU-vs-oracle.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence, Tuple

import numpy as np
import scipy.sparse as sp


# --------------------------------------------------------------------------------------------
# operator  (D's P:38-40)
# --------------------------------------------------------------------------------------------
def csr_matrices(M: int, row_ptr, col_idx, vals: Sequence[np.ndarray]) -> List[sp.csr_matrix]:
    """The six M x M matrices A0, A1, A2, J_rho, J_mu, J_lambda (J is M x M, S11)."""
    return [sp.csr_matrix((np.asarray(v, dtype=np.float64), col_idx, row_ptr), shape=(M, M))
            for v in vals]


def term_list(mats, rho_f: float, lambda_s: float, d_mu, d_nu):
    """[(c_t, A_t, e_t)] of P:30-36: A0 S, A1 S Dmu, rho_f A2 S Dnu, rho_f Jrho S, Jmu S Dmu, lambda_s Jlam S.
    (Other operators of the paper: term_list_fourparam, term_list_theta, term_list_picard below.)"""
    n = len(d_mu)
    one = np.ones(n)
    d_mu = np.asarray(d_mu, dtype=np.float64)
    d_nu = np.asarray(d_nu, dtype=np.float64)
    return [
        (1.0, mats[0], one),
        (1.0, mats[1], d_mu),
        (rho_f, mats[2], d_nu),
        (rho_f, mats[3], one),
        (1.0, mats[4], d_mu),
        (lambda_s, mats[5], one),
    ]


# --------------------------------------------------------------------------------------------
# generalized term lists: every operator below is a list of terms (c_t, A_t, e_t)
# with L(S) = sum_t c_t A_t S diag(e_t), so apply_*, kron_operator and chebyshevt take them as they are
# --------------------------------------------------------------------------------------------
def term_list_general(mats, coef, diags):
    """L(S) = sum_g (sum_t C[t][g] A_t) S diag(d_g) (the library's general form): one term per array
    with the combined diagonal e_t = sum_g C[t][g] d_g."""
    coef = np.asarray(coef, dtype=np.float64)
    diags = np.asarray(diags, dtype=np.float64)
    return [(1.0, A, coef[t] @ diags) for t, A in enumerate(mats)]


def term_list_fourparam(mats, mu, nurho, lam, rho, mu_ref, nurho_ref, lam_ref):
    """The four-parameter Newton operator of P:478-482 (`equation_matrix_fourpars1`), term by term:
    A0 S + A1 S D_mu- + A2 S D_nurho- + A3 S D_lambda- + Jmu S D_mu + Jlam S D_lambda + Jrho S D_rho,
    D_x- = D_x - x_ref I; mats = [A0, A1, A2, A3, Jmu, Jlam, Jrho]."""
    one = np.ones(len(mu))
    mu, nurho, lam, rho = (np.asarray(x, dtype=np.float64) for x in (mu, nurho, lam, rho))
    return [(1.0, mats[0], one), (1.0, mats[1], mu - mu_ref), (1.0, mats[2], nurho - nurho_ref),
            (1.0, mats[3], lam - lam_ref), (1.0, mats[4], mu), (1.0, mats[5], lam), (1.0, mats[6], rho)]


def term_list_theta(mats, rho_f, lambda_s, d_mu, d_nu, mass_f, mass_s, rho_s, dt, theta):
    """The theta-scheme Newton operator of P:388-396 (`equation_timedep_matrix1`):
    (1/dt)(rho_f A_t^f + rho_s A_t^s) S + theta F(S), F the operator of P:30-36."""
    one = np.ones(len(d_mu))
    return [(rho_f / dt, mass_f, one), (rho_s / dt, mass_s, one)] + \
        [(theta * c, A, e) for (c, A, e) in term_list(mats, rho_f, lambda_s, d_mu, d_nu)]


def term_list_picard(mats, rho_f, lambda_s, mu, nu, mu_ref, nu_ref):
    """The fixed-point (Picard) operator of P:647-651 (`equation_picard_matrix1`), term by term:
    A0 X + A1 X D_mu- + rho_f A2 X D_nu- + F_mu X D_mu + lambda_s F_lam X + rho_f F_rho X;
    mats = [A0, A1, A2, F_mu, F_lam, F_rho]."""
    one = np.ones(len(mu))
    mu, nu = np.asarray(mu, dtype=np.float64), np.asarray(nu, dtype=np.float64)
    return [(1.0, mats[0], one), (1.0, mats[1], mu - mu_ref), (rho_f, mats[2], nu - nu_ref),
            (1.0, mats[3], mu), (lambda_s, mats[4], one), (rho_f, mats[5], one)]


def apply_dense(terms, S: np.ndarray) -> np.ndarray:
    """L(S) for a dense M x n S, term by term: sum_t c_t (A_t S) diag(e_t).  The A_t may
    be row blocks A_t[R, :] of the operator (then the result is L(S)[R, :])."""
    Y = np.zeros((terms[0][1].shape[0], S.shape[1]), dtype=np.float64)
    for c, A, e in terms:
        Y += c * (A @ S) * e[None, :]
    return Y


def apply_lowrank(terms, U: np.ndarray, V: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """L(U V^T) in factored form: A S D = (A U)(D V)^T for each term.

    Returns (U_L, V_L) with U_L = [A_0 U | ... | A_5 U], V_L = [c_0 e_0*V | ... | c_5 e_5*V].
    """
    Us = [A @ U for (_, A, _) in terms]
    Vs = [c * (e[:, None] * V) for (c, _, e) in terms]
    return np.hstack(Us), np.hstack(Vs)


def kron_operator(terms) -> sp.csr_matrix:
    """Vector notation: vec(L(S)) = (sum_t c_t diag(e_t) (x) A_t) vec(S),
    vec = column stacking; block-diagonal with blocks A(mu_j, nu_j)."""
    acc = None
    for c, A, e in terms:
        k = sp.kron(sp.diags(c * e), A, format="csr")
        acc = k if acc is None else acc + k
    return acc.tocsr()


def vec(S: np.ndarray) -> np.ndarray:
    """Column stacking."""
    return np.asarray(S).reshape(-1, order="F")


def unvec(s: np.ndarray, M: int) -> np.ndarray:
    """Inverse of vec."""
    return np.asarray(s).reshape(M, -1, order="F")


# --------------------------------------------------------------------------------------------
# truncation operator T (readings S5, S12, S13)
# --------------------------------------------------------------------------------------------
def truncate(U: np.ndarray, V: np.ndarray, tau: float, R: int):
    """T_{tau,R}(U V^T): Householder QR of U (LAPACK geqrf via numpy), SVD of the core C = R_u V^T.

    Returns (U', V', sigma) where sigma is the full singular-value vector of the core and
    U' V'^T is the best rank-r' approximation, r' = min(R, #{sigma_i > tau sigma_1}); r' = 0
    if sigma_1 = 0 or the factor is empty.
    """
    M, n = U.shape[0], V.shape[0]
    if U.shape[1] == 0:
        return np.zeros((M, 0)), np.zeros((n, 0)), np.zeros(0)
    Q, Ru = np.linalg.qr(U, mode="reduced")
    C = Ru @ V.T
    P, s, Yt = np.linalg.svd(C, full_matrices=False)
    if s[0] == 0.0:
        return np.zeros((M, 0)), np.zeros((n, 0)), s
    r = int(min(R, np.count_nonzero(s > tau * s[0])))
    return Q @ P[:, :r], Yt[:r].T * s[:r][None, :], s


def frobenius_lowrank(U: np.ndarray, V: np.ndarray) -> float:
    """||U V^T||_F without densifying: ||R_u V^T||_F with U = Q R_u (Householder)."""
    if U.shape[1] == 0:
        return 0.0
    _, Ru = np.linalg.qr(U, mode="reduced")
    return float(np.linalg.norm(Ru @ V.T))


# --------------------------------------------------------------------------------------------
# Chebyshev coefficients (reading S1/S2/S18)
# --------------------------------------------------------------------------------------------
def chebyshev_cd(lam_min: float, lam_max: float) -> Tuple[float, float]:
    """Interval [d - c, d + c] = [lam_min, lam_max] (reading S2): d centre, c half-width."""
    return 0.5 * (lam_max - lam_min), 0.5 * (lam_max + lam_min)


def omegas(lam_min: float, lam_max: float, N: int) -> np.ndarray:
    """w_1..w_N of the three-term recurrence: w_1 = 1, w_2 = 1/(1 - c^2/(2d^2)),
    w_{k+1} = 1/(1 - w_k c^2/(4 d^2))."""
    c, d = chebyshev_cd(lam_min, lam_max)
    w = np.empty(N)
    for k in range(N):
        if k == 0:
            w[k] = 1.0
        elif k == 1:
            w[k] = 1.0 / (1.0 - c * c / (2.0 * d * d))
        else:
            w[k] = 1.0 / (1.0 - w[k - 1] * c * c / (4.0 * d * d))
    return w


# --------------------------------------------------------------------------------------------
# ChebyshevT-S2 (reading S1, S4, S6, S7, S8)
# --------------------------------------------------------------------------------------------
@dataclasses.dataclass
class Result:
    U: np.ndarray
    V: np.ndarray
    ranks: List[int]
    sigmas: List[np.ndarray]
    iterates: List[Tuple[np.ndarray, np.ndarray]]   # X_1..X_N as factors (if recorded)
    rel_residual: float


# --------------------------------------------------------------------------------------------
# mean-based preconditioner (PAPER.md P:332-343 section "Preconditioner", LU-applied
# P:544 "the preconditioners were decomposed into a permuted LU decomposition")
# --------------------------------------------------------------------------------------------
def mean_preconditioner(terms) -> sp.csr_matrix:
    """P_T = A(x, mu_bar, nu_bar): the operator's block at the midpoint of the subset's
    parameter range, mu_bar = (min mu + max mu) / 2 (likewise nu); every right diagonal e_t of the
    term list is a parameter (or 1), so its midpoint is e_t at the mean parameters."""
    P = None
    for c, A, e in terms:
        eb = 0.5 * (float(np.min(e)) + float(np.max(e)))
        P = c * eb * A if P is None else P + c * eb * A
    return P.tocsc()


def lu_solver(P):
    """Z = P^{-1} R by a sparse permuted LU decomposition (SuperLU)."""
    import scipy.sparse.linalg as spla
    lu = spla.splu(sp.csc_matrix(P))
    return lambda R: lu.solve(np.asarray(R, dtype=np.float64)) if R.shape[1] > 0 else R


def chebyshevt_step(terms, BU, BV, Uk, Vk, Ukm1, Vkm1, omega: float, gamma: float, tau: float, R: int,
                    pinv=None):
    """One update X_{k+1} = T( w [X_k + gamma P^{-1}(B - L(X_k))] + (1 - w) X_{k-1} ) via the literal
    six-term concatenation  U = [P^{-1}B_U | U_k | P^{-1}A_0U_k ... P^{-1}A_5U_k | U_{k-1}],
    V = [w gamma B_V | w V_k | -w gamma c_t e_t*V_k ... | (1-w) V_{k-1}]  (empty blocks dropped;
    pinv = None: unpreconditioned, P = I).  (P^{-1}B_U may be passed in already applied.)"""
    Ublocks = [BU]
    Vblocks = [omega * gamma * BV]
    if Uk.shape[1] > 0:
        UL, VL = apply_lowrank(terms, Uk, Vk)
        if pinv is not None:
            UL = pinv(UL)
        Ublocks += [Uk, UL]
        Vblocks += [omega * Vk, -omega * gamma * VL]
    if Ukm1.shape[1] > 0:
        Ublocks.append(Ukm1)
        Vblocks.append((1.0 - omega) * Vkm1)
    return truncate(np.hstack(Ublocks), np.hstack(Vblocks), tau, R)


def residual(terms, BU, BV, U, V) -> float:
    """Honest relative residual ||B - L(U V^T)||_F / ||B||_F, untruncated (reading S14)."""
    nb = frobenius_lowrank(BU, BV)
    if nb == 0.0:
        return 0.0
    if U.shape[1] == 0:
        return 1.0
    UL, VL = apply_lowrank(terms, U, V)
    return frobenius_lowrank(np.hstack([BU, UL]), np.hstack([BV, -VL])) / nb


def chebyshevt(terms, BU, BV, lam_min: float, lam_max: float, tau: float, R: int, N: int,
               record_iterates: bool = True, final_residual: bool = True,
               restart_every: Optional[int] = None, on_iterate=None, precond=None) -> Result:
    """N updates X_1..X_N from X_0 = X_{-1} = 0 (readings S6, S7).  Optional restart (S8,
    P:546 'restarted once after 6 iterations'): the w sequence restarts with X_{-1} := X_k.
    on_iterate(k, U_k, V_k, sigma) (optional, no arithmetic) sees every X_k as it is produced,
    so a caller can keep selected iterates of a long solve without recording all of them.
    precond = P_T: the preconditioned iteration on P^{-1} L with the
    spectrum bounds [lam_min, lam_max] of P^{-1} L, P^{-1} by LU (lu_solver); the reported residual
    stays the honest unpreconditioned ||B - L(X_N)|| / ||B||."""
    M, n = BU.shape[0], BV.shape[0]
    pinv = lu_solver(precond) if precond is not None else None
    BU_step = pinv(BU) if pinv is not None else BU
    c, d = chebyshev_cd(lam_min, lam_max)
    gamma = 1.0 / d
    w_all = omegas(lam_min, lam_max, N)
    Uk, Vk = np.zeros((M, 0)), np.zeros((n, 0))
    Ukm1, Vkm1 = np.zeros((M, 0)), np.zeros((n, 0))
    ranks, sigmas, iterates = [], [], []
    j = 0
    for k in range(N):
        if restart_every and k > 0 and k % restart_every == 0:
            j = 0
            Ukm1, Vkm1 = Uk, Vk
        Un, Vn, s = chebyshevt_step(terms, BU_step, BV, Uk, Vk, Ukm1, Vkm1, w_all[j], gamma, tau, R, pinv)
        j += 1
        Ukm1, Vkm1, Uk, Vk = Uk, Vk, Un, Vn
        ranks.append(Un.shape[1])
        sigmas.append(s)
        if on_iterate is not None:
            on_iterate(k + 1, Un, Vn, s)
        if record_iterates:
            iterates.append((Un, Vn))
    rho = residual(terms, BU, BV, Uk, Vk) if final_residual else float("nan")
    return Result(Uk, Vk, ranks, sigmas, iterates, rho)


# --------------------------------------------------------------------------------------------
# GMREST: truncated restarted GMRES (named P:41, run P:513, restarted
# once after 6 iterations P:546; algorithm text absent from the paper -- DESIGN.md reading R14:
# Arnoldi with modified Gram-Schmidt on the low-rank iterates, every operator application and every
# linear combination truncated by T, the small Hessenberg least-squares problem solved densely)
# --------------------------------------------------------------------------------------------
GMRES_BREAKDOWN = 1e-14     # h_{j+1,j} <= 1e-14 max_i |h_ij| counts as a breakdown (reading R14)


def inner(U1: np.ndarray, V1: np.ndarray, U2: np.ndarray, V2: np.ndarray) -> float:
    """Frobenius inner product <U1 V1^T, U2 V2^T> = tr((U1^T U2)(V2^T V1))."""
    if U1.shape[1] == 0 or U2.shape[1] == 0:
        return 0.0
    return float(np.sum((U1.T @ U2) * (V1.T @ V2)))


@dataclasses.dataclass
class GmresResult:
    U: np.ndarray
    V: np.ndarray
    cycles: int
    inner_steps: List[int]              # Arnoldi steps per cycle
    cycle_residuals: List[float]        # honest relative residual after every cycle
    rel_residual: float
    hessenbergs: List[np.ndarray]


def gmrest(terms, BU, BV, tau: float, R: int, m: int, max_cycles: int, tol: float) -> GmresResult:
    """Restarted GMRES(m) on L(X) = B with low-rank iterates (reading R14).  Per cycle:
    R0 = T(B - L(X)), beta = ||R0||, V_1 = R0 / beta; for j = 1..m: W = T(L(V_j)); for i = 1..j:
    h_ij = <W, V_i>, W = T(W - h_ij V_i); h_{j+1,j} = ||W||; V_{j+1} = W / h_{j+1,j} (stop at a
    breakdown h_{j+1,j} <= 1e-14 max_i |h_ij|); y = argmin ||beta e_1 - H y||; X = T(... T(T(X + y_1 V_1) + y_2 V_2) ...).
    Stops when the honest relative residual ||B - L(X)||_F / ||B||_F <= tol or after max_cycles."""
    M, n = BU.shape[0], BV.shape[0]
    XU, XV = np.zeros((M, 0)), np.zeros((n, 0))
    steps, res, Hs = [], [], []
    bnorm = frobenius_lowrank(BU, BV)
    if bnorm == 0.0:
        return GmresResult(XU, XV, 0, [], [], 0.0, [])
    rho = 1.0
    cyc = 0
    for cyc in range(1, max_cycles + 1):
        if XU.shape[1] == 0:
            RU, RV, _ = truncate(BU, BV, tau, R)
        else:
            UL, VL = apply_lowrank(terms, XU, XV)
            RU, RV, _ = truncate(np.hstack([BU, UL]), np.hstack([BV, -VL]), tau, R)
        beta = frobenius_lowrank(RU, RV)
        if beta == 0.0:
            break
        basis = [(RU, RV / beta)]
        H = np.zeros((m + 1, m))
        k = 0
        for j in range(m):
            Uj, Vj = basis[j]
            UL, VL = apply_lowrank(terms, Uj, Vj)
            WU, WV, _ = truncate(UL, VL, tau, R)
            for i in range(j + 1):
                Ui, Vi = basis[i]
                h = inner(WU, WV, Ui, Vi)
                H[i, j] = h
                WU, WV, _ = truncate(np.hstack([WU, Ui]), np.hstack([WV, -h * Vi]), tau, R)
            hn = frobenius_lowrank(WU, WV)
            H[j + 1, j] = hn
            k = j + 1
            if hn <= GMRES_BREAKDOWN * np.max(np.abs(H[:j + 2, j])):   # (happy) breakdown
                H[j + 1, j] = 0.0
                break
            basis.append((WU, WV / hn))
        e1 = np.zeros(k + 1)
        e1[0] = beta
        y = np.linalg.lstsq(H[:k + 1, :k], e1, rcond=None)[0]
        for j in range(k):
            Uj, Vj = basis[j]
            XU, XV, _ = truncate(np.hstack([XU, Uj]), np.hstack([XV, y[j] * Vj]), tau, R)
        steps.append(k)
        Hs.append(H[:k + 1, :k].copy())
        rho = residual(terms, BU, BV, XU, XV)
        res.append(rho)
        if rho <= tol:
            break
    return GmresResult(XU, XV, cyc, steps, res, rho, Hs)


def dense_product(U: np.ndarray, V: np.ndarray) -> np.ndarray:
    return U @ V.T
