/*
 * lrcheb.h -- C ABI of the B200-native truncated low-rank ChebyshevT solver ("liblrcheb").
 *
 * What is solved (equation `equation_intro_mat1`; the Newton step on one
 * parameter subset, P:251-256 / reading S3 of DESIGN.md):
 *
 *     A0 S + A1 S Dmu + rho_f A2 S Dnu + rho_f Jrho S + Jmu S Dmu + lambda_s Jlam S = B,
 *
 * with B = B_U B_V^T of low rank, S = U V^T kept factored,
 * the six M x M sparse matrices sharing one CSR pattern, Dmu = diag(d_mu),
 * Dnu = diag(d_nu) the parameters of the subset.  The solver is the truncated
 * Chebyshev semi-iteration "ChebyshevT" (named P:14; parameters c, d
 * P:547-569; the iteration itself is DESIGN.md reading S1) with the truncation operator T of
 * P:544 (best rank-r' approximation, r' = min(cap, #{sigma_i > tol * sigma_1}), reading S5).
 *
 * Conventions (all calls):
 *   - fp64 everywhere; every dense factor is ROW-MAJOR with an explicit leading dimension
 *     counted in elements (ld >= number of columns).
 *   - CSR: row_ptr int32[M+1] (row_ptr[0] = 0, non-decreasing, row_ptr[M] = nnz),
 *     col_idx int32[nnz] with 0 <= col < M, strictly increasing inside a row.
 *   - `where` says where caller pointers live: LRC_MEM_HOST (pageable or pinned host memory;
 *     the library copies), LRC_MEM_DEVICE (device memory on ctx's device; inputs are copied
 *     into ctx-owned memory, outputs are written in place), LRC_MEM_DEVICE_BORROW (set_operator
 *     only: the library keeps the caller's device pointers; the caller keeps them alive and
 *     unchanged until the next set_operator or lrc_destroy).
 *   - Every call returns an lrc_status; nothing throws or exits.  On error the outputs are
 *     untouched and lrc_last_error(ctx) holds a one-line message.  (lrc_solve: an error found on
 *     the device -- LRC_ERR_NUMERIC -- still fills *info for diagnosis; U_out / V_out are not
 *     written.  SPEC S:508's "best iterate" of a diverging run is the OK case info->diverged = 1.)
 *   - All work is ordered on ctx's stream; calls return after the work completed (host
 *     synchronous) unless stated otherwise.  One ctx per host thread; no internal locking.
 *
 * Limits of this build (checked, LRC_ERR_ARG otherwise): M < 2^31, nnz < 2^31,
 *   rank_cap <= 128, r_B <= 64, min(n, r_B + (G + 1) rank_cap) <= 112 (G = 3 right-diagonal
 *   groups for the operator of P:30-36), r_B + (G + 1) rank_cap <= 256, n <= 1024,
 *   lrc_apply_dense: ncols <= 256.
 */
#ifndef LRCHEB_H
#define LRCHEB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lrc_ctx lrc_ctx;

typedef enum {
  LRC_OK = 0,
  LRC_ERR_ARG = 1,      /* invalid argument (null pointer, bad CSR, bad bounds, over a limit) */
  LRC_ERR_SHAPE = 2,    /* shapes inconsistent with the operator / parameters already set */
  LRC_ERR_STATE = 3,    /* call order: solve before set_operator + set_params, etc. */
  LRC_ERR_NOMEM = 4,    /* device allocation failed */
  LRC_ERR_CUDA = 5,     /* a CUDA runtime error (message has the CUDA error string) */
  LRC_ERR_NUMERIC = 6   /* shifted Cholesky failed after all shift escalations */
} lrc_status;

typedef enum { LRC_MEM_HOST = 0, LRC_MEM_DEVICE = 1, LRC_MEM_DEVICE_BORROW = 2 } lrc_mem;

/* lrc_solve_opts.flags */
#define LRC_RECORD_ITERATES      1u  /* keep every X_k = U_k V_k^T on the device for lrc_get_iterate */
#define LRC_SKIP_FINAL_RESIDUAL  2u  /* do not compute info->rel_residual (set to NaN) */
#define LRC_NO_GRAPH             4u  /* launch the iteration kernels directly instead of a CUDA graph */
#define LRC_NO_WARM_START        8u  /* start every core Jacobi SVD from W = I (default: warm start from the
                                        previous iteration's right singular basis when p == n) */
#define LRC_ASYNC               16u  /* DEVICE inputs/outputs only: lrc_solve returns once the work is
                                        enqueued on ctx's stream; lrc_solve_wait completes the call */
#define LRC_PRECONDITIONED      32u  /* iterate on P^{-1} L with the mean-based preconditioner of
                                        lrc_set_preconditioner (lambda_min/max then bound P^{-1} L) */

/* lrc_apply_lowrank modes */
#define LRC_APPLY_PLAIN3  0u  /* W = [W0 | W1 | W2], W0 = (A0+rho Jrho+lam Jlam)U, W1 = (A1+Jmu)U, W2 = rho A2 U */
#define LRC_APPLY_SIX     1u  /* W = [c_0 A0 U | c_1 A1 U | ... | c_5 Jlam U], (c_t) = (1,1,rho,rho,1,lam) */
#define LRC_APPLY_S2STEP  2u  /* W = [U - gamma W0 | W1 | W2]  (the fused Chebyshev-step epilogue) */

/* Context lifetime.  device: CUDA ordinal; cuda_stream: a cudaStream_t on that device to order
 * all work on, or NULL for a ctx-owned non-blocking stream. */
lrc_status  lrc_create(lrc_ctx **out, int device, void *cuda_stream);
void        lrc_destroy(lrc_ctx *ctx);                 /* NULL-safe; frees everything ctx owns */
const char *lrc_last_error(const lrc_ctx *ctx);        /* valid until the next call on ctx */
const char *lrc_version(void);

/* The operator: shared CSR pattern + six value arrays in the order
 * A0, A1, A2, Jrho, Jmu, Jlambda (zeros stored explicitly where a matrix has no entry),
 * and the scalars rho_f, lambda_s.  Validates the CSR (LRC_ERR_ARG on a violation) and
 * detects runs of consecutive rows with identical column lists (node blocks, <= 8 rows)
 * that the fused SpMM exploits.  Invalidates parameters and workspaces that depend on M. */
lrc_status lrc_set_operator(lrc_ctx *ctx, int64_t M, int64_t nnz,
                            const int32_t *row_ptr, const int32_t *col_idx,
                            const double *const vals[6], double rho_f, double lambda_s,
                            lrc_mem where);

/* General term list: the four-parameter operator of P:478-482
 * (A0 S + A1 S D_mu- + A2 S D_nurho- + A3 S D_lambda- + Jmu S Dmu + Jlam S Dlam + Jrho S Drho), the
 * theta-scheme mass term of P:388-396, the Picard operators of P:647-651 -- any
 *     L(S) = sum_{g < G} ( sum_{t < T} coef[t*G + g] A_t ) S diag(d_g)
 * with T <= 8 value arrays on the shared CSR pattern (same rules as lrc_set_operator), G <= 6 right
 * diagonals (set by lrc_set_diagonals), at most 6 nonzero coefficients per group, and one group
 * id_group whose diagonal is the identity (it carries the Chebyshev step U - gamma W).  The solve
 * then concatenates w = r_B + (G + 1) rank_cap columns (<= 256).  Runs on the persistent TMA SpMM
 * only: LRC_ERR_ARG unless the pattern forms FE node-block tiles (<= 900 nnz, <= 90 U rows,
 * <= 4 row runs) -- true for the synthetic FE operators of BASELINE.json.  lrc_apply_lowrank then
 * writes G blocks (PLAIN3 / S2STEP, r <= 64) or T blocks A_t U (SIX); lrc_apply_dense is unavailable. */
lrc_status lrc_set_operator_terms(lrc_ctx *ctx, int64_t M, int64_t nnz, const int32_t *row_ptr,
                                  const int32_t *col_idx, int T, const double *const *vals, int G,
                                  const double *coef, int id_group, lrc_mem where);

/* The right diagonals of a general term list: diags is G x n row-major (row g = d_g, finite; row
 * id_group all ones).  Replaces lrc_set_params for such an operator. */
lrc_status lrc_set_diagonals(lrc_ctx *ctx, int64_t n, int G, const double *diags, lrc_mem where);

/* The subset's parameters: d_mu, d_nu of length n (finite). where: HOST or DEVICE. */
lrc_status lrc_set_params(lrc_ctx *ctx, int64_t n, const double *d_mu, const double *d_nu,
                          lrc_mem where);

/* Mean-based preconditioner ("Preconditioner"): P_T = the operator's
 * block at the midpoint of the subset's parameter range, P_T = sum_t c_t A_t * (min e_t + max e_t) / 2
 * over the current parameters (lrc_set_params / lrc_set_diagonals; setting them again discards the
 * preconditioner).  A solve with LRC_PRECONDITIONED runs
 *     X_{k+1} = T( w [X_k + gamma P_T^{-1}(B - L(X_k))] + (1 - w) X_{k-1} ),
 * the factor concatenation [P^{-1}B_U | U_k - gamma P^{-1}W0 | P^{-1}W1 | ... | U_{k-1}], with
 * lambda_min/lambda_max bounding the spectrum of P_T^{-1} L; info->rel_residual stays the
 * unpreconditioned ||B - L(X_N)||_F / ||B||_F.  The paper applies P_T^{-1} by a permuted LU;
 * here every P_T^{-1} R is inner_steps steps of a Chebyshev semi-iteration on P_T with its spectrum in
 * [p_min, p_max] (reading R15: error <= 2 q^inner_steps with
 * q = (sqrt(p_max) - sqrt(p_min)) / (sqrt(p_max) + sqrt(p_min)) relative to ||P_T^{-1} R||, for P_T
 * symmetric positive definite).  0 < p_min <= p_max, 1 <= inner_steps <= 1000; LRC_ERR_STATE before
 * the operator and parameters are set. */
lrc_status lrc_set_preconditioner(lrc_ctx *ctx, double p_min, double p_max, int64_t inner_steps);

typedef struct {
  double lambda_min, lambda_max;  /* spectrum bounds [d-c, d+c] (reading S2); 0 < min <= max */
  double tol;                     /* relative truncation tolerance tau >= 0 (reading S5) */
  int64_t rank_cap;               /* R, 1 <= R <= min(M, n, 128) */
  int64_t n_iter;                 /* N >= 1 updates X_1..X_N from X_0 = 0 (readings S6, S7) */
  int64_t restart_every;          /* 0: no restart; else the omega sequence restarts every k iterations (S8) */
  uint32_t flags;                 /* LRC_RECORD_ITERATES | LRC_SKIP_FINAL_RESIDUAL | LRC_NO_GRAPH | LRC_NO_WARM_START */
} lrc_solve_opts;

typedef struct {
  int64_t rank;               /* rank of X_N */
  double rel_residual;        /* ||B - L(X_N)||_F / ||B||_F (0 if B = 0; NaN if skipped) */
  double b_norm;              /* ||B||_F */
  int32_t diverged;           /* 1 if rel_residual > 1 (last iterate still returned) */
  int32_t shift_escalations;  /* total shift escalations in the Cholesky passes */
  float ms_iterations;        /* device time of the N iterations (CUDA events) */
  float ms_total;             /* device time of the whole call */
  int64_t *rank_history;      /* caller array[n_iter] or NULL: rank of X_1..X_N */
  double *sigma_history;      /* caller array[n_iter * 128] or NULL: core singular values per
                                 iteration, descending, zero padded */
  int64_t jacobi_sweeps;      /* total one-sided Jacobi sweeps over all truncations of the call */
  double chol2_cycles[3];     /* SM cycles in the core step: Cholesky + R, Jacobi, rank/Z/V' (summed) */
} lrc_solve_info;

/* Solve F(S) = B for the current operator/params.
 * B_U: M x r_B (ld_bu), B_V: n x r_B (ld_bv); r_B may be 0 (then X = 0, rank 0, residual 0).
 * Outputs: U_out M x rank_cap (ld_u >= rank_cap), V_out n x rank_cap (ld_v >= rank_cap);
 * columns >= info->rank are set to 0.  U has orthonormal columns, V = Y Sigma (reading S12).
 * where: HOST (pointers are host memory; copies are inside the call) or DEVICE.
 * info may be NULL.
 * Device workspace (kept in ctx between calls, reallocated when a shape grows): about
 * 8 * M * (r_B + 3 rank_cap + 3 rank_cap + pmax) bytes plus small buffers, pmax = 8 ceil(min(n,
 * r_B + 4 rank_cap) / 8) -- B_U, the three grouped SpMM outputs, three rotating U factors and
 * Y = Ucat R_V^T of the truncation (about 4.8 GB on BASELINE's Large config). */
lrc_status lrc_solve(lrc_ctx *ctx,
                     const double *B_U, int64_t ld_bu, const double *B_V, int64_t ld_bv, int64_t r_B,
                     const lrc_solve_opts *opts,
                     double *U_out, int64_t ld_u, double *V_out, int64_t ld_v,
                     lrc_mem where, lrc_solve_info *info);

/* Batched lockstep solve of S (1..4) parameter subsets (Algorithm 1's loop
 * over the subsets I_k, P:304-327 -- the subsets are independent given the operator).
 * ctxs[q] holds subset q's parameters (lrc_set_params) and all contexts borrow the SAME operator
 * arrays (lrc_set_operator with LRC_MEM_DEVICE_BORROW on identical device pointers; LRC_ERR_ARG
 * otherwise).  Every iteration reads the operator once for all S subsets' U factors (one batched
 * fused SpMM on ctxs[0]'s stream) and then runs the S truncations concurrently on the contexts'
 * own streams.  Per subset q: B_U[q] (ld_bu[q]), B_V[q] (ld_bv[q]), outputs U_out[q] / V_out[q]
 * (ld_u[q], ld_v[q]) and infos[q] (infos may be NULL) exactly as lrc_solve.  r_B >= 1 and the same
 * opts for all; LRC_ASYNC / LRC_NO_GRAPH / LRC_RECORD_ITERATES are not supported here.  Returns the
 * first error of any subset (outputs of a failing subset untouched, as lrc_solve). */
lrc_status lrc_solve_batch(lrc_ctx *const *ctxs, int S, const double *const *B_U, const int64_t *ld_bu,
                           const double *const *B_V, const int64_t *ld_bv, int64_t r_B,
                           const lrc_solve_opts *opts, double *const *U_out, const int64_t *ld_u,
                           double *const *V_out, const int64_t *ld_v, lrc_mem where, lrc_solve_info *infos);

/* Completes a solve started with LRC_ASYNC: waits for ctx's stream, fills *info (may be NULL) and
 * returns the solve's status (LRC_ERR_STATE if no solve is pending).  The caller keeps B_U, B_V,
 * U_out and V_out alive until then.  A pending solve is also completed (info discarded) by the
 * next lrc_solve / lrc_set_workspace on ctx. */
lrc_status lrc_solve_wait(lrc_ctx *ctx, lrc_solve_info *info);

/* Workspace ownership.  By default ctx allocates its solve workspace (cudaMalloc) and keeps it
 * between calls.  lrc_workspace_bytes returns the bytes a solve with (r_B, rank_cap, n_iter,
 * flags & LRC_RECORD_ITERATES) needs for the current operator / params; lrc_set_workspace hands ctx
 * a caller-owned device buffer (256-byte aligned, on ctx's device; the caller keeps it alive until
 * the next lrc_set_workspace or lrc_destroy) that all later workspaces are carved from (NULL: back
 * to library-owned memory).  A solve that does not fit the buffer fails with LRC_ERR_NOMEM.  The
 * test hooks (lrc_apply_*, lrc_truncate) keep their own library-owned scratch. */
lrc_status lrc_workspace_bytes(lrc_ctx *ctx, int64_t r_B, int64_t rank_cap, int64_t n_iter, uint32_t flags,
                               size_t *bytes);
lrc_status lrc_set_workspace(lrc_ctx *ctx, void *dev_ptr, size_t bytes);

/* GMREST -- truncated restarted GMRES (named P:41, run P:513, "restarted
 * once after 6 iterations" P:546; reading R14): GMRES(restart) on L(S) = B with every Krylov
 * basis element and the iterate held as U V^T, T_{trunc_tol, rank_cap} applied after every
 * operator application and every modified Gram-Schmidt / update step; the (restart+1) x restart
 * Hessenberg least-squares problem is solved on the host.  Stops when the honest relative residual
 * ||B - L(X)||_F / ||B||_F <= tol or after max_cycles restart cycles.  Outputs as lrc_solve (U_out
 * M x rank_cap, V_out n x rank_cap, columns >= rank zero).  Host-synchronous (no graph): each Arnoldi
 * step reads its coefficients back.  rank_cap <= 64, 1 <= restart <= 32, r_B >= 1. */
typedef struct {
  double trunc_tol;      /* tau of the truncation operator */
  double tol;            /* stopping tolerance on the honest relative residual */
  int64_t rank_cap;      /* R */
  int64_t restart;       /* Arnoldi steps per cycle m */
  int64_t max_cycles;    /* restart cycles */
} lrc_gmres_opts;

typedef struct {
  int64_t cycles;              /* restart cycles run */
  int64_t rank;                /* rank of X */
  double rel_residual;         /* honest relative residual of X */
  double b_norm;               /* ||B||_F */
  int64_t *inner_steps;        /* caller array[max_cycles] or NULL: Arnoldi steps per cycle */
  double *cycle_residuals;     /* caller array[max_cycles] or NULL: honest residual after each cycle */
} lrc_gmres_info;

lrc_status lrc_solve_gmres(lrc_ctx *ctx, const double *B_U, int64_t ld_bu, const double *B_V, int64_t ld_bv,
                           int64_t r_B, const lrc_gmres_opts *opts, double *U_out, int64_t ld_u,
                           double *V_out, int64_t ld_v, lrc_mem where, lrc_gmres_info *info);

/* Test / bench hooks (same ctx state; where = HOST or DEVICE for all pointers of the call). */

/* W = L-pieces of U (M x r, ld_u): mode LRC_APPLY_PLAIN3 / LRC_APPLY_S2STEP write M x 3r,
 * LRC_APPLY_SIX writes M x 6r into W (ld_w).  gamma is used by S2STEP only.  r <= 128. */
lrc_status lrc_apply_lowrank(lrc_ctx *ctx, const double *U, int64_t ld_u, int64_t r,
                             double *W, int64_t ld_w, uint32_t mode, double gamma, lrc_mem where);

/* Dense operator application (BASELINE config 5): Y = sum_t c_t A_t S diag(e_t) for a dense
 * S (M x ncols, ld_s), with e_t in {1, d_mu, d_nu} taken from the params (n == ncols). */
lrc_status lrc_apply_dense(lrc_ctx *ctx, const double *S, int64_t ld_s, int64_t ncols,
                           double *Y, int64_t ld_y, lrc_mem where);

/* Truncation operator T_{tol,cap}(U V^T): U M x w (ld_u), V n x w (ld_v), w <= 256.
 * Writes U_out M x cap (ld cap), V_out n x cap (ld cap), *rank, and sigma (min(n,w) values,
 * descending) if non-NULL. */
lrc_status lrc_truncate(lrc_ctx *ctx, const double *U, int64_t ld_u, const double *V, int64_t ld_v,
                        int64_t w, double tol, int64_t cap,
                        double *U_out, double *V_out, int64_t *rank, double *sigma, lrc_mem where);

/* Iterate X_k (1 <= k <= n_iter) of the last solve run with LRC_RECORD_ITERATES:
 * U (M x rank_cap, ld rank_cap), V (n x rank_cap, ld rank_cap), *rank. */
lrc_status lrc_get_iterate(lrc_ctx *ctx, int64_t k, double *U, double *V, int64_t *rank, lrc_mem where);

/* Device time (ms, CUDA events on ctx's stream) of the last lrc_apply_lowrank / lrc_apply_dense
 * call's kernel, for the bench's SpMM roofline. */
float lrc_last_kernel_ms(const lrc_ctx *ctx);

/* Concurrent subset solves: the persistent M-level kernels of this ctx use
 * (SM count - n) CTAs so that n SMs stay free for the single-CTA core steps of other contexts
 * solving other subsets on other streams (subsets are independent).  Default 0. */
lrc_status lrc_set_reserved_sms(lrc_ctx *ctx, int n);

/* Number of liblrcheb kernels launched on ctx so far (a graph replay counts its kernel nodes). */
int64_t lrc_kernel_launches(const lrc_ctx *ctx);

/* Per-kernel-class profiling with CUDA events on the launching stream (bench roofline pass).
 * on != 0 resets the accumulators and makes lrc_solve launch directly (no graph) with an event
 * pair around every kernel.  lrc_get_profile(ctx, cls, &name, &ms, &count) returns the number of
 * classes and, for 0 <= cls < that number, the class name, its accumulated device ms and launch
 * count (classes: spmm, vside_qr, ts_gram, gram_reduce, chol1, chol2_svd, ts_store, trace, misc). */
void lrc_set_profiling(lrc_ctx *ctx, int on);
int  lrc_get_profile(const lrc_ctx *ctx, int cls, const char **name, double *ms_total, int64_t *count);

#ifdef __cplusplus
}
#endif
#endif /* LRCHEB_H */
