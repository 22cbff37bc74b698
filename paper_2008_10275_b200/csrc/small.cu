// a2 / a3 / a4 / a5 -- the small dense steps of one ChebyshevT iteration, one CTA each
// (DESIGN.md "Truncation").  All operands are <= 112 x 256 and live in shared
// memory; everything is fp64.
//
//   vside      : Vcat = [w g B_V | w V_k | -w g d_mu*V_k | -w g d_nu*V_k | (1-w) V_{k-1}] (n x w,
//                the D_mu/D_nu scaling is applied on the V side only), then its
//                Householder QR  Vcat = Q_V [R_V; 0]  (p = min(n, w)).  Writes T1 = R_V^T (w x p)
//                and Q_V[:, :p] (n x p).  X = Ucat Vcat^T = (Ucat R_V^T) Q_V^T, so the left factor
//                to re-orthogonalise is Y = Ucat R_V^T (M x p, formed and stored by Gram pass 1).
//   chol1      : R1 = chol(G1 + s1 I), s1 = delta tr(G1) (escalated x100 on breakdown), and
//                R1^{-1} (pass 2 then forms Q1 = Y R1^{-1} tile by tile from the stored Y).
//   chol2_svd  : R2 = chol(G2 + s2 I) (s2 = 0 first, escalated on breakdown), R = R2 R1,
//                one-sided (Hestenes) Jacobi SVD R = P Sigma W^T, rank rule
//                r' = min(cap, #{sigma_i > tol sigma_1}) (reading S5), and
//                Wz = W_r Sigma_r^{-1} (so U_{k+1} = Y Wz = Q_Y P_r),  V_{k+1} = Q_V W_r Sigma_r.
#include <cmath>
#include "lrc_internal.cuh"

namespace lrc {

namespace {

constexpr int kT = 1024;
constexpr double kShiftRel = 1e-12;   // pass-1 shift s1 = kShiftRel * tr(G1)  (reading S17')
constexpr int kMaxEsc = 3;            // escalations x100
constexpr double kJacobiTol = 1e-14;  // rotate while |a_i.a_j| > tol ||a_i|| ||a_j||
constexpr double kJacobiFloor = 1e-30;   // (1e-15)^2: column-norm^2 floor relative to ||R||_F^2
constexpr int kMaxSweeps = 40;
constexpr int kJacE = 7;              // Jacobi elements per lane of a pair (16 lanes, p <= 112)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// In-place upper Cholesky of the p x p row-major matrix a (stride ld) after adding `shift` to the
// diagonal.  Returns true on success.  Called by all threads of the CTA.  One barrier per column: the
// trailing update of step j uses the unscaled row j (a[i][c] -= a[j][i] a[j][c] / a[j][j]), and the
// rows are scaled by 1/sqrt(a[j][j]) once at the end.  Threads form a 32 x (blockDim/32) grid over the
// trailing triangle (no integer division in the update).
__device__ bool chol_upper(double* a, int ld, int p, double shift, int* s_fail) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, ny = blockDim.x >> 5;
  for (int i = threadIdx.x; i < p; i += blockDim.x) a[i * ld + i] += shift;
  __syncthreads();
  for (int j = 0; j < p; ++j) {
    const double d = a[j * ld + j];
    if (!(d > 0.0) || !isfinite(d)) {       // uniform across the CTA
      if (threadIdx.x == 0) *s_fail = 1;
      __syncthreads();
      return false;
    }
    const double invd = 1.0 / d;
    const double* rj = a + j * ld;
    for (int i = j + 1 + ty; i < p; i += ny) {
      const double f = rj[i] * invd;
      double* ri = a + i * ld;
      for (int c = i + tx; c < p; c += 32) ri[c] = fma(-f, rj[c], ri[c]);
    }
    __syncthreads();
  }
  // scale: R[j][c] = a[j][c] / sqrt(a[j][j]) (c > j), R[j][j] = sqrt(a[j][j])
  for (int j = ty; j < p; j += ny) {
    const double d = a[j * ld + j], r = sqrt(d), inv = 1.0 / r;
    for (int c = j + 1 + tx; c < p; c += 32) a[j * ld + c] *= inv;
    if (tx == 0) a[j * ld + j] = r;
  }
  if (threadIdx.x == 0) *s_fail = 0;
  __syncthreads();
  return true;
}

// X = R^{-1} (R upper triangular p x p, row-major stride ld; X the same layout, upper), bottom-up with
// one barrier per row: row k of X is final once every row below it has been folded into the running
// sums acc[k][j] = sum_{l > k} R[k][l] X[l][j]; X[k][j] = (delta_kj - acc[k][j]) / R[k][k].
__device__ void tri_inv_upper(const double* R, int ld, double* X, int p) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, ny = blockDim.x >> 5;
  for (int e = threadIdx.x; e < p * ld; e += blockDim.x) X[e] = 0.0;
  __syncthreads();
  // k = p - 1: row p-1 final right away
  if (threadIdx.x == 0) X[(p - 1) * ld + (p - 1)] = 1.0 / R[(p - 1) * ld + (p - 1)];
  __syncthreads();
  for (int k = p - 1; k >= 1; --k) {
    // fold row k into the rows i < k; the threads owning row k - 1 finish it in the same pass
    const double* xk = X + k * ld;
    for (int i = ty; i < k; i += ny) {
      const double rik = R[i * ld + k];
      double* xi = X + i * ld;
      if (i == k - 1) {
        const double inv = 1.0 / R[i * ld + i];
        for (int j = i + tx; j < p; j += 32) {
          const double acc = (j >= k) ? fma(rik, xk[j], xi[j]) : xi[j];
          xi[j] = ((j == i) ? 1.0 - acc : -acc) * inv;
        }
      } else {
        for (int j = k + tx; j < p; j += 32) xi[j] = fma(rik, xk[j], xi[j]);
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------
// vside: build Vcat, Householder QR, write T1 = R_V^T and Q_V
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kT) vside_kernel(VDesc d, int n, const double* __restrict__ dtab,
                                                   const double* __restrict__ omega, int k,
                                                   State st, SmallBufs b, int ncols_alloc) {
  extern __shared__ double sm[];
  const int NL = n | 1;                     // odd column stride: conflict-free column walks
  double* s_v = sm;                         // column-major [ncols_alloc][NL]
  __shared__ double s_tau[kMaxP];
  __shared__ int s_off[kMaxUBlocks + 1];
  const int tid = threadIdx.x;

  if (tid == 0) {
    int off = 0;
    for (int bi = 0; bi < d.nb; ++bi) {
      const VBlock& B = d.b[bi];
      const int wdt = B.w_fixed + (B.w_idx >= 0 ? B.w_mul * st.rk[B.w_idx] : 0);
      s_off[bi] = off;
      off += d.pad_even ? wdt + (wdt & 1) : wdt;     // zero pad column (see UDesc::pad_even)
    }
    s_off[d.nb] = off;
  }
  __syncthreads();
  const int w = s_off[d.nb];
  const int p = min(n, w);
  if (tid == 0) { *st.w = w; *st.p = p; }
  if (w == 0) return;

  const double om = omega ? omega[k] : 1.0;
  for (int bi = 0; bi < d.nb; ++bi) {
    const VBlock& B = d.b[bi];
    const int o = s_off[bi], wlog = s_off[bi + 1] - o;
    const int wdt = B.w_fixed + (B.w_idx >= 0 ? B.w_mul * st.rk[B.w_idx] : 0);
    const double sc = B.use_omega == 0 ? B.scale : (B.use_omega == 1 ? B.scale * om : B.scale * (1.0 - om));
    for (int e = tid; e < wlog * n; e += kT) {
      const int c = e / n, i = e - (e / n) * n;
      double v = 0.0;                                   // pad column: exactly zero
      if (c < wdt) {
        v = sc * B.ptr[(size_t)i * B.ld + c];
        if (B.diag >= 0) v *= dtab[(size_t)B.diag * n + i];   // right diagonal d_g (general: f4)
      }
      s_v[(o + c) * NL + i] = v;
    }
  }
  __syncthreads();

  // Householder QR (LAPACK dgeqr2 convention: H_j = I - tau v v^T, v_j = 1)
  const int lane = tid & 31;
  for (int j = 0; j < p; ++j) {
    if (tid < 32) {
      double* x = s_v + j * NL;
      double ss = 0.0;
      for (int i = j + 1 + lane; i < n; i += 32) ss += x[i] * x[i];
      ss = warp_sum(ss);
      const double alpha = x[j];
      double tau = 0.0, beta = alpha, scal = 0.0;
      if (ss > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + ss), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      __syncwarp();
      for (int i = j + 1 + lane; i < n; i += 32) x[i] *= scal;
      if (lane == 0) { x[j] = beta; s_tau[j] = tau; }
    }
    __syncthreads();
    const double tau = s_tau[j];
    if (tau != 0.0) {
      const double* v = s_v + j * NL;
      const int part = tid & 3;
      // 4 lanes per column, 8 columns per warp; the loop bound is warp-uniform (shuffles)
      for (int cb = j + 1 + (tid >> 5) * 8; cb < w; cb += kT / 4) {
        const int c = cb + ((tid >> 2) & 7);
        const bool act = c < w;
        double* col = s_v + (act ? c : 0) * NL;
        double dot = (act && part == 0) ? col[j] : 0.0;
        if (act)
          for (int i = j + 1 + part; i < n; i += 4) dot += v[i] * col[i];
        dot += __shfl_xor_sync(0xffffffffu, dot, 1);
        dot += __shfl_xor_sync(0xffffffffu, dot, 2);
        dot *= tau;
        if (act) {
          if (part == 0) col[j] -= dot;
          for (int i = j + 1 + part; i < n; i += 4) col[i] -= dot * v[i];
        }
      }
    }
    __syncthreads();
  }
  // T1 = R_V^T  (w x ldT), R_V[i][c] = s_v[c][i] for i <= c, i < p
  for (int e = tid; e < w * b.ldT; e += kT) {
    const int c = e / b.ldT, i = e - (e / b.ldT) * b.ldT;
    b.T1[(size_t)c * b.ldT + i] = (i < p && i <= c) ? s_v[c * NL + i] : 0.0;
  }
  // Q_V[:, :p] explicitly (dorg2r), stored in columns [p, 2p) of s_v (host guarantees room)
  double* s_q = s_v + p * NL;
  __syncthreads();
  for (int e = tid; e < p * n; e += kT) {
    const int c = e / n, i = e - (e / n) * n;
    s_q[c * NL + i] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = p - 1; j >= 0; --j) {
    const double tau = s_tau[j];
    if (tau != 0.0) {
      const double* v = s_v + j * NL;
      const int part = tid & 3;
      for (int cb = j + (tid >> 5) * 8; cb < p; cb += kT / 4) {
        const int c = cb + ((tid >> 2) & 7);
        const bool act = c < p;
        double* col = s_q + (act ? c : 0) * NL;
        double dot = (act && part == 0) ? col[j] : 0.0;
        if (act)
          for (int i = j + 1 + part; i < n; i += 4) dot += v[i] * col[i];
        dot += __shfl_xor_sync(0xffffffffu, dot, 1);
        dot += __shfl_xor_sync(0xffffffffu, dot, 2);
        dot *= tau;
        if (act) {
          if (part == 0) col[j] -= dot;
          for (int i = j + 1 + part; i < n; i += 4) col[i] -= dot * v[i];
        }
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < n * b.ldT; e += kT) {
    const int i = e / b.ldT, c = e - (e / b.ldT) * b.ldT;
    b.QV[(size_t)i * b.ldT + c] = (c < p) ? s_q[c * NL + i] : 0.0;
  }
}

// ------------------------------------------------------------------------------------------
// chol1: R1 = chol(G1 + s1 I); R1^{-1}
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kT) chol1_kernel(State st, SmallBufs b, int pmax) {
  extern __shared__ double sm[];
  const int LD = pmax + 1;
  double* s_r = sm;                               // row-major [pmax][LD]
  __shared__ int s_fail;
  __shared__ double s_tr;
  const int tid = threadIdx.x;
  const int p = *st.p;
  if (p <= 0) return;
  if (tid == 0) {
    double tr = 0.0;
    for (int i = 0; i < p; ++i) tr += b.G[i * pmax + i];
    s_tr = tr;
  }
  __syncthreads();
  double shift = kShiftRel * s_tr;
  if (!(shift > 0.0)) shift = 1.0;               // G1 == 0 (X == 0): any positive shift
  bool ok = false;
  for (int att = 0; att <= kMaxEsc && !ok; ++att) {
    for (int e = tid; e < p * p; e += kT) {
      const int i = e / p, c = e - (e / p) * p;
      s_r[i * LD + c] = b.G[i * pmax + c];
    }
    __syncthreads();
    ok = chol_upper(s_r, LD, p, shift, &s_fail);
    if (!ok) {
      if (tid == 0) atomicAdd(st.esc, 1);
      shift *= 100.0;
    }
    __syncthreads();
  }
  if (!ok) {                                     // give up: flag, continue with R1 = I
    if (tid == 0) atomicOr(st.flags, 1);
    for (int e = tid; e < p * p; e += kT) {
      const int i = e / p, c = e - (e / p) * p;
      s_r[i * LD + c] = (i == c) ? 1.0 : 0.0;
    }
    __syncthreads();
  }
  // keep R1 (upper, zero below) and the shift actually used (for the core step's floor correction)
  for (int e = tid; e < pmax * pmax; e += kT) {
    const int i = e / pmax, c = e - (e / pmax) * pmax;
    b.R1[e] = (i < p && c < p && c >= i) ? s_r[i * LD + c] : 0.0;
  }
  if (tid == 0) st.scal[2] = ok ? shift : 0.0;
  __syncthreads();
  double* s_x = sm + pmax * LD;                  // R1^{-1}
  tri_inv_upper(s_r, LD, s_x, p);
  // R1^{-1} (upper, zero outside p x p) -> global: the T matrix of Gram pass 2 (Q1 = Y R1^{-1})
  for (int e = tid; e < pmax * pmax; e += kT) {
    const int i = e / pmax, c = e - (e / pmax) * pmax;
    b.R1i[e] = (i < p && c < p && c >= i) ? s_x[i * LD + c] : 0.0;
  }
}

// ------------------------------------------------------------------------------------------
// chol2 + Jacobi SVD + rank rule + Z, V'
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kT) chol2_svd_kernel(State st, SmallBufs b, int pmax, int n,
                                                       double tol, int cap, int rank_slot,
                                                       int sigma_row, double* __restrict__ Vout,
                                                       int ldv) {
  extern __shared__ double sm[];
  const int LD = pmax + 1;
  double* s_a = sm;                  // column-major A = R, [pmax][LD]
  double* s_w = sm + pmax * LD;      // row-major R2 scratch, then column-major W
  __shared__ double s_sig[kMaxP];
  __shared__ int s_perm[kMaxP];
  __shared__ int s_fail, s_rot, s_rank;
  __shared__ double s_tr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p = *st.p;
  if (p <= 0) {
    if (tid == 0) st.rk[rank_slot] = 0;
    for (int e = tid; e < n * cap; e += kT) Vout[(e / cap) * (size_t)ldv + e % cap] = 0.0;
    return;
  }
  if (tid == 0) {
    double tr = 0.0;
    for (int i = 0; i < p; ++i) tr += b.G[i * pmax + i];
    s_tr = tr;
  }
  __syncthreads();
  long long tclk0 = clock64();
  // R2 = chol(G2 + s2 I): unshifted first (keeps R^T R = X^T X exactly), then escalate
  double shift = 0.0;
  bool ok = false;
  for (int att = 0; att <= kMaxEsc + 1 && !ok; ++att) {
    for (int e = tid; e < p * p; e += kT) {
      const int i = e / p, c = e - (e / p) * p;
      s_w[i * LD + c] = b.G[i * pmax + c];
    }
    __syncthreads();
    ok = chol_upper(s_w, LD, p, shift, &s_fail);
    if (!ok) {
      if (tid == 0 && att > 0) atomicAdd(st.esc, 1);
      shift = (att == 0) ? kShiftRel * s_tr : shift * 100.0;
      if (!(shift > 0.0)) shift = 1.0;
    }
    __syncthreads();
  }
  if (!ok) {
    if (tid == 0) atomicOr(st.flags, 1);
    for (int e = tid; e < p * p; e += kT) {
      const int i = e / p, c = e - (e / p) * p;
      s_w[i * LD + c] = (i == c) ? 1.0 : 0.0;
    }
    __syncthreads();
  }
  const double s2_used = ok ? shift : 0.0;
  // R1 (row-major) -> s_a
  for (int e = tid; e < p * p; e += kT) {
    const int i = e / p, c = e - (e / p) * p;
    s_a[i * LD + c] = b.R1[i * pmax + c];
  }
  __syncthreads();
  // R = R2 R1, one warp per row, in place in s_w (row i of R needs only row i of R2)
  for (int i = warp; i < p; i += kT / 32) {
    double acc[kMaxP / 32];
#pragma unroll
    for (int t = 0; t < kMaxP / 32; ++t) acc[t] = 0.0;
    for (int k = i; k < p; ++k) {
      const double r2 = s_w[i * LD + k];
#pragma unroll
      for (int t = 0; t < kMaxP / 32; ++t) {
        const int j = lane + 32 * t;
        if (j < p) acc[t] = fma(r2, s_a[k * LD + j], acc[t]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < kMaxP / 32; ++t) {
      const int j = lane + 32 * t;
      if (j < p) s_w[i * LD + j] = (j >= i) ? acc[t] : 0.0;
    }
  }
  __syncthreads();
  // Jacobi start.  Cold: A = R, W = I.  Warm (p == n in this and the previous iteration): the previous
  // right singular basis B = Q_V,prev W_prev of X in R^n maps into the new coordinates exactly
  // orthogonally, W0 = Q_V^T B (tiny_gemm on the V-side stream), and A0 = R W0 is nearly column-
  // orthogonal once the iteration settles, so far fewer sweeps are needed (R9).
  const bool warm = (b.W0 != nullptr) && (*st.prevp == n) && (p == n);
  double* A = s_a;
  double* Wm = s_w;
  if (warm) {
    for (int e = tid; e < p * p; e += kT) {
      const int i = e / p, c = e - (e / p) * p;
      s_a[i * LD + c] = b.W0[i * pmax + c];
    }
    __syncthreads();
    for (int i = warp; i < p; i += kT / 32) {     // A0 = R W0, row i in place (R upper triangular)
      double acc[kMaxP / 32];
#pragma unroll
      for (int t = 0; t < kMaxP / 32; ++t) acc[t] = 0.0;
      for (int k = i; k < p; ++k) {
        const double rk = s_w[i * LD + k];
#pragma unroll
        for (int t = 0; t < kMaxP / 32; ++t) {
          const int j = lane + 32 * t;
          if (j < p) acc[t] = fma(rk, s_a[k * LD + j], acc[t]);
        }
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < kMaxP / 32; ++t) {
        const int j = lane + 32 * t;
        if (j < p) s_w[i * LD + j] = acc[t];
      }
    }
    __syncthreads();
    for (int e = tid; e < p * p; e += kT) {        // in-place transposes -> column-major
      const int i = e / p, j = e - (e / p) * p;
      if (i < j) {
        double t0 = s_w[i * LD + j]; s_w[i * LD + j] = s_w[j * LD + i]; s_w[j * LD + i] = t0;
        double t1 = s_a[i * LD + j]; s_a[i * LD + j] = s_a[j * LD + i]; s_a[j * LD + i] = t1;
      }
    }
    A = s_w;
    Wm = s_a;
    __syncthreads();
  } else {
    for (int e = tid; e < p * p; e += kT) {          // column-major A = R
      const int i = e / p, j = e - (e / p) * p;
      s_a[j * LD + i] = s_w[i * LD + j];
    }
    __syncthreads();
    for (int e = tid; e < p * p; e += kT) {
      const int j = e / p, i = e - (e / p) * p;
      s_w[j * LD + i] = (i == j) ? 1.0 : 0.0;
    }
  }
  if (warp == 0) {
    double ss = 0.0;
    for (int e = lane; e < p * p; e += 32) {
      const double x = A[(e / p) * LD + (e % p)];
      ss += x * x;
    }
    ss = warp_sum(ss);
    if (lane == 0) s_tr = ss;
  }
  __syncthreads();
  long long tclk1 = clock64();

  // One-sided (Hestenes) Jacobi on the columns of R, round-robin ordering, 16 lanes per pair
  // (all p/2 pairs of a round in flight at once).  Columns whose squared norm is below
  // kJacobiFloor ||R||_F^2 are rounding noise and are not rotated.
  const double floor2 = kJacobiFloor * s_tr;
  const double tol2 = kJacobiTol * kJacobiTol;
  const int half = lane >> 4, hl = lane & 15;
  const int P = p + (p & 1), NP = P / 2;
  // only the warps that own pairs (two per warp) take part; they synchronise on a named barrier
  const int nwj = (NP + 1) / 2;
  const unsigned jbar = 32u * (unsigned)nwj;
  int sweeps_done = 0;
  if (warp < nwj) {
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    ++sweeps_done;
    if (tid == 0) s_rot = 0;
    asm volatile("bar.sync 1, %0;\n" ::"r"(jbar) : "memory");
    for (int r = 0; r < P - 1; ++r) {
      for (int qb = warp * 2; qb < NP; qb += kT / 16) {
        const int q = qb + half;
        int i = 0, j = 0;
        bool act = q < NP;
        if (act) {
          if (q == 0) { i = P - 1; j = r; }
          else { i = (r + q) % (P - 1); j = (r - q + P - 1) % (P - 1); }
          act = (i < p) && (j < p);
          if (i > j) { const int t = i; i = j; j = t; }
        }
        double* ai = A + i * LD;
        double* aj = A + j * LD;
        // the pair's two columns in registers (p <= 112, the host-checked limit: <= 7 elements per lane),
        // read once per round
        double xa[kJacE], ya[kJacE];
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int t = 0; t < kJacE; ++t) {
          const int e = hl + 16 * t;
          const bool in = act && e < p;
          xa[t] = in ? ai[e] : 0.0;
          ya[t] = in ? aj[e] : 0.0;
          al = fma(xa[t], xa[t], al); be = fma(ya[t], ya[t], be); ga = fma(xa[t], ya[t], ga);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (act && ga != 0.0 && al > floor2 && be > floor2 && ga * ga > tol2 * al * be) {
          // tan of the rotation angle, smaller root: t = sgn(d) 2g / (|d| + sqrt(d^2 + 4 g^2))
          const double dd = be - al;
          const double t = ((dd >= 0.0) ? 2.0 * ga : -2.0 * ga) / (fabs(dd) + sqrt(fma(dd, dd, 4.0 * ga * ga)));
          const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
#pragma unroll
          for (int t = 0; t < kJacE; ++t) {
            const int e = hl + 16 * t;
            if (e < p) {
              ai[e] = c * xa[t] - sn * ya[t];
              aj[e] = sn * xa[t] + c * ya[t];
            }
          }
          double* wi = Wm + i * LD;
          double* wj = Wm + j * LD;
          for (int e = hl; e < p; e += 16) {
            const double x = wi[e], y = wj[e];
            wi[e] = c * x - sn * y;
            wj[e] = sn * x + c * y;
          }
          if (hl == 0) s_rot = 1;
        }
      }
      asm volatile("bar.sync 1, %0;\n" ::"r"(jbar) : "memory");
    }
    const int rot = s_rot;
    asm volatile("bar.sync 1, %0;\n" ::"r"(jbar) : "memory");
    if (rot == 0) break;
  }
  }
  __syncthreads();   // the idle warps rejoin here
  if (tid == 0) atomicAdd(st.sweeps, sweeps_done);
  long long tclk2 = clock64();
  // singular values of R, then of X:  R^T R = (1 + s2) X^T X + s1 s2 I  (exact for the shifted
  // CholeskyQR2; same singular vectors), so sigma_X^2 = (sigma_R^2 - s1 s2) / (1 + s2).
  const double s1s2 = st.scal[2] * s2_used;
  for (int j = warp; j < p; j += kT / 32) {
    const double* aj = A + j * LD;
    double ss = 0.0;
    for (int e = lane; e < p; e += 32) ss += aj[e] * aj[e];
    ss = warp_sum(ss);
    if (lane == 0) s_sig[j] = sqrt(fmax(ss - s1s2, 0.0) / (1.0 + s2_used));
  }
  __syncthreads();
  if (tid < p) {
    const double sj = s_sig[tid];
    int rk = 0;
    for (int i = 0; i < p; ++i) {
      const double si = s_sig[i];
      rk += (si > sj) || (si == sj && i < tid);
    }
    s_perm[rk] = tid;
  }
  __syncthreads();
  if (tid == 0) {
    const double s1 = s_sig[s_perm[0]];
    int r = 0;
    if (!isfinite(s1)) {
      atomicOr(st.flags, 2);
    } else if (s1 > 0.0) {
      for (int i = 0; i < p; ++i) r += (s_sig[s_perm[i]] > tol * s1);
      r = min(r, cap);
    }
    s_rank = r;
    st.rk[rank_slot] = r;
  }
  __syncthreads();
  const int rr = s_rank;
  if (sigma_row >= 0)
    for (int i = tid; i < kSigmaStride; i += kT)
      st.sigma[(size_t)sigma_row * kSigmaStride + i] = (i < p) ? s_sig[s_perm[i]] : 0.0;
  // Wz = W_r Sigma_r^{-1} (basis pass U' = Y Wz), Wv = W_r Sigma_r (V' = Q_V Wv), p x ldZ
  for (int e = tid; e < pmax * b.ldZ; e += kT) {
    const int k = e / b.ldZ, q = e - (e / b.ldZ) * b.ldZ;
    double wz = 0.0, wv = 0.0;
    if (q < rr && k < p) {
      const int jq = s_perm[q];
      const double wk = Wm[jq * LD + k];
      wz = wk / s_sig[jq];
      wv = wk * s_sig[jq];
    }
    b.Wz[e] = wz;
    b.Wv[e] = wv;
  }
  if (b.Wfull) {                                   // full right basis W (for the next warm start)
    for (int e = tid; e < pmax * pmax; e += kT) {
      const int i = e / pmax, j = e - (e / pmax) * pmax;
      b.Wfull[e] = (i < p && j < p) ? Wm[j * LD + i] : 0.0;
    }
  }
  if (tid == 0) *st.prevp = p;
  __syncthreads();
  if (tid == 0 && st.scal) {   // phase cycle counters (DESIGN.md profiling notes)
    long long tclk3 = clock64();
    atomicAdd(st.scal + 4, (double)(tclk1 - tclk0));
    atomicAdd(st.scal + 5, (double)(tclk2 - tclk1));
    atomicAdd(st.scal + 6, (double)(tclk3 - tclk2));
  }
}

// C (m x ncols, ldc) = A (m x k, lda) B (k x ncols, ldb); m, k device-resident or fixed.  8 rows of C
// per CTA; the A rows are staged in shared memory, B rows stream from L2 coalesced.
__global__ void __launch_bounds__(256) tiny_gemm_kernel(const double* __restrict__ A, int lda,
                                                         const double* __restrict__ B, int ldb,
                                                         double* __restrict__ C, int ldc, int ncols,
                                                         const int* d_m, int m_fixed, const int* d_k,
                                                         int k_fixed, int transA) {
  const int m = d_m ? *d_m : m_fixed;
  const int k = d_k ? *d_k : k_fixed;
  const int r0 = blockIdx.x * 8;
  if (r0 >= m) return;
  __shared__ double s_a[8][kMaxW];
  const int rows = min(8, m - r0);
  for (int e = threadIdx.x; e < 8 * k; e += 256) {
    const int i = e / k, kk = e - (e / k) * k;
    s_a[i][kk] = (i < rows) ? (transA ? A[(size_t)kk * lda + r0 + i] : A[(size_t)(r0 + i) * lda + kk]) : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < rows * ncols; e += 256) {
    const int i = e / ncols, c = e - (e / ncols) * ncols;
    double acc = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < k; ++kk) acc = fma(s_a[i][kk], __ldg(B + (size_t)kk * ldb + c), acc);
    C[(size_t)(r0 + i) * ldc + c] = acc;
  }
}

__global__ void trace_kernel(State st, const double* __restrict__ G, int pmax, int slot) {
  const int p = *st.p;
  double s = 0.0;
  for (int i = threadIdx.x; i < p; i += 32) s += G[i * pmax + i];
  s = warp_sum(s);
  if (threadIdx.x == 0) st.scal[slot] = (p > 0) ? s : 0.0;
}

__global__ void fill_int_kernel(int* p, int v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void zero_cols_kernel(double* X, int rows, int ld, const int* d_r, int r_fixed, int cols) {
  const int r = d_r ? *d_r : r_fixed;
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)rows * cols) return;
  const int i = (int)(e / cols), c = (int)(e % cols);
  if (c >= r) X[(size_t)i * ld + c] = 0.0;
}

// dst (rows x cols, ld_dst) = src with the columns >= *d_rank zeroed -- unless *flags != 0 (an
// error was flagged on the device), in which case dst is left untouched
__global__ void copy_out_kernel(const double* __restrict__ src, int ld_src, double* __restrict__ dst,
                                int ld_dst, int rows, int cols, const int* d_rank, const int* flags) {
  if (*flags) return;
  const int r = *d_rank;
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)rows * cols) return;
  const int i = (int)(e / cols), c = (int)(e % cols);
  dst[(size_t)i * ld_dst + c] = (c < r) ? src[(size_t)i * ld_src + c] : 0.0;
}

// the mean-based preconditioner P_T: its values on the shared pattern,
// p = sum_t e_t v_t (e_t = the term's coefficient times its right diagonal at the mean parameters)
__global__ void form_pvals_kernel(PvalArgs pa, int T, long long nnz, double* __restrict__ p) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  double acc = 0.0;
  for (int t = 0; t < T; ++t) acc = fma(pa.e[t], pa.v[t][i], acc);
  p[i] = acc;
}

// one step of the inner Chebyshev semi-iteration for P Z = R on nb blocks (rows x ncols, ld, block
// stride bs): Zout = w (Zc + g (R - Y)) + (1 - w) Zp with Y = P Zc (Zp null: Z_0 = 0); first: Zout = g R
__global__ void cheb_inner_kernel(int nb, int rows, int ncols, int ld, long long bs, const double* __restrict__ R,
                                  const double* __restrict__ Y, const double* __restrict__ Zc,
                                  const double* __restrict__ Zp, double* __restrict__ Zout, double w, double g,
                                  int first, const int* __restrict__ d_r, int r_fixed) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per = (long long)rows * ncols;
  if (e >= per * nb) return;
  const int b = (int)(e / per);
  const long long q = e - (long long)b * per;
  const int i = (int)(q / ncols), c = (int)(q - (long long)(q / ncols) * ncols);
  if (c >= (d_r ? *d_r : r_fixed)) return;        // columns past the rank (and the zero pad) untouched
  const long long o = (long long)b * bs + (long long)i * ld + c;
  Zout[o] = first ? g * R[o] : fma(w, fma(g, R[o] - Y[o], Zc[o]), (1.0 - w) * (Zp ? Zp[o] : 0.0));
}

// W = U - g W (the Chebyshev-step block of the preconditioned iteration), rows x ncols, ld
__global__ void s2_update_kernel(int rows, int ncols, int ld, const double* __restrict__ U, int ldu,
                                 double* __restrict__ W, double g) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)rows * ncols) return;
  const int i = (int)(e / ncols), c = (int)(e - (e / ncols) * ncols);
  W[(size_t)i * ld + c] = fma(-g, W[(size_t)i * ld + c], U[(size_t)i * ldu + c]);
}

template <typename K>
cudaError_t set_smem(K kern, size_t bytes) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, kern);
  if (e != cudaSuccess) return e;
  const size_t room = bytes > fa.sharedSizeBytes ? bytes - fa.sharedSizeBytes : 0;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)room);
}

}  // namespace

cudaError_t small_prepare() {
  constexpr size_t kMax = 232448;
  cudaError_t e;
  if ((e = set_smem(vside_kernel, kMax)) != cudaSuccess) return e;
  if ((e = set_smem(chol1_kernel, kMax)) != cudaSuccess) return e;
  return set_smem(chol2_svd_kernel, kMax);
}

cudaError_t launch_tiny_gemm(const double* A, int lda, const double* B, int ldb, double* C, int ldc,
                             int ncols, const int* d_m, int m_fixed, int m_max, const int* d_k,
                             int k_fixed, cudaStream_t s, int transA) {
  if (m_max <= 0 || ncols <= 0) return cudaSuccess;
  tiny_gemm_kernel<<<(m_max + 7) / 8, 256, 0, s>>>(A, lda, B, ldb, C, ldc, ncols, d_m, m_fixed, d_k,
                                                    k_fixed, transA);
  return cudaGetLastError();
}

size_t vside_smem_bytes(int n, int wmax, int pmax) {
  const int NL = n | 1;
  const int cols = wmax > 2 * pmax ? wmax : 2 * pmax;
  return sizeof(double) * (size_t)NL * cols;
}

cudaError_t launch_vside(const VDesc& d, int n, const double* dtab,
                         const double* omega, int k, State st, SmallBufs b, int wmax,
                         cudaStream_t s) {
  const int pmax = b.ldT;
  const size_t smem = vside_smem_bytes(n, wmax, pmax);
  vside_kernel<<<1, kT, smem, s>>>(d, n, dtab, omega, k, st, b, 0);
  return cudaGetLastError();
}

cudaError_t launch_chol1(State st, SmallBufs b, int pmax, int wmax, cudaStream_t s) {
  (void)wmax;
  const size_t smem = sizeof(double) * 2 * (size_t)pmax * (pmax + 1);
  chol1_kernel<<<1, kT, smem, s>>>(st, b, pmax);
  return cudaGetLastError();
}

cudaError_t launch_chol2_svd(State st, SmallBufs b, int pmax, int wmax, int n, double tol,
                             int cap, int rank_slot, int sigma_row, double* Vout, int ldv,
                             cudaStream_t s) {
  (void)wmax;
  const size_t smem = sizeof(double) * 2 * (size_t)pmax * (pmax + 1);
  chol2_svd_kernel<<<1, kT, smem, s>>>(st, b, pmax, n, tol, cap, rank_slot, sigma_row, Vout, ldv);
  return cudaGetLastError();
}

cudaError_t launch_trace(State st, const double* G, int pmax, int slot, cudaStream_t s) {
  trace_kernel<<<1, 32, 0, s>>>(st, G, pmax, slot);
  return cudaGetLastError();
}

cudaError_t launch_fill_int(int* p, int v, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  fill_int_kernel<<<(n + 255) / 256, 256, 0, s>>>(p, v, n);
  return cudaGetLastError();
}

cudaError_t launch_copy_out(const double* src, int ld_src, double* dst, int ld_dst, int rows, int cols,
                            const int* d_rank, const int* flags, cudaStream_t s) {
  const size_t tot = (size_t)rows * cols;
  if (tot == 0) return cudaSuccess;
  copy_out_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(src, ld_src, dst, ld_dst, rows, cols, d_rank, flags);
  return cudaGetLastError();
}

cudaError_t launch_form_pvals(const PvalArgs& pa, int T, long long nnz, double* p, cudaStream_t s) {
  if (nnz <= 0) return cudaSuccess;
  form_pvals_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(pa, T, nnz, p);
  return cudaGetLastError();
}

cudaError_t launch_cheb_inner(int nb, int rows, int ncols, int ld, long long bs, const double* R, const double* Y,
                              const double* Zc, const double* Zp, double* Zout, double w, double g, int first,
                              const int* d_r, int r_fixed, cudaStream_t s) {
  const long long tot = (long long)nb * rows * ncols;
  if (tot == 0) return cudaSuccess;
  cheb_inner_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(nb, rows, ncols, ld, bs, R, Y, Zc, Zp, Zout, w, g,
                                                                   first, d_r, r_fixed);
  return cudaGetLastError();
}

cudaError_t launch_s2_update(int rows, int ncols, int ld, const double* U, int ldu, double* W, double g,
                             cudaStream_t s) {
  const long long tot = (long long)rows * ncols;
  if (tot == 0) return cudaSuccess;
  s2_update_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(rows, ncols, ld, U, ldu, W, g);
  return cudaGetLastError();
}

cudaError_t launch_zero_cols(double* X, int rows, int ld, const int* d_r, int r_fixed, int cols,
                             cudaStream_t s) {
  const size_t tot = (size_t)rows * cols;
  if (tot == 0) return cudaSuccess;
  zero_cols_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(X, rows, ld, d_r, r_fixed, cols);
  return cudaGetLastError();
}

}  // namespace lrc
