// a1 -- fused six-array CSR SpMM (`equation_intro_mat1`).
//
// One pass over the shared CSR pattern reads col_idx once and each of the six fp64 value arrays
// once, and produces the operator grouped by right diagonal (exact, Kronecker identity
// I(x)(A0+rho Jrho+lam Jlam) + Dmu(x)(A1+Jmu) + Dnu(x)(rho A2)):
//     W0 = (A0 + rho Jrho + lam Jlam) U,  W1 = (A1 + Jmu) U,  W2 = rho A2 U,
// with the Chebyshev-step epilogue W0' = U - gamma W0 fused (S2STEP).  The D_mu / D_nu scaling
// of the terms lives on the V side (n rows), never on the M side (vside kernel).
//
// Mapping: rows come in node blocks -- runs of <= 8 consecutive rows with
// identical column lists (the 5 field rows of an FE node share one list), detected at
// set_operator -- and node blocks are packed into CTA tiles of <= kSpmmCap nnz.  A CTA streams its
// tile's contiguous CSR segment (six value arrays + col_idx, coalesced, evict-first so U keeps
// L1/L2) into shared memory, combining the six arrays into the three grouped streams on the way,
// then each warp computes one node block: every U row (lanes over the r columns, read-only path)
// is loaded once per block and reused by all its rows and all three groups (15 FMA per load).
#include "lrc_internal.cuh"

namespace lrc {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

template <int MODE>
struct Nacc { static constexpr int v = (MODE == SPMM_S2STEP || MODE == SPMM_PLAIN3) ? 3 : 1; };
template <int MODE>
struct Nstage { static constexpr int v = (MODE == SPMM_SINGLE) ? 1 : 3; };

template <int MODE>
__device__ __forceinline__ void stage_entry(const SpmmArgs& a, int idx, int slot, double* s_v, double cs) {
  if constexpr (MODE == SPMM_SINGLE) {
    s_v[slot] = cs * __ldcs(a.v[a.single_t] + idx);
  } else {
    const double v0 = __ldcs(a.v[0] + idx), v1 = __ldcs(a.v[1] + idx), v2 = __ldcs(a.v[2] + idx);
    const double v3 = __ldcs(a.v[3] + idx), v4 = __ldcs(a.v[4] + idx), v5 = __ldcs(a.v[5] + idx);
    s_v[slot] = fma(a.lam, v5, fma(a.rho, v3, v0));      // A0 + rho Jrho + lam Jlam
    s_v[kSpmmCap + slot] = v1 + v4;                      // A1 + Jmu
    s_v[2 * kSpmmCap + slot] = a.rho * v2;               // rho A2
  }
}

// acc[q][t][i] += sum_j vals_t[q, j] * U[col_j, lane + 32 i] over the staged entries
template <int MODE, int NC, int GM>
__device__ __forceinline__ void block_accumulate(const SpmmArgs& a, int r, int lane, int g, int jn,
                                                 int off, int rstride, const double* s_v,
                                                 const int* s_col, const double (&dmu_c)[NC],
                                                 const double (&dnu_c)[NC],
                                                 double (&acc)[GM][Nacc<MODE>::v][NC]) {
#pragma unroll 2
  for (int j = 0; j < jn; ++j) {
    const int col = s_col[j];
    const double* urow = a.U + (size_t)col * a.ldu;
    double u[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = lane + 32 * i;
      u[i] = (c < r) ? __ldg(urow + c) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < GM; ++q) {
      if (q < g) {
        const int e = off + q * rstride + j;
        if constexpr (MODE == SPMM_S2STEP || MODE == SPMM_PLAIN3) {
          const double va = s_v[e], vb = s_v[kSpmmCap + e], vc = s_v[2 * kSpmmCap + e];
#pragma unroll
          for (int i = 0; i < NC; ++i) {
            acc[q][0][i] = fma(va, u[i], acc[q][0][i]);
            acc[q][1][i] = fma(vb, u[i], acc[q][1][i]);
            acc[q][2][i] = fma(vc, u[i], acc[q][2][i]);
          }
        } else if constexpr (MODE == SPMM_DENSE) {
          const double va = s_v[e], vb = s_v[kSpmmCap + e], vc = s_v[2 * kSpmmCap + e];
#pragma unroll
          for (int i = 0; i < NC; ++i) {
            const double coef = fma(dnu_c[i], vc, fma(dmu_c[i], vb, va));
            acc[q][0][i] = fma(coef, u[i], acc[q][0][i]);
          }
        } else {
          const double va = s_v[e];
#pragma unroll
          for (int i = 0; i < NC; ++i) acc[q][0][i] = fma(va, u[i], acc[q][0][i]);
        }
      }
    }
  }
}

template <int MODE, int NC, int GM>
__device__ __forceinline__ void block_store(const SpmmArgs& a, int r, int lane, int row0, int g,
                                            const double (&acc)[GM][Nacc<MODE>::v][NC]) {
#pragma unroll
  for (int q = 0; q < GM; ++q) {
    if (q < g) {
      const size_t row = (size_t)(row0 + q);
      double* orow = a.out + row * a.ldo + a.out_off;
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int c = lane + 32 * i;
        if (c < r) {
          if constexpr (MODE == SPMM_S2STEP) {
            const double uk = __ldg(a.U + row * a.ldu + c);
            __stcs(orow + c, fma(-a.gamma, acc[q][0][i], uk));
            __stcs(orow + r + c, acc[q][1][i]);
            __stcs(orow + 2 * r + c, acc[q][2][i]);
          } else if constexpr (MODE == SPMM_PLAIN3) {
            __stcs(orow + c, acc[q][0][i]);
            __stcs(orow + r + c, acc[q][1][i]);
            __stcs(orow + 2 * r + c, acc[q][2][i]);
          } else {
            __stcs(orow + c, acc[q][0][i]);
          }
        }
      }
    }
  }
}

template <int MODE, int NC, int GM>
__global__ void __launch_bounds__(kThreads, 2)
spmm_kernel(SpmmArgs a) {
  const int r = a.d_r ? *a.d_r : a.r_fixed;
  if (r <= 0) return;
  constexpr int NACC = Nacc<MODE>::v;
  extern __shared__ double smem_dyn[];
  double* s_v = smem_dyn;                                          // [NSTAGE][kSpmmCap]
  int* s_col = reinterpret_cast<int*>(smem_dyn + Nstage<MODE>::v * kSpmmCap);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  double dmu_c[NC], dnu_c[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int c = lane + 32 * i;
    dmu_c[i] = (MODE == SPMM_DENSE && c < r) ? a.dmu[c] : 0.0;
    dnu_c[i] = (MODE == SPMM_DENSE && c < r) ? a.dnu[c] : 0.0;
  }
  double cs = 1.0;
  if constexpr (MODE == SPMM_SINGLE)
    cs = (a.single_t == 2 || a.single_t == 3) ? a.rho : (a.single_t == 5 ? a.lam : 1.0);

  const int t = blockIdx.x;
  const int g0 = a.tile_ptr[t], g1 = a.tile_ptr[t + 1];
  const int rbeg = a.group_ptr[g0], rend = a.group_ptr[g1];
  const int e0 = a.row_ptr[rbeg], e1 = a.row_ptr[rend];
  const int tot = e1 - e0;

  if (tot <= kSpmmCap) {
    // ---- whole tile staged at once (the common case: <= 8 node blocks)
    for (int e = tid; e < tot; e += kThreads) {
      s_col[e] = __ldcs(a.col_idx + e0 + e);
      stage_entry<MODE>(a, e0 + e, e, s_v, cs);
    }
    __syncthreads();
    const int grp = g0 + warp;
    if (grp < g1) {
      const int gr0 = a.group_ptr[grp], gr1 = a.group_ptr[grp + 1];
      const int gb = a.row_ptr[gr0] - e0;
      const int L = a.row_ptr[gr0 + 1] - a.row_ptr[gr0];
      for (int sb = gr0; sb < gr1; sb += GM) {
        const int g = min(GM, gr1 - sb);
        double acc[GM][NACC][NC];
#pragma unroll
        for (int q = 0; q < GM; ++q)
#pragma unroll
          for (int tt = 0; tt < NACC; ++tt)
#pragma unroll
            for (int i = 0; i < NC; ++i) acc[q][tt][i] = 0.0;
        const int off = gb + (sb - gr0) * L;
        block_accumulate<MODE, NC, GM>(a, r, lane, g, L, off, L, s_v, s_col + gb, dmu_c, dnu_c, acc);
        block_store<MODE, NC, GM>(a, r, lane, sb, g, acc);
      }
    }
  } else {
    // ---- one group longer than the stage (generic long rows): chunks over its column list,
    //      warp 0 accumulates, the whole CTA stages
    const int L = a.row_ptr[rbeg + 1] - e0;
    for (int sb = rbeg; sb < rend; sb += GM) {
      const int g = min(GM, rend - sb);
      const int jc = kSpmmCap / g;
      double acc[GM][NACC][NC];
#pragma unroll
      for (int q = 0; q < GM; ++q)
#pragma unroll
        for (int tt = 0; tt < NACC; ++tt)
#pragma unroll
          for (int i = 0; i < NC; ++i) acc[q][tt][i] = 0.0;
      const int base = e0 + (sb - rbeg) * L;
      for (int j0 = 0; j0 < L; j0 += jc) {
        const int jn = min(jc, L - j0);
        __syncthreads();
        for (int e = tid; e < jn; e += kThreads) s_col[e] = __ldcs(a.col_idx + base + j0 + e);
        for (int e = tid; e < g * jn; e += kThreads) {
          const int q = e / jn, j = e - (e / jn) * jn;
          stage_entry<MODE>(a, base + q * L + j0 + j, q * jn + j, s_v, cs);
        }
        __syncthreads();
        if (warp == 0)
          block_accumulate<MODE, NC, GM>(a, r, lane, g, jn, 0, jn, s_v, s_col, dmu_c, dnu_c, acc);
      }
      if (warp == 0) block_store<MODE, NC, GM>(a, r, lane, sb, g, acc);
    }
  }
}

template <int MODE>
constexpr size_t smem_bytes() {
  return (size_t)kSpmmCap * (Nstage<MODE>::v * sizeof(double) + sizeof(int));
}

template <int MODE, int NC, int GM>
cudaError_t launch_t(const SpmmArgs& a, cudaStream_t s) {
  if (a.ntiles == 0) return cudaSuccess;
  spmm_kernel<MODE, NC, GM><<<a.ntiles, kThreads, smem_bytes<MODE>(), s>>>(a);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_m(const SpmmArgs& a, int rmax, cudaStream_t s) {
  if (rmax <= 32) return launch_t<MODE, 1, 8>(a, s);
  if (rmax <= 64) return launch_t<MODE, 2, 5>(a, s);
  if (rmax <= 128) return launch_t<MODE, 4, 3>(a, s);
  return cudaErrorInvalidValue;
}

template <int MODE, int NC, int GM>
cudaError_t prep_t() {
  return cudaFuncSetAttribute(spmm_kernel<MODE, NC, GM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem_bytes<MODE>());
}

template <int MODE>
cudaError_t prep_m() {
  cudaError_t e;
  if ((e = prep_t<MODE, 1, 8>()) != cudaSuccess) return e;
  if ((e = prep_t<MODE, 2, 5>()) != cudaSuccess) return e;
  return prep_t<MODE, 4, 3>();
}

}  // namespace

// Kernel attributes are set once per process/device, outside any graph capture.
cudaError_t spmm_prepare() {
  cudaError_t e;
  if ((e = prep_m<SPMM_S2STEP>()) != cudaSuccess) return e;
  if ((e = prep_m<SPMM_PLAIN3>()) != cudaSuccess) return e;
  if ((e = prep_m<SPMM_SINGLE>()) != cudaSuccess) return e;
  if ((e = prep_m<SPMM_DENSE>()) != cudaSuccess) return e;
  return prep_t<SPMM_DENSE, 8, 4>();
}

cudaError_t launch_spmm(int mode, const SpmmArgs& a, int rmax, cudaStream_t s) {
  switch (mode) {
    case SPMM_S2STEP: return launch_m<SPMM_S2STEP>(a, rmax, s);
    case SPMM_PLAIN3: return launch_m<SPMM_PLAIN3>(a, rmax, s);
    case SPMM_SINGLE: return launch_m<SPMM_SINGLE>(a, rmax, s);
    case SPMM_DENSE:
      if (rmax <= 128) return launch_m<SPMM_DENSE>(a, rmax, s);
      if (rmax <= 256) return launch_t<SPMM_DENSE, 8, 4>(a, s);
      return cudaErrorInvalidValue;
  }
  return cudaErrorInvalidValue;
}

}  // namespace lrc
