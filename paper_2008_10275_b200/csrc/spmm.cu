// a1 -- fused six-array CSR SpMM (`equation_intro_mat1`).
//
// One pass over the shared CSR pattern reads col_idx once and each of the six fp64 value arrays
// once, and produces the operator grouped by right diagonal (exact, Kronecker identity
// I(x)(A0+rho Jrho+lam Jlam) + Dmu(x)(A1+Jmu) + Dnu(x)(rho A2)):
//     W0 = (A0 + rho Jrho + lam Jlam) U,  W1 = (A1 + Jmu) U,  W2 = rho A2 U,
// with the Chebyshev-step epilogue W0' = U - gamma W0 fused (S2STEP).  The D_mu / D_nu scaling
// of the terms lives on the V side (n rows), never on the M side (vside kernel).
//
// Layout / mapping: rows are processed in node blocks -- runs of <= 8 consecutive
// rows with identical column lists (the 5 field rows of an FE node share one list) -- one warp
// per block.  The warp stages the block's column indices and the *combined* values a, b, c
// (3 doubles per nnz, combined on the fly from the six streamed arrays) in shared memory with
// fully coalesced loads of the contiguous CSR segment, then every staged U row (lanes over the
// r columns, __ldg, 256 B coalesced) is reused by all rows of the block and all three groups.
#include "lrc_internal.cuh"

namespace lrc {

namespace {

constexpr int kWarps = 8;
constexpr int kStage = 256;   // staged nnz entries per warp per chunk (g * jc <= kStage)

template <int MODE, int NC, int GM>
__global__ void __launch_bounds__(kWarps * 32)
spmm_kernel(SpmmArgs a) {
  const int r = a.d_r ? *a.d_r : a.r_fixed;
  if (r <= 0) return;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int grp = blockIdx.x * kWarps + wid;
  if (grp >= a.ngroups) return;

  constexpr int NV = (MODE == SPMM_SINGLE) ? 1 : 3;   // staged value streams
  extern __shared__ double smem_dyn[];
  double (*s_val)[NV][kStage] = reinterpret_cast<double (*)[NV][kStage]>(smem_dyn);
  int (*s_col)[kStage] = reinterpret_cast<int (*)[kStage]>(smem_dyn + kWarps * NV * kStage);

  const int row_begin = a.group_ptr[grp];
  const int row_end = a.group_ptr[grp + 1];
  const int base0 = a.row_ptr[row_begin];
  const int L = a.row_ptr[row_begin + 1] - base0;   // common row length of the block

  // per-lane columns c = lane + 32*i, i < NC
  double dmu_c[MODE == SPMM_DENSE ? NC : 1], dnu_c[MODE == SPMM_DENSE ? NC : 1];
  if constexpr (MODE == SPMM_DENSE) {
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = lane + 32 * i;
      dmu_c[i] = (c < r) ? a.dmu[c] : 0.0;
      dnu_c[i] = (c < r) ? a.dnu[c] : 0.0;
    }
  }
  const double rho = a.rho, lam = a.lam;
  double cs = 1.0;
  if constexpr (MODE == SPMM_SINGLE) {
    cs = (a.single_t == 2 || a.single_t == 3) ? rho : (a.single_t == 5 ? lam : 1.0);
  }

  for (int sb = row_begin; sb < row_end; sb += GM) {          // sub-blocks of <= GM rows
    const int g = min(GM, row_end - sb);
    const int base = base0 + (sb - row_begin) * L;
    constexpr int NACC = (MODE == SPMM_S2STEP || MODE == SPMM_PLAIN3) ? 3 : 1;
    double acc[GM][NACC][NC];
#pragma unroll
    for (int q = 0; q < GM; ++q)
#pragma unroll
      for (int t = 0; t < NACC; ++t)
#pragma unroll
        for (int i = 0; i < NC; ++i) acc[q][t][i] = 0.0;

    const int jc = kStage / g;     // entries of each row per chunk
    for (int j0 = 0; j0 < L; j0 += jc) {
      const int jn = min(jc, L - j0);
      __syncwarp();
      for (int e = lane; e < jn; e += 32) s_col[wid][e] = __ldg(a.col_idx + base + j0 + e);
      const int tot = g * jn;
      for (int e = lane; e < tot; e += 32) {
        const int q = e / jn;
        const int j = e - q * jn;
        const int idx = base + q * L + j0 + j;
        if constexpr (MODE == SPMM_SINGLE) {
          s_val[wid][0][q * jn + j] = cs * __ldg(a.v[a.single_t] + idx);
        } else {
          const double v0 = __ldg(a.v[0] + idx), v1 = __ldg(a.v[1] + idx), v2 = __ldg(a.v[2] + idx);
          const double v3 = __ldg(a.v[3] + idx), v4 = __ldg(a.v[4] + idx), v5 = __ldg(a.v[5] + idx);
          s_val[wid][0][q * jn + j] = fma(lam, v5, fma(rho, v3, v0));   // A0 + rho Jrho + lam Jlam
          s_val[wid][1][q * jn + j] = v1 + v4;                          // A1 + Jmu
          s_val[wid][2][q * jn + j] = rho * v2;                         // rho A2
        }
      }
      __syncwarp();
      for (int j = 0; j < jn; ++j) {
        const int col = s_col[wid][j];
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
            if constexpr (MODE == SPMM_S2STEP || MODE == SPMM_PLAIN3) {
              const double va = s_val[wid][0][q * jn + j];
              const double vb = s_val[wid][1][q * jn + j];
              const double vc = s_val[wid][2][q * jn + j];
#pragma unroll
              for (int i = 0; i < NC; ++i) {
                acc[q][0][i] = fma(va, u[i], acc[q][0][i]);
                acc[q][1][i] = fma(vb, u[i], acc[q][1][i]);
                acc[q][2][i] = fma(vc, u[i], acc[q][2][i]);
              }
            } else if constexpr (MODE == SPMM_DENSE) {
              const double va = s_val[wid][0][q * jn + j];
              const double vb = s_val[wid][1][q * jn + j];
              const double vc = s_val[wid][2][q * jn + j];
#pragma unroll
              for (int i = 0; i < NC; ++i) {
                const double coef = fma(dnu_c[i], vc, fma(dmu_c[i], vb, va));
                acc[q][0][i] = fma(coef, u[i], acc[q][0][i]);
              }
            } else {
              const double va = s_val[wid][0][q * jn + j];
#pragma unroll
              for (int i = 0; i < NC; ++i) acc[q][0][i] = fma(va, u[i], acc[q][0][i]);
            }
          }
        }
      }
    }
    // epilogue
#pragma unroll
    for (int q = 0; q < GM; ++q) {
      if (q < g) {
        const size_t row = (size_t)(sb + q);
        double* orow = a.out + row * a.ldo + a.out_off;
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          const int c = lane + 32 * i;
          if (c < r) {
            if constexpr (MODE == SPMM_S2STEP) {
              const double uk = __ldg(a.U + row * a.ldu + c);
              orow[c] = fma(-a.gamma, acc[q][0][i], uk);
              orow[r + c] = acc[q][1][i];
              orow[2 * r + c] = acc[q][2][i];
            } else if constexpr (MODE == SPMM_PLAIN3) {
              orow[c] = acc[q][0][i];
              orow[r + c] = acc[q][1][i];
              orow[2 * r + c] = acc[q][2][i];
            } else {
              orow[c] = acc[q][0][i];
            }
          }
        }
      }
    }
  }
}

template <int MODE, int NC, int GM>
cudaError_t launch_t(const SpmmArgs& a, cudaStream_t s) {
  const int blocks = (a.ngroups + kWarps - 1) / kWarps;
  if (blocks == 0) return cudaSuccess;
  constexpr int NV = (MODE == SPMM_SINGLE) ? 1 : 3;
  constexpr size_t smem = (size_t)kWarps * kStage * (NV * sizeof(double) + sizeof(int));
  spmm_kernel<MODE, NC, GM><<<blocks, kWarps * 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_m(const SpmmArgs& a, int rmax, cudaStream_t s) {
  if (rmax <= 32) return launch_t<MODE, 1, 8>(a, s);
  if (rmax <= 64) return launch_t<MODE, 2, 8>(a, s);
  if (rmax <= 128) return launch_t<MODE, 4, 4>(a, s);
  return cudaErrorInvalidValue;
}

template <int MODE, int NC, int GM>
cudaError_t prep_t() {
  constexpr int NV = (MODE == SPMM_SINGLE) ? 1 : 3;
  constexpr size_t smem = (size_t)kWarps * kStage * (NV * sizeof(double) + sizeof(int));
  return cudaFuncSetAttribute(spmm_kernel<MODE, NC, GM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem);
}

template <int MODE>
cudaError_t prep_m() {
  cudaError_t e;
  if ((e = prep_t<MODE, 1, 8>()) != cudaSuccess) return e;
  if ((e = prep_t<MODE, 2, 8>()) != cudaSuccess) return e;
  return prep_t<MODE, 4, 4>();
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
      if (rmax <= 64) return launch_m<SPMM_DENSE>(a, rmax, s);
      if (rmax <= 256) return launch_t<SPMM_DENSE, 8, 4>(a, s);
      return cudaErrorInvalidValue;
  }
  return cudaErrorInvalidValue;
}

}  // namespace lrc
