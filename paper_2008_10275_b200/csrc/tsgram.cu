// a3 / a4 / a6 -- tall-skinny fp64 DMMA kernels of the truncation (
// truncation operator T of PAPER.md P:544).
//
// All three M-level passes of the truncation have the same shape: a row tile of the logical
// concatenation Ucat = [A | B] (M x w, two strided blocks, widths read from device-resident ranks)
// is multiplied by a small w x p matrix T held in L2, on the fp64 tensor pipe
// (mma.sync.m8n8k4.f64, "DMMA"), and the p-wide tile is then either
//   GRAM  : contracted with itself, G += X_tile^T X_tile (upper 8x8 tiles, DMMA), accumulated in
//           registers across the CTA's tiles and written once as a per-CTA partial
//           (deterministic fixed-order reduction in gram_reduce_kernel), or
//   STORE : written out (U_{k+1} = Ucat Z, row-major).
// Gram pass 1 uses T = R_V^T, pass 2 T = R_V^T R1^{-1}, the basis GEMM T = Z.
#include "lrc_internal.cuh"

namespace lrc {

namespace {

constexpr int kThreads = 256;   // 8 warps
constexpr int kBM = 64;         // rows per tile
constexpr int kBK = 32;         // k chunk
constexpr int kSU = kBK + 4;    // smem row stride of the U tile (== 4 mod 16 doubles: conflict free)

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int ucat_widths(const TsArgs& a, int& wa) {
  wa = a.u.wa_fixed + (a.u.wa_idx >= 0 ? a.u.wa_mul * a.rk[a.u.wa_idx] : 0);
  const int wb = a.u.B ? (a.u.wb_idx >= 0 ? a.rk[a.u.wb_idx] : a.u.wb_fixed) : 0;
  return wa + wb;
}

template <int PT, int MODE>
__global__ void __launch_bounds__(kThreads)
ts_kernel(TsArgs a) {
  constexpr int PMAX = PT * 8;
  constexpr int SX = PMAX + 4;                      // row stride of T chunk / X tile in smem
  constexpr int NT = PT * (PT + 1) / 2;             // upper 8x8 tiles of the Gram
  constexpr int TPW = (NT + 7) / 8;                 // Gram tiles per warp

  int wa;
  const int w = ucat_widths(a, wa);
  const int p = a.d_p ? *a.d_p : a.p_fixed;
  if (w <= 0 || p <= 0) {
    if (MODE == 0) {   // still publish a zero partial so the reduction is well defined
      double* part = a.partials + (size_t)blockIdx.x * PMAX * PMAX;
      for (int e = threadIdx.x; e < PMAX * PMAX; e += kThreads) part[e] = 0.0;
    }
    return;
  }

  extern __shared__ double sm[];
  double* s_u = sm;                        // [kBM][kSU]
  double* s_t = s_u + kBM * kSU;           // [kBK][SX]
  double* s_x = s_t + kBK * SX;            // [kBM][SX]

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;

  double gacc[TPW][2];
#pragma unroll
  for (int s = 0; s < TPW; ++s) gacc[s][0] = gacc[s][1] = 0.0;
  // Gram tile coordinates of this warp
  int tI[TPW], tJ[TPW];
#pragma unroll
  for (int s = 0; s < TPW; ++s) {
    int t = warp + 8 * s, I = 0;
    if (t >= NT) { tI[s] = -1; tJ[s] = -1; continue; }
    while (t >= PT - I) { t -= PT - I; ++I; }
    tI[s] = I; tJ[s] = I + t;
  }

  const int ntiles = (a.M + kBM - 1) / kBM;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int m0 = tile * kBM;
    double xacc[PT][2];
#pragma unroll
    for (int n = 0; n < PT; ++n) xacc[n][0] = xacc[n][1] = 0.0;

    for (int k0 = 0; k0 < w; k0 += kBK) {
      // stage the Ucat tile [m0, m0+64) x [k0, k0+32)
      for (int e = tid; e < kBM * kBK; e += kThreads) {
        const int i = e / kBK, j = e - (e / kBK) * kBK;
        const int m = m0 + i, c = k0 + j;
        double v = 0.0;
        if (m < a.M && c < w) {
          v = (c < wa) ? __ldg(a.u.A + (size_t)m * a.u.lda + c)
                       : __ldg(a.u.B + (size_t)m * a.u.ldb + (c - wa));
        }
        s_u[i * kSU + j] = v;
      }
      // stage the T chunk [k0, k0+32) x [0, PMAX)
      for (int e = tid; e < kBK * PMAX; e += kThreads) {
        const int i = e / PMAX, j = e - (e / PMAX) * PMAX;
        const int c = k0 + i;
        s_t[i * SX + j] = (c < w && j < p) ? __ldg(a.T + (size_t)c * a.ldt + j) : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kBK; kk += 4) {
        const double av = s_u[(warp * 8 + gid) * kSU + kk + tig];
#pragma unroll
        for (int n = 0; n < PT; ++n) {
          const double bv = s_t[(kk + tig) * SX + n * 8 + gid];
          dmma884(xacc[n], av, bv);
        }
      }
      __syncthreads();
    }
    // X tile -> smem
#pragma unroll
    for (int n = 0; n < PT; ++n) {
      s_x[(warp * 8 + gid) * SX + n * 8 + 2 * tig] = xacc[n][0];
      s_x[(warp * 8 + gid) * SX + n * 8 + 2 * tig + 1] = xacc[n][1];
    }
    __syncthreads();
    if constexpr (MODE == 0) {
#pragma unroll 4
      for (int k = 0; k < kBM; k += 4) {
#pragma unroll
        for (int s = 0; s < TPW; ++s) {
          if (tI[s] >= 0) {
            const double av = s_x[(k + tig) * SX + tI[s] * 8 + gid];
            const double bv = s_x[(k + tig) * SX + tJ[s] * 8 + gid];
            dmma884(gacc[s], av, bv);
          }
        }
      }
    } else {
      for (int e = tid; e < kBM * PMAX; e += kThreads) {
        const int i = e / PMAX, j = e - (e / PMAX) * PMAX;
        const int m = m0 + i;
        if (m < a.M && j < p) a.out[(size_t)m * a.ldo + j] = s_x[i * SX + j];
      }
    }
    // the next tile's first k-chunk __syncthreads() orders these s_x reads before its writes
  }

  if constexpr (MODE == 0) {
    double* part = a.partials + (size_t)blockIdx.x * PMAX * PMAX;
    // zero the lower 8x8 tiles (never computed) so the reduction reads defined data
    for (int e = tid; e < PMAX * PMAX; e += kThreads) {
      const int i = e / PMAX, j = e - (e / PMAX) * PMAX;
      if ((i >> 3) > (j >> 3)) part[e] = 0.0;
    }
#pragma unroll
    for (int s = 0; s < TPW; ++s) {
      if (tI[s] >= 0) {
        const int row = tI[s] * 8 + gid, col = tJ[s] * 8 + 2 * tig;
        part[row * PMAX + col] = gacc[s][0];
        part[row * PMAX + col + 1] = gacc[s][1];
      }
    }
  }
}

template <int PT, int MODE>
cudaError_t launch_pt(const TsArgs& a, int grid, cudaStream_t s) {
  constexpr int PMAX = PT * 8;
  constexpr size_t smem = sizeof(double) * ((size_t)kBM * kSU + (size_t)kBK * (PMAX + 4) +
                                            (size_t)kBM * (PMAX + 4));
  ts_kernel<PT, MODE><<<grid, kThreads, smem, s>>>(a);
  return cudaGetLastError();
}

template <int PT, int MODE>
cudaError_t prep_pt() {
  constexpr int PMAX = PT * 8;
  constexpr size_t smem = sizeof(double) * ((size_t)kBM * kSU + (size_t)kBK * (PMAX + 4) +
                                            (size_t)kBM * (PMAX + 4));
  return cudaFuncSetAttribute(ts_kernel<PT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem);
}

template <int MODE>
cudaError_t prep_mode() {
  cudaError_t e;
  if ((e = prep_pt<2, MODE>()) != cudaSuccess) return e;
  if ((e = prep_pt<4, MODE>()) != cudaSuccess) return e;
  if ((e = prep_pt<6, MODE>()) != cudaSuccess) return e;
  if ((e = prep_pt<8, MODE>()) != cudaSuccess) return e;
  if ((e = prep_pt<10, MODE>()) != cudaSuccess) return e;
  if ((e = prep_pt<12, MODE>()) != cudaSuccess) return e;
  if ((e = prep_pt<14, MODE>()) != cudaSuccess) return e;
  return prep_pt<16, MODE>();
}

template <int MODE>
cudaError_t launch_mode(const TsArgs& a, int pmax, int grid, cudaStream_t s) {
  switch (pmax) {
    case 16: return launch_pt<2, MODE>(a, grid, s);
    case 32: return launch_pt<4, MODE>(a, grid, s);
    case 48: return launch_pt<6, MODE>(a, grid, s);
    case 64: return launch_pt<8, MODE>(a, grid, s);
    case 80: return launch_pt<10, MODE>(a, grid, s);
    case 96: return launch_pt<12, MODE>(a, grid, s);
    case 112: return launch_pt<14, MODE>(a, grid, s);
    case 128: return launch_pt<16, MODE>(a, grid, s);
  }
  return cudaErrorInvalidValue;
}

__global__ void gram_reduce_kernel(const double* __restrict__ partials, int nblocks, int pmax,
                                   double* __restrict__ G) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int n2 = pmax * pmax;
  if (e >= n2) return;
  const int i = e / pmax, j = e - (e / pmax) * pmax;
  if (i > j) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += partials[(size_t)b * n2 + e];   // fixed order
  G[i * pmax + j] = s;
  G[j * pmax + i] = s;
}

}  // namespace

cudaError_t ts_prepare() {
  cudaError_t e = prep_mode<0>();
  return e != cudaSuccess ? e : prep_mode<1>();
}

int ts_pmax_for(int p) {
  if (p <= 16) return 16;
  if (p <= 32) return 32;
  if (p <= 48) return 48;
  if (p <= 64) return 64;
  if (p <= 80) return 80;
  if (p <= 96) return 96;
  if (p <= 112) return 112;
  if (p <= 128) return 128;
  return -1;
}

int ts_grid_for(int M) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int ntiles = (M + kBM - 1) / kBM;
  const int g = 2 * sms;
  return ntiles < g ? (ntiles > 0 ? ntiles : 1) : g;
}

cudaError_t launch_ts(int mode, const TsArgs& a, int pmax, int grid, cudaStream_t s) {
  return mode == 0 ? launch_mode<0>(a, pmax, grid, s) : launch_mode<1>(a, pmax, grid, s);
}

cudaError_t launch_gram_reduce(const double* partials, int nblocks, int pmax, double* G,
                               cudaStream_t s) {
  const int n2 = pmax * pmax;
  gram_reduce_kernel<<<(n2 + 255) / 256, 256, 0, s>>>(partials, nblocks, pmax, G);
  return cudaGetLastError();
}

}  // namespace lrc
