// a3 / a4 / a6 -- tall-skinny fp64 DMMA kernels of the truncation (
// truncation operator T of PAPER.md P:544).
//
// All three M-level passes of the truncation have the same shape: a row tile of the logical
// concatenation Ucat = [A | B] (M x w, two strided blocks, widths read from device-resident ranks)
// is multiplied by a small w x p matrix T held in L2, on the fp64 tensor pipe
// (mma.sync.m8n8k4.f64, "DMMA"), and the p-wide tile X = Ucat_tile T is then either
//   GRAM  : contracted with itself, G += X^T X (upper 8x8 tiles in 2x2 register blocks, DMMA),
//           accumulated in registers across the CTA's tiles and written once as a per-CTA partial
//           (deterministic fixed-order reduction in gram_reduce_kernel), or
//   STORE : written out (U_{k+1} = Ucat Z, row-major).
// Gram pass 1 uses T = R_V^T, pass 2 T = R_V^T R1^{-1}, the basis GEMM T = Z.
//
// Tile: 128 rows x p, 16 warps, warp w owns rows [8w, 8w+8) (one 8-row DMMA tile) and all p
// columns.  The K loop streams 32-column chunks of Ucat and 32-row chunks of T into a cp.async
// double buffer (8-byte copies: the two Ucat blocks meet at an odd column; zero fill past M / w).
// The X tile is parked in the (then idle) stage buffers for the Gram / store epilogue.
#include "lrc_internal.cuh"

namespace lrc {

namespace {

constexpr int kThreads = 512;   // 16 warps
constexpr int kWarps = kThreads / 32;
constexpr int kBM = 128;        // rows per tile
constexpr int kBK = 32;         // k chunk
constexpr int kSU = kBK + 4;    // smem row stride of the U chunk (== 4 mod 16 doubles: conflict free)

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// column offsets of the Ucat blocks (off[nb] = w)
__device__ __forceinline__ int ucat_offsets(const TsArgs& a, int (&off)[kMaxUBlocks + 1]) {
  int o = 0;
#pragma unroll
  for (int bi = 0; bi < kMaxUBlocks; ++bi) {
    off[bi] = o;
    if (bi < a.u.nb) {
      const int wd = a.u.b[bi].w_fixed + (a.u.b[bi].w_idx >= 0 ? a.rk[a.u.b[bi].w_idx] : 0);
      o += a.u.pad_even ? wd + (wd & 1) : wd;
    }
  }
  off[kMaxUBlocks] = o;
  return o;
}

template <int PT>
struct TsShape {
  static constexpr int PMAX = PT * 8;
  static constexpr int SX = PMAX + 4;                    // T chunk / X tile row stride
  static constexpr int STAGE = kBM * kSU + kBK * SX;     // doubles per pipeline stage
  static constexpr int SMEM = (2 * STAGE > kBM * SX ? 2 * STAGE : kBM * SX);
  static constexpr int PT2 = (PT + 1) / 2;               // 2x2 super tiles of the Gram
  static constexpr int NS = PT2 * (PT2 + 1) / 2;
  static constexpr int SPW = (NS + kWarps - 1) / kWarps;  // super tiles per warp
};

template <int PT>
__device__ __forceinline__ void issue_chunk(const TsArgs& a, double* stage, int m0, int k0, int w,
                                            const int (&off)[kMaxUBlocks + 1], int tid) {
  using S = TsShape<PT>;
  double* s_u = stage;
  double* s_t = stage + kBM * kSU;
  if (a.u16) {
    // 16-byte copies: every block starts at an even logical column with an even ld
#pragma unroll 4
    for (int e = tid; e < kBM * kBK / 2; e += kThreads) {
      const int i = e >> 4, j = (e & 15) * 2;
      const int m = m0 + i, c = k0 + j;
      const bool ok = (m < a.M) && (c < w);
      const double* src = a.u.b[0].p;
      if (ok) {
        int bi = 0;
#pragma unroll
        for (int q = 1; q < kMaxUBlocks; ++q) bi += (c >= off[q]);
        src = a.u.b[bi].p + (size_t)m * a.u.b[bi].ld + (c - off[bi]);
      }
      const unsigned sa = (unsigned)__cvta_generic_to_shared(s_u + i * kSU + j);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(ok ? 16 : 0));
    }
  } else {
#pragma unroll 4
    for (int e = tid; e < kBM * kBK; e += kThreads) {
      const int i = e >> 5, j = e & 31;
      const int m = m0 + i, c = k0 + j;
      const bool ok = (m < a.M) && (c < w);
      const double* src = a.u.b[0].p;
      if (ok) {
        int bi = 0;
#pragma unroll
        for (int q = 1; q < kMaxUBlocks; ++q) bi += (c >= off[q]);
        src = a.u.b[bi].p + (size_t)m * a.u.b[bi].ld + (c - off[bi]);
      }
      cp_async8(s_u + i * kSU + j, src, ok);
    }
  }
  // T rows are 16-byte aligned (ldt even): two doubles per copy
  constexpr int HP = S::PMAX / 2;
#pragma unroll 4
  for (int e = tid; e < kBK * HP; e += kThreads) {
    const int i = e / HP, j2 = e - (e / HP) * HP;
    const int c = k0 + i;
    const bool ok = c < w;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s_t + i * S::SX + 2 * j2);
    const double* g = ok ? a.T + (size_t)c * a.ldt + 2 * j2 : a.T;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 16 : 0));
  }
}

template <int PT, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
ts_kernel(TsArgs a) {
  using S = TsShape<PT>;
  constexpr int PMAX = S::PMAX, SX = S::SX;

  int off[kMaxUBlocks + 1];
  const int w = ucat_offsets(a, off);
  const int p = a.d_p ? *a.d_p : a.p_fixed;
  if (w <= 0 || p <= 0) {
    if (MODE == 0) {   // still publish a zero partial so the reduction is well defined
      double* part = a.partials + (size_t)blockIdx.x * PMAX * PMAX;
      for (int e = threadIdx.x; e < PMAX * PMAX; e += kThreads) part[e] = 0.0;
    }
    return;
  }

  extern __shared__ double sm[];
  double* s_x = sm;                                      // aliases the two stages after the K loop

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;

  // Gram super tiles (I2, J2), I2 <= J2, of this warp
  double gacc[S::SPW][4][2];
  int sI[S::SPW], sJ[S::SPW];
#pragma unroll
  for (int s = 0; s < S::SPW; ++s) {
#pragma unroll
    for (int q = 0; q < 4; ++q) gacc[s][q][0] = gacc[s][q][1] = 0.0;
    int t = warp + kWarps * s, I = 0;
    if (t >= S::NS) { sI[s] = -1; sJ[s] = -1; continue; }
    while (t >= S::PT2 - I) { t -= S::PT2 - I; ++I; }
    sI[s] = I; sJ[s] = I + t;
  }

  const int nk = (w + kBK - 1) / kBK;
  const int ntiles = (a.M + kBM - 1) / kBM;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int m0 = tile * kBM;
    double x0[PT][2];
#pragma unroll
    for (int n = 0; n < PT; ++n) x0[n][0] = x0[n][1] = 0.0;

    issue_chunk<PT>(a, sm, m0, 0, w, off, tid);
    cp_commit();
    for (int kc = 0; kc < nk; ++kc) {
      if (kc + 1 < nk) {
        issue_chunk<PT>(a, sm + ((kc + 1) & 1) * S::STAGE, m0, (kc + 1) * kBK, w, off, tid);
        cp_commit();
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
      const double* s_u = sm + (kc & 1) * S::STAGE;
      const double* s_t = s_u + kBM * kSU;
      const int k0 = kc * kBK;
#pragma unroll
      for (int kk = 0; kk < kBK; kk += 4) {
        const double a0 = s_u[(warp * 8 + gid) * kSU + kk + tig];
#pragma unroll
        for (int n = 0; n < PT; ++n) {
          // T1 = R_V^T is lower trapezoidal: blocks with all i > c are zero (warp-uniform skip)
          if (a.t_lower && n * 8 > k0 + kk + 3) continue;
          const double bv = s_t[(kk + tig) * SX + n * 8 + gid];
          dmma884(x0[n], a0, bv);
        }
      }
      __syncthreads();
    }
    // X tile -> smem (stage buffers are idle now)
#pragma unroll
    for (int n = 0; n < PT; ++n) {
      const int c = n * 8 + 2 * tig;
      *reinterpret_cast<double2*>(s_x + (warp * 8 + gid) * SX + c) = make_double2(x0[n][0], x0[n][1]);
    }
    __syncthreads();
    if constexpr (MODE == 0) {
#pragma unroll 2
      for (int k = 0; k < kBM; k += 4) {
        const double* xr = s_x + (k + tig) * SX + gid;
#pragma unroll
        for (int s = 0; s < S::SPW; ++s) {
          if (sI[s] >= 0) {
            const int I0 = 2 * sI[s], J0 = 2 * sJ[s];
            const double a0 = xr[I0 * 8];
            const double a1 = (I0 + 1 < PT) ? xr[(I0 + 1) * 8] : 0.0;
            const double b0 = xr[J0 * 8];
            const double b1 = (J0 + 1 < PT) ? xr[(J0 + 1) * 8] : 0.0;
            dmma884(gacc[s][0], a0, b0);
            dmma884(gacc[s][1], a0, b1);
            if (sI[s] != sJ[s]) dmma884(gacc[s][2], a1, b0);
            dmma884(gacc[s][3], a1, b1);
          }
        }
      }
    } else {
      for (int e = tid; e < kBM * PMAX; e += kThreads) {
        const int i = e / PMAX, j = e - (e / PMAX) * PMAX;
        const int m = m0 + i;
        // padded (solver) mode also writes the zero pad column of an odd-width U block
        if (m < a.M && j < p + (a.u.pad_even ? (p & 1) : 0)) a.out[(size_t)m * a.ldo + j] = s_x[i * SX + j];
      }
    }
    __syncthreads();   // s_x (= stage memory) is overwritten by the next tile's first chunk
  }

  if constexpr (MODE == 0) {
    double* part = a.partials + (size_t)blockIdx.x * PMAX * PMAX;
    // lower 8x8 tiles are never computed: zero them so the reduction reads defined data
    for (int e = tid; e < PMAX * PMAX; e += kThreads) {
      const int i = e / PMAX, j = e - (e / PMAX) * PMAX;
      if ((i >> 3) > (j >> 3)) part[e] = 0.0;
    }
#pragma unroll
    for (int s = 0; s < S::SPW; ++s) {
      if (sI[s] >= 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int I = 2 * sI[s] + (q >> 1), J = 2 * sJ[s] + (q & 1);
          if (I < PT && J < PT && I <= J) {
            const int row = I * 8 + gid, col = J * 8 + 2 * tig;
            part[row * PMAX + col] = gacc[s][q][0];
            part[row * PMAX + col + 1] = gacc[s][q][1];
          }
        }
      }
    }
  }
}

template <int PT, int MODE>
cudaError_t launch_pt(const TsArgs& a, int grid, cudaStream_t s) {
  ts_kernel<PT, MODE><<<grid, kThreads, sizeof(double) * TsShape<PT>::SMEM, s>>>(a);
  return cudaGetLastError();
}

template <int PT, int MODE>
cudaError_t prep_pt() {
  return cudaFuncSetAttribute(ts_kernel<PT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(sizeof(double) * TsShape<PT>::SMEM));
}

template <int MODE, int PT>
struct Dispatch {
  static cudaError_t launch(const TsArgs& a, int pt, int grid, cudaStream_t s) {
    if (pt == PT) return launch_pt<PT, MODE>(a, grid, s);
    return Dispatch<MODE, PT - 1>::launch(a, pt, grid, s);
  }
  static cudaError_t prep() {
    cudaError_t e = prep_pt<PT, MODE>();
    return e != cudaSuccess ? e : Dispatch<MODE, PT - 1>::prep();
  }
};
template <int MODE>
struct Dispatch<MODE, 0> {
  static cudaError_t launch(const TsArgs&, int, int, cudaStream_t) { return cudaErrorInvalidValue; }
  static cudaError_t prep() { return cudaSuccess; }
};

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
  cudaError_t e = Dispatch<0, 16>::prep();
  return e != cudaSuccess ? e : Dispatch<1, 16>::prep();
}

int ts_pmax_for(int p) {
  if (p < 1 || p > 128) return -1;
  return 8 * ((p + 7) / 8);
}

int ts_grid_for(int M, int reserved) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int ntiles = (M + kBM - 1) / kBM;
  int g = sms - (reserved > 0 ? reserved : 0);
  if (g < 1) g = 1;
  return ntiles < g ? (ntiles > 0 ? ntiles : 1) : g;
}

cudaError_t launch_ts(int mode, const TsArgs& a0, int pmax, int grid, cudaStream_t s) {
  if (pmax % 8 || pmax < 8 || pmax > 128) return cudaErrorInvalidValue;
  TsArgs a = a0;
  bool u16 = a.u.pad_even != 0;
  for (int bi = 0; bi < a.u.nb; ++bi)
    u16 = u16 && (a.u.b[bi].ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.u.b[bi].p) & 15) == 0);
  a.u16 = u16 ? 1 : 0;
  return mode == 0 ? Dispatch<0, 16>::launch(a, pmax / 8, grid, s)
                   : Dispatch<1, 16>::launch(a, pmax / 8, grid, s);
}

cudaError_t launch_gram_reduce(const double* partials, int nblocks, int pmax, double* G,
                               cudaStream_t s) {
  const int n2 = pmax * pmax;
  gram_reduce_kernel<<<(n2 + 255) / 256, 256, 0, s>>>(partials, nblocks, pmax, G);
  return cudaGetLastError();
}

}  // namespace lrc
