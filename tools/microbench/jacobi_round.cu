// Micro-benchmark: SM cycles per round-robin round of the single-CTA one-sided Jacobi used in the
// core SVD (small.cu), on a random p x p matrix, with parts of the round switched off.
// MODE 0: full round; 1: dots + reductions only (no rotation); 2: barrier + pair indexing only.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE, int LPP>
__global__ void __launch_bounds__(1024) jac(double* A_g, int p, int rounds, long long* cyc) {
  extern __shared__ double sm[];
  const int LD = 105;
  double* s_a = sm;
  double* s_w = sm + 104 * LD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < p * p; e += 1024) {
    s_a[(e / p) * LD + e % p] = A_g[e];
    s_w[(e / p) * LD + e % p] = (e / p == e % p) ? 1.0 : 0.0;
  }
  __syncthreads();
  constexpr int PPW = 32 / LPP;   // pairs per warp
  const int sub = lane / LPP, sl = lane % LPP;
  const int P = p + (p & 1), NP = P / 2;
  long long t0 = clock64();
  for (int rr = 0; rr < rounds; ++rr) {
    const int r = rr % (P - 1);
    for (int qb = warp * PPW; qb < NP; qb += 32 * PPW) {
      const int q = qb + sub;
      int i = 0, j = 0;
      bool act = q < NP;
      if (act) {
        if (q == 0) { i = P - 1; j = r; } else { i = (r + q) % (P - 1); j = (r - q + P - 1) % (P - 1); }
        act = (i < p) && (j < p);
        if (i > j) { const int t = i; i = j; j = t; }
      }
      if (MODE == 2) continue;
      double* ai = s_a + i * LD;
      double* aj = s_a + j * LD;
      double al = 0.0, be = 0.0, ga = 0.0;
      if (act)
        for (int e = sl; e < p; e += LPP) {
          const double x = ai[e], y = aj[e];
          al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
        }
#pragma unroll
      for (int o = LPP / 2; o > 0; o >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, o);
        be += __shfl_xor_sync(0xffffffffu, be, o);
        ga += __shfl_xor_sync(0xffffffffu, ga, o);
      }
      if (MODE == 0 && act && ga != 0.0 && ga * ga > 1e-28 * al * be) {
        const double dd = be - al;
        const double t = ((dd >= 0.0) ? 2.0 * ga : -2.0 * ga) / (fabs(dd) + sqrt(fma(dd, dd, 4.0 * ga * ga)));
        const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
        for (int e = sl; e < p; e += LPP) {
          const double x = ai[e], y = aj[e];
          ai[e] = c * x - sn * y;
          aj[e] = sn * x + c * y;
        }
        double* wi = s_w + i * LD;
        double* wj = s_w + j * LD;
        for (int e = sl; e < p; e += LPP) {
          const double x = wi[e], y = wj[e];
          wi[e] = c * x - sn * y;
          wj[e] = sn * x + c * y;
        }
      }
      if (MODE == 1 && act && sl == 0) s_w[0] += ga * 1e-300;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) *cyc = t1 - t0;
  for (int e = tid; e < p * p; e += 1024) A_g[e] = s_a[(e / p) * LD + e % p];
}

int main() {
  const int p = 100, rounds = 990;
  double* h = new double[p * p];
  unsigned s = 1;
  for (int i = 0; i < p * p; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
  double* d; long long* cyc;
  cudaMalloc(&d, p * p * 8);
  cudaMalloc(&cyc, 8);
  const int smem = 2 * 104 * 105 * 8;
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemcpy(d, h, p * p * 8, cudaMemcpyHostToDevice);
      kern<<<1, 1024, smem>>>(d, p, rounds, cyc);
      cudaDeviceSynchronize();
    }
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"variant\": \"%s\", \"cycles_per_round\": %.0f, \"err\": \"%s\"}\n", name, (double)c / rounds,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(jac<0, 16>, "full, 16 lanes/pair");
  run(jac<1, 16>, "dots+reduce only, 16 lanes/pair");
  run(jac<2, 16>, "barrier+indexing only");
  run(jac<0, 32>, "full, 32 lanes/pair");
  run(jac<0, 8>, "full, 8 lanes/pair");
  run(jac<0, 4>, "full, 4 lanes/pair");
  return 0;
}
