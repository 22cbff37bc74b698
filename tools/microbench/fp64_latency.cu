// Phase-0 micro-benchmark: dependent-chain latency (SM cycles per op) of fp64 DFMA, DADD, sqrt,
// division, rsqrt, 64-bit warp shuffle and __syncthreads on sm_100a -- the ops on the critical path
// of the single-CTA Jacobi rounds.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, double x0, long long* cyc, int n) {
  double x = x0 + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) x = fma(x, 0.9999999, 1e-7);
    if (OP == 1) x = x + 1e-7;
    if (OP == 2) x = sqrt(x + 1.0);
    if (OP == 3) x = 1.0 / (x + 1.0);
    if (OP == 4) x = rsqrt(x + 1.0);
    if (OP == 5) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-9;
    if (OP == 6) { __syncthreads(); x += 1e-9; }
    if (OP == 7) x = (float)sqrtf((float)x + 1.0f);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  out[threadIdx.x] = x;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  const char* names[] = {"dfma", "dadd", "dsqrt", "ddiv", "drsqrt", "shfl64+dadd", "syncthreads(1024)+dadd", "fsqrt"};
  const int n = 4096;
  for (int op = 0; op < 8; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      int threads = (op == 6) ? 1024 : 32;
      switch (op) {
        case 0: chain<0><<<1, threads>>>(out, 1.0, cyc, n); break;
        case 1: chain<1><<<1, threads>>>(out, 1.0, cyc, n); break;
        case 2: chain<2><<<1, threads>>>(out, 1.0, cyc, n); break;
        case 3: chain<3><<<1, threads>>>(out, 1.0, cyc, n); break;
        case 4: chain<4><<<1, threads>>>(out, 1.0, cyc, n); break;
        case 5: chain<5><<<1, threads>>>(out, 1.0, cyc, n); break;
        case 6: chain<6><<<1, threads>>>(out, 1.0, cyc, n); break;
        case 7: chain<7><<<1, threads>>>(out, 1.0, cyc, n); break;
      }
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
      if (rep == 1) printf("{\"op\": \"%s\", \"cycles_per_op\": %.1f}\n", names[op], (double)c / n);
    }
  }
  return 0;
}
