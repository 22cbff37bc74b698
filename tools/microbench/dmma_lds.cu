// Micro-benchmark: the ts_kernel inner loop (shared-memory fed fp64 DMMA) in isolation, no global
// traffic and no barriers.  Variant V: warps x (m-tiles per warp) x (n-tiles PT).
//   V0: 16 warps, 1 m-tile, PT 13 (current ts_kernel)      V1: 8 warps, 2 m-tiles, PT 13
//   V2: 16 warps, 2 m-tiles, PT 13                          V3: 16 warps, 1 m-tile, PT 8 (store)
// Reports fp64 TFLOP/s over all 148 SMs (1 CTA / SM).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int MT, int PT>
__global__ void loop_kernel(double* out, int iters) {
  constexpr int SX = PT * 8 + 4, SU = 36;
  extern __shared__ double smx[];
  double* s_u = smx;                  // [128][SU]
  double* s_t = smx + 128 * SU;       // [32][SX]
  for (int i = threadIdx.x; i < 128 * SU; i += blockDim.x) s_u[i] = 1e-3 * (i % 7);
  for (int i = threadIdx.x; i < 32 * SX; i += blockDim.x) s_t[i] = 1e-3 * (i % 5);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  double x[MT][PT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < PT; ++n) x[m][n][0] = x[m][n][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      double a[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) a[m] = s_u[((warp * MT + m) * 8 % 128 + gid) * SU + kk + tig];
#pragma unroll
      for (int n = 0; n < PT; ++n) {
        const double b = s_t[(kk + tig) * SX + n * 8 + gid];
#pragma unroll
        for (int m = 0; m < MT; ++m) dmma884(x[m][n], a[m], b);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < PT; ++n) s += x[m][n][0] + x[m][n][1];
  if (s == 1234.5) out[0] = s;
}

template <int MT, int PT>
void run(const char* name, int threads) {
  double* out; cudaMalloc(&out, 8);
  const int iters = 2000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int smem = (128 * 36 + 32 * (PT * 8 + 4)) * 8;
  cudaFuncSetAttribute(loop_kernel<MT, PT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  loop_kernel<MT, PT><<<148, threads, smem>>>(out, 10);
  cudaEventRecord(e0);
  loop_kernel<MT, PT><<<148, threads, smem>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 148.0 * (threads / 32) * MT * PT * 8.0 * iters * 512.0;
  printf("{\"variant\": \"%s\", \"tflops\": %.2f, \"err\": \"%s\"}\n", name, flops / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<1, 13>("16 warps, 1 m-tile, PT 13 (ts_kernel GRAM phase A)", 512);
  run<2, 13>("8 warps, 2 m-tiles, PT 13", 256);
  run<2, 13>("16 warps, 2 m-tiles, PT 13", 512);
  run<1, 8>("16 warps, 1 m-tile, PT 8 (ts_kernel STORE)", 512);
  run<2, 8>("16 warps, 2 m-tiles, PT 8", 512);
  return 0;
}
