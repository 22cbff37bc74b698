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

__device__ __forceinline__ void dmma1684(double (&d)[4], double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b));
}

// m16n8k4: each warp owns 16 rows; PRED: every other DMMA carries a runtime-false predicate
template <int PT>
__global__ void loop16_kernel(double* out, int iters) {
  constexpr int SX = PT * 8 + 4, SU = 36;
  extern __shared__ double smx[];
  double* s_u = smx;
  double* s_t = smx + 256 * SU;
  for (int i = threadIdx.x; i < 256 * SU; i += blockDim.x) s_u[i] = 1e-3 * (i % 7);
  for (int i = threadIdx.x; i < 32 * SX; i += blockDim.x) s_t[i] = 1e-3 * (i % 5);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  double x[PT][4];
#pragma unroll
  for (int n = 0; n < PT; ++n) x[n][0] = x[n][1] = x[n][2] = x[n][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      const double a0 = s_u[((warp * 16) % 256 + gid) * SU + kk + tig];
      const double a1 = s_u[((warp * 16) % 256 + gid + 8) * SU + kk + tig];
#pragma unroll
      for (int n = 0; n < PT; ++n) dmma1684(x[n], a0, a1, s_t[(kk + tig) * SX + n * 8 + gid]);
    }
  }
  double s = 0;
#pragma unroll
  for (int n = 0; n < PT; ++n) s += x[n][0] + x[n][1] + x[n][2] + x[n][3];
  if (s == 1234.5) out[0] = s;
}

// PT m8n8k4 steps of which only the first NACT are meant: the rest are issued under a runtime-false
// predicate (does a predicated-off DMMA cost pipe time?)
template <int PT, int NACT>
__global__ void pred_kernel(double* out, int iters, int lim) {
  constexpr int SX = PT * 8 + 4, SU = 36;
  extern __shared__ double smx[];
  double* s_u = smx;
  double* s_t = smx + 128 * SU;
  for (int i = threadIdx.x; i < 128 * SU; i += blockDim.x) s_u[i] = 1e-3 * (i % 7);
  for (int i = threadIdx.x; i < 32 * SX; i += blockDim.x) s_t[i] = 1e-3 * (i % 5);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  double x[PT][2];
#pragma unroll
  for (int n = 0; n < PT; ++n) x[n][0] = x[n][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      const double a = s_u[(warp * 8 % 128 + gid) * SU + kk + tig];
#pragma unroll
      for (int n = 0; n < PT; ++n) {
        if (n >= NACT && n * 8 > lim + kk) continue;   // lim is large: never true at run time
        dmma884(x[n], a, s_t[(kk + tig) * SX + n * 8 + gid]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int n = 0; n < PT; ++n) s += x[n][0] + x[n][1];
  if (s == 1234.5) out[0] = s;
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

template <int PT>
void run16(const char* name, int threads) {
  double* out; cudaMalloc(&out, 8);
  const int iters = 2000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int smem = (256 * 36 + 32 * (PT * 8 + 4)) * 8;
  cudaFuncSetAttribute(loop16_kernel<PT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  loop16_kernel<PT><<<148, threads, smem>>>(out, 10);
  cudaEventRecord(e0);
  loop16_kernel<PT><<<148, threads, smem>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 148.0 * (threads / 32) * PT * 8.0 * iters * 1024.0;
  printf("{\"variant\": \"%s\", \"tflops\": %.2f, \"err\": \"%s\"}\n", name, flops / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

template <int PT, int NACT>
void runpred(const char* name, int lim) {
  double* out; cudaMalloc(&out, 8);
  const int iters = 2000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int smem = (128 * 36 + 32 * (PT * 8 + 4)) * 8;
  cudaFuncSetAttribute(pred_kernel<PT, NACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  pred_kernel<PT, NACT><<<148, 512, smem>>>(out, 10, lim);
  cudaEventRecord(e0);
  pred_kernel<PT, NACT><<<148, 512, smem>>>(out, iters, lim);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"variant\": \"%s\", \"ms\": %.3f, \"err\": \"%s\"}\n", name, ms,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run16<13>("m16n8k4: 8 warps x 16 rows, PT 13", 256);
  run16<13>("m16n8k4: 16 warps x 16 rows, PT 13", 512);
  run16<8>("m16n8k4: 8 warps x 16 rows, PT 8", 256);
  runpred<13, 13>("13 DMMA per step, all active (lim large)", 1 << 20);
  runpred<13, 6>("13 DMMA per step, 7 under a predicate that is true (all issued)", 1 << 20);
  runpred<13, 6>("13 DMMA per step, 7 predicated off (lim = -1000)", -1000);
  run<1, 13>("16 warps, 1 m-tile, PT 13 (ts_kernel GRAM phase A)", 512);
  run<2, 13>("8 warps, 2 m-tiles, PT 13", 256);
  run<2, 13>("16 warps, 2 m-tiles, PT 13", 512);
  run<1, 8>("16 warps, 1 m-tile, PT 8 (ts_kernel STORE)", 512);
  run<2, 8>("16 warps, 2 m-tiles, PT 8", 512);
  return 0;
}
