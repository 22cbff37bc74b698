// Phase-0 micro-benchmark: fp64 FFMA (DFMA) and DMMA (mma.sync f64) throughput on sm_100a.
// Measures sustained issue rate with independent accumulator chains; prints TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int ITERS>
__global__ void dfma_kernel(double* out, double a, double b) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

template<int ITERS>
__global__ void dmma884_kernel(double* out, double a0, double b0) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template<int ITERS>
__global__ void dmma16816_kernel(double* out, double a0, double b0) {
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = a0 + i * 1e-9 + threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = b0 + i * 1e-9;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

// Mixed: half the warps do DMMA, half DFMA (tests whether the pipes are separate).
template<int ITERS>
__global__ void mixed_kernel(double* out, double a0, double b0) {
  int w = threadIdx.x / 32;
  if (w & 1) {
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS * 2; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a0, b0);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == 12345.678) out[0] = s;
  } else {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
    double a = a0 + threadIdx.x * 1e-9, b = b0;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
  }
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_block_optin\": %zu, \"clock_khz\": %d}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, clk);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int IT = 4096;
  for (int blocksPerSM : {2, 4, 8}) {
    for (int threads : {256, 512}) {
      int grid = p.multiProcessorCount * blocksPerSM;
      float ms;
      // DFMA
      dfma_kernel<IT><<<grid, threads>>>(out, 1.0000001, 1e-7);
      cudaEventRecord(e0); dfma_kernel<IT><<<grid, threads>>>(out, 1.0000001, 1e-7); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 16 * IT * (double)grid * threads;
      printf("{\"kernel\": \"dfma\", \"grid\": %d, \"threads\": %d, \"tflops\": %.2f}\n", grid, threads, fl / ms / 1e9);
      // DMMA m8n8k4
      dmma884_kernel<IT><<<grid, threads>>>(out, 1.0, 1e-7);
      cudaEventRecord(e0); dmma884_kernel<IT><<<grid, threads>>>(out, 1.0, 1e-7); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 256 * 8 * IT * (double)grid * (threads / 32);
      printf("{\"kernel\": \"dmma_m8n8k4\", \"grid\": %d, \"threads\": %d, \"tflops\": %.2f}\n", grid, threads, fl / ms / 1e9);
      // DMMA m16n8k16
      dmma16816_kernel<IT / 4><<<grid, threads>>>(out, 1.0, 1e-7);
      cudaEventRecord(e0); dmma16816_kernel<IT / 4><<<grid, threads>>>(out, 1.0, 1e-7); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 16 * 8 * 16 * 4 * (IT / 4) * (double)grid * (threads / 32);
      printf("{\"kernel\": \"dmma_m16n8k16\", \"grid\": %d, \"threads\": %d, \"tflops\": %.2f}\n", grid, threads, fl / ms / 1e9);
      // mixed
      mixed_kernel<IT><<<grid, threads>>>(out, 1.0, 1e-7);
      cudaEventRecord(e0); mixed_kernel<IT><<<grid, threads>>>(out, 1.0, 1e-7); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      fl = (2.0 * 256 * 8 * IT + 2.0 * 16 * 2 * IT * 32) * (double)grid * (threads / 64);
      printf("{\"kernel\": \"mixed_dmma_dfma\", \"grid\": %d, \"threads\": %d, \"tflops\": %.2f}\n", grid, threads, fl / ms / 1e9);
    }
  }
  // HBM copy bandwidth (fp64), 2 GiB
  size_t n = (size_t)1 << 28; double *a, *b; CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8));
  cudaMemset(a, 0, n * 8);
  for (int r = 0; r < 3; ++r) cudaMemcpy(b, a, n * 8, cudaMemcpyDeviceToDevice);
  float best = 1e9;
  for (int r = 0; r < 10; ++r) { float ms; cudaEventRecord(e0); cudaMemcpy(b, a, n * 8, cudaMemcpyDeviceToDevice); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
  printf("{\"kernel\": \"d2d_copy\", \"gbs\": %.1f}\n", 2.0 * n * 8 / best / 1e6);
  return 0;
}
