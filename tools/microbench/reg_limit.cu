// Register allocation granularity probe: the largest CTA a kernel of R registers/thread can launch.
// Measured on B200 (round 2): 124/126 regs -> 512 threads, 140..166 regs -> 384 threads, i.e. a CTA
// above 128 registers/thread is limited to 12 warps (registers are granted in 4-warp units).
#include <cstdio>
template <int R>
__global__ void __maxnreg__(R) k(double* out, int n) {
  double a[R / 2 - 8];
#pragma unroll
  for (int i = 0; i < R / 2 - 8; ++i) a[i] = out[(threadIdx.x + i) % n];
  double s = 0;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < R / 2 - 8; ++i) { a[i] = a[i] * a[(i + 1) % (R / 2 - 8)] + 1.0; s += a[i]; }
  out[threadIdx.x] = s;
}
template <int R>
void probe(double* d) {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k<R>);
  k<R><<<1, fa.maxThreadsPerBlock>>>(d, 4);
  cudaError_t e = cudaDeviceSynchronize();
  printf("regs=%d -> maxThreadsPerBlock %d (%s)\n", fa.numRegs, fa.maxThreadsPerBlock,
         e == cudaSuccess ? "launch ok" : cudaGetErrorString(e));
}
int main() {
  double* d;
  cudaMalloc(&d, 4096 * sizeof(double));
  cudaMemset(d, 0, 4096 * sizeof(double));
  probe<128>(d); probe<136>(d); probe<144>(d); probe<152>(d); probe<168>(d);
  return 0;
}
