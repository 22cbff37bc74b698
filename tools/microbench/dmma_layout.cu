// Fragment-layout check of the fp64 mma.sync shapes the kernels use (m16n8k4, m16n8k8): one warp
// multiplies a known A (16 x K) by B (K x 8) with the register mapping the kernels assume, and the
// result is compared with a host triple loop.  Prints one JSON line per shape; exit code 1 on a
// mismatch.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k8(const double* A, const double* B, double* C) {   // A 16x8, B 8x8, row-major
  const int lane = threadIdx.x, gid = lane >> 2, tig = lane & 3;
  double a[4], b[2], c[4] = {0, 0, 0, 0};
  for (int i = 0; i < 4; ++i) a[i] = A[(gid + 8 * (i & 1)) * 8 + tig + 4 * (i >> 1)];
  for (int i = 0; i < 2; ++i) b[i] = B[(tig + 4 * i) * 8 + gid];
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  for (int i = 0; i < 4; ++i) C[(gid + 8 * (i >> 1)) * 8 + 2 * tig + (i & 1)] = c[i];
}

__global__ void k4(const double* A, const double* B, double* C) {   // A 16x4, B 4x8
  const int lane = threadIdx.x, gid = lane >> 2, tig = lane & 3;
  double a0 = A[gid * 4 + tig], a1 = A[(gid + 8) * 4 + tig], b = B[tig * 8 + gid];
  double c[4] = {0, 0, 0, 0};
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
  for (int i = 0; i < 4; ++i) C[(gid + 8 * (i >> 1)) * 8 + 2 * tig + (i & 1)] = c[i];
}

int check(const char* name, int K, void (*kern)(const double*, const double*, double*)) {
  double hA[16 * 8], hB[8 * 8], hC[16 * 8], ref[16 * 8];
  for (int i = 0; i < 16 * K; ++i) hA[i] = (double)((i * 7 + 3) % 23) - 11.0;
  for (int i = 0; i < K * 8; ++i) hB[i] = (double)((i * 5 + 1) % 19) - 9.0;
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 8; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += hA[i * K + k] * hB[k * 8 + j];
      ref[i * 8 + j] = s;
    }
  double *dA, *dB, *dC;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dC, sizeof hC);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  kern<<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(hC, dC, sizeof hC, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 128; ++i) bad += hC[i] != ref[i];
  printf("{\"shape\": \"%s\", \"mismatches\": %d, \"err\": \"%s\"}\n", name, bad, cudaGetErrorString(cudaGetLastError()));
  return bad;
}

int main() {
  int bad = check("m16n8k4", 4, k4) + check("m16n8k8", 8, k8);
  return bad ? 1 : 0;
}
