// Micro-benchmark: the pure memory pattern of the fused SpMM on the Large operator, no arithmetic.
//   read  : each CTA (256 threads) streams its tile's six value segments (900 fp64 each, contiguous)
//   write : each CTA writes 20 node-rows x 3 streams x 60 fp64 into a row-major M x 186 matrix
//   both  : read + write (what the SpMM must move, minus U and descriptors)
// Reports GB/s of the bytes actually moved.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kTileNnz = 900, kRows = 20, kR = 60, kLd = 186;

// MODE 0 read, 1 write (interleaved ld 186), 2 read + write, 3 write three separate M x 60 arrays,
// 4 write interleaved with default (write-back) stores, 5 read + write separate arrays
template <int MODE>
__global__ void __launch_bounds__(256) pattern(const double* const* v, double* out, int ntiles, double* sink) {
  const int t = blockIdx.x;
  if (t >= ntiles) return;
  double acc = 0.0;
  if (MODE == 0 || MODE == 2 || MODE == 5) {
    const size_t e0 = (size_t)t * kTileNnz;
    double raw[4][6];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = threadIdx.x + k * 256;
      if (e < kTileNnz)
#pragma unroll
        for (int s = 0; s < 6; ++s) raw[k][s] = __ldcs(v[s] + e0 + e);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (threadIdx.x + k * 256 < kTileNnz)
#pragma unroll
        for (int s = 0; s < 6; ++s) acc += raw[k][s];
  }
  const size_t row0 = (size_t)t * kRows;
  if (MODE == 1 || MODE == 2) {
    for (int e = threadIdx.x; e < kRows * 3 * kR; e += 256) {
      const int q = e / (3 * kR), rem = e - q * 3 * kR;
      __stcs(out + (row0 + q) * kLd + 5 + rem, acc + e);
    }
  } else if (MODE == 4) {
    for (int e = threadIdx.x; e < kRows * 3 * kR; e += 256) {
      const int q = e / (3 * kR), rem = e - q * 3 * kR;
      out[(row0 + q) * kLd + 5 + rem] = acc + e;
    }
  } else if (MODE == 3 || MODE == 5) {
    const size_t Mtot = (size_t)gridDim.x * kRows;
    for (int e = threadIdx.x; e < kRows * 3 * kR; e += 256) {
      const int st = e / (kRows * kR), rem = e - st * kRows * kR;
      __stcs(out + st * Mtot * kR + row0 * kR + rem, acc + e);
    }
  } else if (acc == 12345.0) {
    sink[0] = acc;
  }
}

int main() {
  const int ntiles = 65536;
  const size_t nnz = (size_t)ntiles * kTileNnz;
  const size_t M = (size_t)ntiles * kRows;
  double* vals[6];
  for (int s = 0; s < 6; ++s) { cudaMalloc(&vals[s], nnz * 8); cudaMemset(vals[s], 0, nnz * 8); }
  double** dv; cudaMalloc(&dv, sizeof(vals)); cudaMemcpy(dv, vals, sizeof(vals), cudaMemcpyHostToDevice);
  double* out; cudaMalloc(&out, M * kLd * 8);
  double* sink; cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double rb = 6.0 * nnz * 8, wb = (double)M * 3 * kR * 8;
  const char* names[6] = {"read six streams", "write interleaved ld186 (stcs)", "read + write interleaved",
                          "write 3 separate arrays (stcs)", "write interleaved (default st)", "read + write separate"};
  for (int mode = 0; mode < 6; ++mode) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) pattern<0><<<ntiles, 256>>>(dv, out, ntiles, sink);
      if (mode == 1) pattern<1><<<ntiles, 256>>>(dv, out, ntiles, sink);
      if (mode == 2) pattern<2><<<ntiles, 256>>>(dv, out, ntiles, sink);
      if (mode == 3) pattern<3><<<ntiles, 256>>>(dv, out, ntiles, sink);
      if (mode == 4) pattern<4><<<ntiles, 256>>>(dv, out, ntiles, sink);
      if (mode == 5) pattern<5><<<ntiles, 256>>>(dv, out, ntiles, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double bytes = ((mode == 0 || mode == 2 || mode == 5) ? rb : 0) + (mode >= 1 ? wb : 0);
    printf("{\"pattern\": \"%s\", \"ms\": %.3f, \"GBps\": %.0f, \"err\": \"%s\"}\n", names[mode], best,
           bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
