// Microbenchmark of the exact z generator pieces (tools only).
#include <cstdio>
#include <cuda_runtime.h>
#include "zgen_warp.cuh"

__global__ void k_philox(uint64_t n_blocks, uint64_t seed, uint64_t *sink) {
  uint64_t acc = 0;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < n_blocks;
       b += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t r[4];
    zo2_raw_block(seed, 0, b, r);
    acc ^= r[0] ^ r[1] ^ r[2] ^ r[3];
  }
  if (acc == 0x12345) *sink = acc;
}
__global__ void k_lane(uint64_t n_blocks, uint64_t seed, double *sink) {
  double acc = 0;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < n_blocks;
       b += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t r[4];
    zo2_raw_block(seed, 0, b, r);
#pragma unroll
    for (int j = 0; j < 4; ++j) acc += zo2_ndtri(zo2_u53(r[j]));
  }
  if (acc == 1234.5) *sink = acc;
}
template <int NB>
__global__ void k_warp(uint64_t n_blocks, uint64_t seed, double *sink) {
  __shared__ ZgenScratch<4 * NB> sc[8];
  double acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * NB;
  for (uint64_t b0 = (blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u)) * NB;
       b0 < n_blocks; b0 += stride) {
    double u[4 * NB], z[4 * NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      uint64_t r[4];
      zo2_raw_block(seed, 0, b0 + (threadIdx.x & 31) + 32 * k, r);
#pragma unroll
      for (int j = 0; j < 4; ++j) u[4 * k + j] = zo2_u53(r[j]);
    }
    warp_ndtri<4 * NB>(u, z, sc[threadIdx.x / 32]);
#pragma unroll
    for (int j = 0; j < 4 * NB; ++j) acc += z[j];
  }
  if (acc == 1234.5) *sink = acc;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  const uint64_t nb = 1ull << 26;  // 2^28 draws
  uint64_t *s64;
  double *sd;
  cudaMalloc(&s64, 8);
  cudaMalloc(&sd, 8);
  const double nz = 4.0 * nb;
  for (int g : {148 * 4, 148 * 8, 148 * 16}) {
    float t0 = timeit([&] { k_philox<<<g, 256>>>(nb, 7, s64); });
    float t1 = timeit([&] { k_lane<<<g, 256>>>(nb, 7, sd); });
    float t2 = timeit([&] { k_warp<1><<<g, 256>>>(nb, 7, sd); });
    float t3 = timeit([&] { k_warp<2><<<g, 256>>>(nb, 7, sd); });
    printf("grid %5d  philox %.1f G/s  lane-ndtri %.1f Gz/s  warp-ndtri(4) %.1f Gz/s  warp-ndtri(8) %.1f Gz/s\n",
           g, nz / t0 / 1e6, nz / t1 / 1e6, nz / t2 / 1e6, nz / t3 / 1e6);
  }
  cudaError_t e = cudaGetLastError();
  printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
