// Pipe-overlap probe for a warp-specialised K2 (tools only): does Philox4x64
// (integer multiply pipe) running in some warps overlap with the exact
// central ndtri (FP64 pipe) running in others on the same SM?
//   philox-only, ndtri-only, and mixed (even warps Philox, odd warps ndtri,
//   each doing the same per-warp work as in the pure kernels).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_12668_b200/csrc \
//      -I include tools/pipe_overlap_probe.cu -o tools/pipe_overlap_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "zo2_zexact.cuh"

__device__ __forceinline__ void philox_work(uint64_t b0, int iters, uint64_t &acc) {
  for (int i = 0; i < iters; ++i) {
    uint64_t r[4];
    zx_philox_block(0x1234567ull, 0, b0 + (uint64_t)i * 7919u, r);
    acc ^= r[0] ^ r[1] ^ r[2] ^ r[3];
  }
}
__device__ __forceinline__ void ndtri_work(double y0, int iters, double &acc) {
  const ZxCentral cc = zx_central_coef(ZX_CENTRAL_C);
  double y = y0;
  for (int i = 0; i < iters; ++i) {
    const double a = zx_ndtri_central(y, cc);
    const double b = zx_ndtri_central(1.0 - y, cc);
    acc += a + b;
    y = 0.2 + 0.6 * (double)((i * 37 + threadIdx.x) & 1023) / 1024.0;
  }
}

// mode 0: all warps Philox; 1: all warps ndtri; 2: even warps Philox, odd ndtri
__global__ void __launch_bounds__(256) k_probe(int mode, int ip, int in, uint64_t *s1, double *s2) {
  const int warp = threadIdx.x >> 5;
  uint64_t a1 = 0;
  double a2 = 0;
  const bool ph = mode == 0 || (mode == 2 && (warp & 1) == 0);
  if (ph) philox_work(blockIdx.x * 256ull + threadIdx.x, ip, a1);
  else ndtri_work(0.3 + threadIdx.x * 1e-4, in, a2);
  if (a1 == 0x5 || a2 == 0.5) { *s1 = a1; *s2 = a2; }
}

int main() {
  uint64_t *s1;
  double *s2;
  cudaMalloc(&s1, 8);
  cudaMalloc(&s2, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 4, ip = 2048, in = 1024;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float t[3];
  for (int mode = 0; mode < 3; ++mode) {
    k_probe<<<grid, 256>>>(mode, ip, in, s1, s2);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_probe<<<grid, 256>>>(mode, ip, in, s1, s2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t[mode], e0, e1);
    t[mode] /= 5;
  }
  // mixed does half the Philox work and half the ndtri work of the pure runs
  printf("philox-only %.3f ms, ndtri-only %.3f ms, mixed (half of each) %.3f ms; "
         "serial half+half would be %.3f ms, perfect overlap %.3f ms\n",
         t[0], t[1], t[2], 0.5f * (t[0] + t[1]), 0.5f * (t[0] > t[1] ? t[0] : t[1]) * 2.0f / 2.0f);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
