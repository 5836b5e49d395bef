// Pipe-throughput probe (tools only): FP64 add/mul/fma, FP32 fma, 64-bit
// integer multiply-high, MUFU rcp64h -- lane-ops per clock per SM on this GPU.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
template <int OP>
__global__ void k_probe(int iters, double seed, double *sink, long long *cycles) {
  double a[CH];
  float f[CH];
  uint64_t u[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    a[i] = seed + i * 1e-3 + threadIdx.x * 1e-7;
    f[i] = (float)a[i];
    u[i] = (uint64_t)(a[i] * 1e9) * 0x9E3779B97F4A7C15ULL;
  }
  const double m = 0.999999, c = 1e-9;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (OP == 0) a[i] = __fma_rn(a[i], m, c);
      if (OP == 1) a[i] = __dmul_rn(a[i], m);
      if (OP == 2) a[i] = __dadd_rn(a[i], c);
      if (OP == 3) f[i] = __fmaf_rn(f[i], (float)m, (float)c);
      if (OP == 4) u[i] = __umul64hi(u[i], 0xD2E7470EE14C6C93ULL) ^ u[i];
      if (OP == 5) u[i] = u[i] * 0xD2E7470EE14C6C93ULL + 1;
      if (OP == 6) a[i] = __drcp_rn(a[i]);
      if (OP == 7) a[i] = __ddiv_rn(c, a[i]) + 1.0;
      if (OP == 8) a[i] = __dsqrt_rn(a[i]) + 1.0;
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += a[i] + f[i] + (double)(u[i] & 0xff);
  if (s == 1234.5) *sink = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

template <int OP>
void run(const char *name, int blocks_per_sm, int threads) {
  double *sink;
  long long *cyc;
  cudaMalloc(&sink, 8);
  cudaMalloc(&cyc, 8);
  const int iters = 4096;
  k_probe<OP><<<148 * blocks_per_sm, threads>>>(iters, 1.0, sink, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double ops_per_sm = (double)blocks_per_sm * threads * iters * CH;
  printf("%-10s blocks/SM %d thr %4d: %.1f lane-ops/clk/SM\n", name, blocks_per_sm, threads,
         ops_per_sm / (double)h);
  cudaFree(sink);
  cudaFree(cyc);
}

int main() {
  for (int b : {2, 4}) {
    run<0>("dfma", b, 256);
    run<1>("dmul", b, 256);
    run<2>("dadd", b, 256);
    run<3>("ffma", b, 256);
    run<4>("umul64hi", b, 256);
    run<5>("mul64lo", b, 256);
    run<6>("drcp_rn", b, 256);
    run<7>("ddiv_rn", b, 256);
    run<8>("dsqrt_rn", b, 256);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
