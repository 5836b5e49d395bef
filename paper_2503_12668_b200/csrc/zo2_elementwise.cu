// zo2_elementwise.cu -- K1 (Gaussian direction), parameter init, K9 (wire
// codecs), the plain reference axpy and K10 (projected gradient) for sm_100a.
// K2 (fused update/perturb) lives in zo2_k2.cu.
//
// All of these are HBM- or FP64-pipe-bound element-wise passes: one thread
// owns one Philox block (4 consecutive parameters), loads/stores are 16-byte
// vectors, grids are sized in multiples of the 148 SMs.
#include "zo2_common.cuh"
#include "zo2_rng.h"
#include "zo2_rng_fast.h"
#include <atomic>
#include <string.h>
#include <stdio.h>

static std::atomic<uint64_t> g_launches{0};
static thread_local char g_err[512] = "";

extern "C" const char *zo2_last_error(void) { return g_err; }
extern "C" int zo2_version(void) { return 1; }
extern "C" uint64_t zo2_launch_count(void) { return g_launches.load(); }
void zo2_count_launch(uint64_t n = 1) { g_launches.fetch_add(n); }

int zo2_set_cuda_error(cudaError_t e) {
  snprintf(g_err, sizeof(g_err), "CUDA error %d: %s", (int)e, cudaGetErrorString(e));
  return ZO2_E_CUDA;
}
int zo2_set_error(int code, const char *msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

static inline cudaStream_t S(void *s) { return (cudaStream_t)s; }

// ------------------------------------------------------------------ K1
__device__ __forceinline__ void z4_at(uint64_t seed, uint64_t stream, uint64_t pos,
                                      double z[4]) {
  // z for positions pos..pos+3; pos % 4 == 0 -> one Philox block.
  if ((pos & 3) == 0) {
    uint64_t r[4];
    zo2_raw_block(seed, stream, pos >> 2, r);
#pragma unroll
    for (int j = 0; j < 4; ++j) z[j] = zo2_ndtri(zo2_u53(r[j]));
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) z[j] = zo2_gauss_at(seed, stream, pos + j);
  }
}

__global__ void k_z_fill(double *out, uint64_t n, uint64_t seed, uint64_t stream,
                         uint64_t counter) {
  const uint64_t b0 = counter >> 2, lane0 = counter & 3;
  const uint64_t nb = (lane0 + n + 3) >> 2;  // blocks touched; positions never wrap
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nb;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = b0 + t;
    uint64_t r[4];
    zo2_raw_block(seed, stream, b, r);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t i = 4 * t + j - lane0;  // wraps for j < lane0 at t == 0
      if (4 * t + j >= lane0 && i < n) out[i] = zo2_ndtri(zo2_u53(r[j]));
    }
  }
}

__global__ void k_raw_fill(uint64_t *out, uint64_t n, uint64_t seed, uint64_t stream,
                           uint64_t counter) {
  const uint64_t b0 = counter >> 2, lane0 = counter & 3;
  const uint64_t nb = (lane0 + n + 3) >> 2;  // blocks touched; positions never wrap
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nb;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = b0 + t;
    uint64_t r[4];
    zo2_raw_block(seed, stream, b, r);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t i = 4 * t + j - lane0;
      if (4 * t + j >= lane0 && i < n) out[i] = r[j];
    }
  }
}

extern "C" int zo2_z_fill(double *out, uint64_t n, uint64_t seed, uint64_t stream,
                          uint64_t counter, void *cs) {
  if (n == 0) return ZO2_OK;
  if (!out) return zo2_set_error(ZO2_E_ARG, "zo2_z_fill: null output");
  const uint64_t blocks = ((counter & 3) + n + 3) >> 2;
  k_z_fill<<<zo2_grid_for(blocks, 256), 256, 0, S(cs)>>>(out, n, seed, stream, counter);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

// rng = "fast" direction probe (zo2_rng_fast.h), binary32.
__global__ void k_z_fill_fast(float *out, uint64_t n, uint64_t seed, uint64_t stream,
                              uint64_t counter) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = zo2f_gauss_at(seed, stream, counter + i);
}

extern "C" int zo2_z_fill_fast(float *out, uint64_t n, uint64_t seed, uint64_t stream,
                               uint64_t counter, void *cs) {
  if (n == 0) return ZO2_OK;
  if (!out) return zo2_set_error(ZO2_E_ARG, "zo2_z_fill_fast: null output");
  k_z_fill_fast<<<zo2_grid_for(n, 256), 256, 0, S(cs)>>>(out, n, seed, stream, counter);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

extern "C" int zo2_host_z_fill_fast(float *out, uint64_t n, uint64_t seed, uint64_t stream,
                                    uint64_t counter) {
  for (uint64_t i = 0; i < n; ++i) out[i] = zo2f_gauss_at(seed, stream, counter + i);
  return ZO2_OK;
}

extern "C" int zo2_raw_fill(uint64_t *out, uint64_t n, uint64_t seed, uint64_t stream,
                            uint64_t counter, void *cs) {
  if (n == 0) return ZO2_OK;
  if (!out) return zo2_set_error(ZO2_E_ARG, "zo2_raw_fill: null output");
  const uint64_t blocks = ((counter & 3) + n + 3) >> 2;
  k_raw_fill<<<zo2_grid_for(blocks, 256), 256, 0, S(cs)>>>(out, n, seed, stream, counter);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

extern "C" int zo2_host_raw_u64(uint64_t *out, uint64_t n, uint64_t seed,
                                uint64_t stream, uint64_t counter) {
  uint64_t r[4], b = counter >> 2, j = counter & 3;
  for (uint64_t i = 0; i < n; ++b, j = 0) {
    zo2_raw_block(seed, stream, b, r);
    for (; j < 4 && i < n; ++j, ++i) out[i] = r[j];
  }
  return ZO2_OK;
}

extern "C" int zo2_host_gaussian_fill(double *out, uint64_t n, uint64_t seed,
                                      uint64_t stream, uint64_t counter) {
  uint64_t r[4], b = counter >> 2, j = counter & 3;
  for (uint64_t i = 0; i < n; ++b, j = 0) {
    zo2_raw_block(seed, stream, b, r);
    for (; j < 4 && i < n; ++j, ++i) out[i] = zo2_ndtri(zo2_u53(r[j]));
  }
  return ZO2_OK;
}

extern "C" uint64_t zo2_host_derive_step_seed(uint64_t base, uint64_t j) {
  return zo2_derive_step_seed(base, j);
}

// init: out = fmt(std * z), model.py:221-223 ((std * z).astype(storage)).
template <typename T>
__global__ void k_init_normal(T *out, uint64_t n, double sd, uint64_t seed,
                              uint64_t counter) {
  const uint64_t b0 = counter >> 2, lane0 = counter & 3;
  const uint64_t nb = (lane0 + n + 3) >> 2;  // blocks touched; positions never wrap
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nb;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = b0 + t;
    uint64_t r[4];
    zo2_raw_block(seed, ZO2_INIT_STREAM, b, r);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t i = 4 * t + j - lane0;
      if (4 * t + j >= lane0 && i < n) out[i] = (T)__dmul_rn(sd, zo2_ndtri(zo2_u53(r[j])));
    }
  }
}

extern "C" int zo2_init_normal(void *out, int fmt, uint64_t n, double sd, uint64_t seed,
                               uint64_t counter, void *cs) {
  if (n == 0) return ZO2_OK;
  const uint64_t blocks = ((counter & 3) + n + 3) >> 2;
  const unsigned g = zo2_grid_for(blocks, 256);
  if (fmt == ZO2_F32)
    k_init_normal<float><<<g, 256, 0, S(cs)>>>((float *)out, n, sd, seed, counter);
  else if (fmt == ZO2_F64)
    k_init_normal<double><<<g, 256, 0, S(cs)>>>((double *)out, n, sd, seed, counter);
  else
    return zo2_set_error(ZO2_E_ARG, "zo2_init_normal: fmt must be F32 or F64");
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

template <typename T>
__global__ void k_fill_const(T *out, uint64_t n, T v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = v;
}

extern "C" int zo2_fill_const(void *out, int fmt, uint64_t n, double v, void *cs) {
  if (n == 0) return ZO2_OK;
  const unsigned g = zo2_grid_for(n, 256);
  if (fmt == ZO2_F32)
    k_fill_const<float><<<g, 256, 0, S(cs)>>>((float *)out, n, (float)v);
  else if (fmt == ZO2_F64)
    k_fill_const<double><<<g, 256, 0, S(cs)>>>((double *)out, n, v);
  else
    return zo2_set_error(ZO2_E_ARG, "zo2_fill_const: fmt must be F32 or F64");
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

#include "zo2_wire.cuh"


template <int FMT>
__global__ void k_encode(const float *src, void *dst, uint64_t n, uint64_t *counts) {
  unsigned nn = 0, ns = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  // full loop trip count so the whole warp reaches the shuffle reduction
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
    const uint64_t i = i0 + threadIdx.x;
    if (i < n) {
      const float x = src[i];
      if (FMT == ZO2_BF16) ((uint16_t *)dst)[i] = enc_bf16(x, nn, ns);
      else if (FMT == ZO2_F16) ((uint16_t *)dst)[i] = enc_f16(x, nn, ns);
      else ((uint8_t *)dst)[i] = enc_e4m3(x, nn, ns);
    }
  }
  add_counts(counts, nn, ns);
}

template <int FMT>
__global__ void k_decode(const void *src, float *dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (FMT == ZO2_BF16) dst[i] = dec_bf16(((const uint16_t *)src)[i]);
    else if (FMT == ZO2_F16) dst[i] = dec_f16(((const uint16_t *)src)[i]);
    else dst[i] = dec_e4m3(((const uint8_t *)src)[i]);
  }
}

extern "C" int zo2_encode(const float *src, void *dst, int fmt, uint64_t n,
                          uint64_t *counts, void *cs) {
  if (n == 0) return ZO2_OK;
  const unsigned g = zo2_grid_for(n, 256);
  if (fmt == ZO2_BF16) k_encode<ZO2_BF16><<<g, 256, 0, S(cs)>>>(src, dst, n, counts);
  else if (fmt == ZO2_F16) k_encode<ZO2_F16><<<g, 256, 0, S(cs)>>>(src, dst, n, counts);
  else if (fmt == ZO2_F8E4M3) k_encode<ZO2_F8E4M3><<<g, 256, 0, S(cs)>>>(src, dst, n, counts);
  else return zo2_set_error(ZO2_E_ARG, "zo2_encode: fmt must be F16, BF16 or F8E4M3");
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

extern "C" int zo2_decode(const void *src, float *dst, int fmt, uint64_t n, void *cs) {
  if (n == 0) return ZO2_OK;
  const unsigned g = zo2_grid_for(n, 256);
  if (fmt == ZO2_BF16) k_decode<ZO2_BF16><<<g, 256, 0, S(cs)>>>(src, dst, n);
  else if (fmt == ZO2_F16) k_decode<ZO2_F16><<<g, 256, 0, S(cs)>>>(src, dst, n);
  else if (fmt == ZO2_F8E4M3) k_decode<ZO2_F8E4M3><<<g, 256, 0, S(cs)>>>(src, dst, n);
  else return zo2_set_error(ZO2_E_ARG, "zo2_decode: fmt must be F16, BF16 or F8E4M3");
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

// Plain axpy with regenerated z (reference-exact single op).
template <typename T>
__global__ void k_axpy_z(T *w, uint64_t n, double coef, uint64_t seed, uint64_t stream,
                         uint64_t counter) {
  const uint64_t b0 = counter >> 2, lane0 = counter & 3;
  const uint64_t nb = (lane0 + n + 3) >> 2;  // blocks touched; positions never wrap
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nb;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = b0 + t;
    uint64_t r[4];
    zo2_raw_block(seed, stream, b, r);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t i = 4 * t + j - lane0;
      if (4 * t + j >= lane0 && i < n) w[i] = axpy1(w[i], coef, zo2_ndtri(zo2_u53(r[j])));
    }
  }
}

extern "C" int zo2_axpy_z(void *w, int fmt, uint64_t n, double coef, uint64_t seed,
                          uint64_t stream, uint64_t counter, void *cs) {
  if (n == 0) return ZO2_OK;
  const uint64_t blocks = ((counter & 3) + n + 3) >> 2;
  const unsigned g = zo2_grid_for(blocks, 256);
  if (fmt == ZO2_F32)
    k_axpy_z<float><<<g, 256, 0, S(cs)>>>((float *)w, n, coef, seed, stream, counter);
  else if (fmt == ZO2_F64)
    k_axpy_z<double><<<g, 256, 0, S(cs)>>>((double *)w, n, coef, seed, stream, counter);
  else
    return zo2_set_error(ZO2_E_ARG, "zo2_axpy_z: fmt must be F32 or F64");
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

// ------------------------------------------------------------------ host pinning
// Page-locks an existing host range (the node-wide shared block masters of a
// data-parallel job, runtime.SharedHostMasters) so cudaMemcpyAsync moves it by
// DMA at full PCIe rate; portable = usable from every device of the process.
extern "C" int zo2_host_register(void *ptr, uint64_t bytes) {
  if (!ptr || bytes == 0) return zo2_set_error(ZO2_E_ARG, "zo2_host_register: empty range");
  ZO2_CUDA_TRY(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable));
  return ZO2_OK;
}
extern "C" int zo2_host_unregister(void *ptr) {
  ZO2_CUDA_TRY(cudaHostUnregister(ptr));
  return ZO2_OK;
}

// ------------------------------------------------------------------ K10
__global__ void k_form_g(const double *sums, double count, double eps, double *out,
                         int *flag) {
  const double lp = sums[0] / count, lm = sums[1] / count;
  out[0] = lp;
  out[1] = lm;
  const bool fin = isfinite(lp) && isfinite(lm);
  out[2] = fin ? (lp - lm) / (2.0 * eps) : 0.0;
  if (flag) *flag = fin ? 0 : 1;
}

extern "C" int zo2_form_g(const double *d_sums, double count, double eps, double *d_out,
                          int *d_flag, void *cs) {
  k_form_g<<<1, 1, 0, S(cs)>>>(d_sums, count, eps, d_out, d_flag);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}
