// zo2_elementwise.cu -- K1 (Gaussian direction), K2 (fused update/perturb),
// K9 (wire codecs), K10 (projected gradient) for sm_100a.
//
// All of these are HBM- or FP64-pipe-bound element-wise passes: one thread
// owns one Philox block (4 consecutive parameters), loads/stores are 16-byte
// vectors, grids are sized in multiples of the 148 SMs.
#include "zo2_common.cuh"
#include "zo2_rng.h"
#include "zo2_zgen.cuh"
#include <atomic>
#include <string.h>
#include <stdio.h>

static std::atomic<uint64_t> g_launches{0};
// K2 grid = 148 x this; 1 leaves room on every SM for the persistent GEMM CTA
// when the prepare lane runs concurrently with the compute lane
static unsigned g_k2_ctas_per_sm = 2;

extern "C" int zo2_set_k2_ctas_per_sm(int n) {
  if (n < 1 || n > 32) return zo2_set_error(ZO2_E_ARG, "zo2_set_k2_ctas_per_sm: 1..32");
  g_k2_ctas_per_sm = (unsigned)n;
  return ZO2_OK;
}
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

// ------------------------------------------------------------------ codecs
// bf16 (numerics.py:232-245)
__device__ __forceinline__ uint16_t enc_bf16(float x, unsigned &nn, unsigned &ns) {
  const uint32_t u = __float_as_uint(x);
  uint16_t r = (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
  const uint16_t sign = r & 0x8000u;
  if (x != x) {
    ++nn;
    return sign | 0x7FC0u;
  }
  if ((r & 0x7FFFu) >= 0x7F80u) {
    ++ns;
    return sign | 0x7F7Fu;
  }
  return r;
}
__device__ __forceinline__ float dec_bf16(uint16_t b) {
  return __uint_as_float((uint32_t)b << 16);
}
// f16 (numerics.py:220-229): numpy RNE cast; NaN keeps sign and the top
// mantissa bits (kept non-zero); finite overflow saturates to +-65504.
__device__ __forceinline__ uint16_t enc_f16(float x, unsigned &nn, unsigned &ns) {
  const uint32_t u = __float_as_uint(x);
  if (x != x) {
    ++nn;
    uint16_t r = (uint16_t)(0x7C00u + ((u & 0x007FFFFFu) >> 13));
    if (r == 0x7C00u) ++r;
    return (uint16_t)(((u >> 16) & 0x8000u) + r);
  }
  uint16_t h = __half_as_ushort(__float2half_rn(x));
  if ((h & 0x7FFFu) == 0x7C00u && (u & 0x7F800000u) != 0x7F800000u) {
    ++ns;
    h = (uint16_t)((h & 0x8000u) | 0x7BFFu);
  }
  return h;
}
// f16 -> f32 widening; NaN payloads are kept (mantissa << 13) as numpy's
// astype does, so a decode/encode round trip is the identity.
__device__ __forceinline__ float dec_f16(uint16_t b) {
  if ((b & 0x7C00u) == 0x7C00u && (b & 0x3FFu))
    return __uint_as_float(((uint32_t)(b & 0x8000u) << 16) | 0x7F800000u |
                           ((uint32_t)(b & 0x3FFu) << 13));
  return __half2float(__ushort_as_half(b));
}
// e4m3 (numerics.py:248-270), evaluated in double exactly as the reference.
__device__ __forceinline__ uint8_t enc_e4m3(float xf, unsigned &nn, unsigned &ns) {
  const double x = (double)xf;
  const bool nan_ = x != x;
  const bool neg = signbit(x);
  double mag = nan_ ? 0.0 : fabs(x);
  if (mag > 448.0) {
    ++ns;
    mag = 448.0;
  }
  int ex;
  frexp(mag, &ex);
  int e = ex - 1;
  if (e < -6) e = -6;
  const double step = ldexp(1.0, e - 3);
  double q = rint(__ddiv_rn(mag, step));
  if (q >= 16.0) {
    e += 1;
    q = 8.0;
  }
  const int qi = (int)q;
  uint8_t code = qi >= 8 ? (uint8_t)(((e + 7) << 3) + (qi - 8)) : (uint8_t)qi;
  if (nan_) {
    code = 0x7F;
    ++nn;
  }
  if (neg) code |= 0x80;
  return code;
}
__device__ __forceinline__ float dec_e4m3(uint8_t c) {
  const int ef = (c >> 3) & 0xF;
  const int m = c & 7;
  float v = ef == 0 ? ldexpf((float)m, -9) : ldexpf((float)(8 + m), ef - 10);
  if (ef == 15 && m == 7) v = __int_as_float(0x7FC00000);
  return (c & 0x80) ? -v : v;
}

__device__ __forceinline__ void add_counts(uint64_t *d, unsigned nn, unsigned ns) {
  if (!d) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nn += __shfl_xor_sync(0xffffffffu, nn, o);
    ns += __shfl_xor_sync(0xffffffffu, ns, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (nn) atomicAdd((unsigned long long *)&d[0], (unsigned long long)nn);
    if (ns) atomicAdd((unsigned long long *)&d[1], (unsigned long long)ns);
  }
}

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

// ------------------------------------------------------------------ K2
// Storage access for the arena in its wire format.  Arithmetic type A is
// double for the F64 wire, float otherwise (codec => f32, config.py:112).
template <int FMT> struct Wire;
template <> struct Wire<ZO2_F64> {
  typedef double A;
  static __device__ __forceinline__ void load4(const void *p, uint64_t i, double w[4]) {
    const double2 *q = (const double2 *)((const double *)p + i);
    double2 a = q[0], b = q[1];
    w[0] = a.x; w[1] = a.y; w[2] = b.x; w[3] = b.y;
  }
  static __device__ __forceinline__ void store4(void *p, uint64_t i, const double w[4],
                                                unsigned &, unsigned &) {
    double2 *q = (double2 *)((double *)p + i);
    q[0] = make_double2(w[0], w[1]);
    q[1] = make_double2(w[2], w[3]);
  }
  static __device__ __forceinline__ double load1(const void *p, uint64_t i) {
    return ((const double *)p)[i];
  }
  static __device__ __forceinline__ void store1(void *p, uint64_t i, double w, unsigned &,
                                                unsigned &) {
    ((double *)p)[i] = w;
  }
};
template <> struct Wire<ZO2_F32> {
  typedef float A;
  static __device__ __forceinline__ void load4(const void *p, uint64_t i, float w[4]) {
    float4 a = *(const float4 *)((const float *)p + i);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
  }
  static __device__ __forceinline__ void store4(void *p, uint64_t i, const float w[4],
                                                unsigned &, unsigned &) {
    *(float4 *)((float *)p + i) = make_float4(w[0], w[1], w[2], w[3]);
  }
  static __device__ __forceinline__ float load1(const void *p, uint64_t i) {
    return ((const float *)p)[i];
  }
  static __device__ __forceinline__ void store1(void *p, uint64_t i, float w, unsigned &,
                                                unsigned &) {
    ((float *)p)[i] = w;
  }
};
template <> struct Wire<ZO2_BF16> {
  typedef float A;
  static __device__ __forceinline__ void load4(const void *p, uint64_t i, float w[4]) {
    uint2 v = *(const uint2 *)((const uint16_t *)p + i);
    w[0] = dec_bf16(v.x & 0xFFFF); w[1] = dec_bf16(v.x >> 16);
    w[2] = dec_bf16(v.y & 0xFFFF); w[3] = dec_bf16(v.y >> 16);
  }
  static __device__ __forceinline__ void store4(void *p, uint64_t i, const float w[4],
                                                unsigned &nn, unsigned &ns) {
    uint2 v;
    v.x = (uint32_t)enc_bf16(w[0], nn, ns) | ((uint32_t)enc_bf16(w[1], nn, ns) << 16);
    v.y = (uint32_t)enc_bf16(w[2], nn, ns) | ((uint32_t)enc_bf16(w[3], nn, ns) << 16);
    *(uint2 *)((uint16_t *)p + i) = v;
  }
  static __device__ __forceinline__ float load1(const void *p, uint64_t i) {
    return dec_bf16(((const uint16_t *)p)[i]);
  }
  static __device__ __forceinline__ void store1(void *p, uint64_t i, float w, unsigned &nn,
                                                unsigned &ns) {
    ((uint16_t *)p)[i] = enc_bf16(w, nn, ns);
  }
};
template <> struct Wire<ZO2_F16> {
  typedef float A;
  static __device__ __forceinline__ void load4(const void *p, uint64_t i, float w[4]) {
    uint2 v = *(const uint2 *)((const uint16_t *)p + i);
    w[0] = dec_f16(v.x & 0xFFFF); w[1] = dec_f16(v.x >> 16);
    w[2] = dec_f16(v.y & 0xFFFF); w[3] = dec_f16(v.y >> 16);
  }
  static __device__ __forceinline__ void store4(void *p, uint64_t i, const float w[4],
                                                unsigned &nn, unsigned &ns) {
    uint2 v;
    v.x = (uint32_t)enc_f16(w[0], nn, ns) | ((uint32_t)enc_f16(w[1], nn, ns) << 16);
    v.y = (uint32_t)enc_f16(w[2], nn, ns) | ((uint32_t)enc_f16(w[3], nn, ns) << 16);
    *(uint2 *)((uint16_t *)p + i) = v;
  }
  static __device__ __forceinline__ float load1(const void *p, uint64_t i) {
    return dec_f16(((const uint16_t *)p)[i]);
  }
  static __device__ __forceinline__ void store1(void *p, uint64_t i, float w, unsigned &nn,
                                                unsigned &ns) {
    ((uint16_t *)p)[i] = enc_f16(w, nn, ns);
  }
};
template <> struct Wire<ZO2_F8E4M3> {
  typedef float A;
  static __device__ __forceinline__ void load4(const void *p, uint64_t i, float w[4]) {
    uint32_t v = *(const uint32_t *)((const uint8_t *)p + i);
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = dec_e4m3((v >> (8 * j)) & 0xFF);
  }
  static __device__ __forceinline__ void store4(void *p, uint64_t i, const float w[4],
                                                unsigned &nn, unsigned &ns) {
    uint32_t v = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) v |= (uint32_t)enc_e4m3(w[j], nn, ns) << (8 * j);
    *(uint32_t *)((uint8_t *)p + i) = v;
  }
  static __device__ __forceinline__ float load1(const void *p, uint64_t i) {
    return dec_e4m3(((const uint8_t *)p)[i]);
  }
  static __device__ __forceinline__ void store1(void *p, uint64_t i, float w, unsigned &nn,
                                                unsigned &ns) {
    ((uint8_t *)p)[i] = enc_e4m3(w, nn, ns);
  }
};

// One axpy rounding (model.py:233): store(f64(w) + coef*z).  NaN handling
// follows the reference's x86 SSE arithmetic, not CUDA's canonical NaN: a NaN
// weight propagates its own (quieted) payload, an invalid operation yields
// the x86 default NaN (sign set) -- visible through the f16 codec.
__device__ __forceinline__ float axpy1(float w, double coef, double z) {
  if (w != w) return __uint_as_float(__float_as_uint(w) | 0x00400000u);
  const double s = __dadd_rn((double)w, __dmul_rn(coef, z));
  if (s != s) return __uint_as_float(0xFFC00000u);
  return __double2float_rn(s);
}
__device__ __forceinline__ double axpy1(double w, double coef, double z) {
  if (w != w)
    return __longlong_as_double(__double_as_longlong(w) | 0x0008000000000000LL);
  const double s = __dadd_rn(w, __dmul_rn(coef, z));
  if (s != s) return __longlong_as_double((long long)0xFFF8000000000000ULL);
  return s;
}

struct K2Params {
  uint64_t base;  // module RNG offset
  int do_update;
  double ucoef;   // -(lr * g), resolved on device
  uint64_t lrs_seed;
  int do_perturb;
  double eps;
  uint64_t rs_seed;
};

// Applies the per-module op sequence to NQ quads of 4 consecutive elements at
// bucket indices idx[q] (RNG positions base+idx[q] ..): deferred update with
// z(lrs) if UPD, then +eps / -2eps / +eps with z(rs) if PERT, returning W+ /
// W- in wp/wm.  cnt[q] = valid elements of quad q (0: inactive lane slot --
// the lane still joins the warp-cooperative z evaluation).
template <typename A, int NQ, bool UPD, bool PERT>
__device__ __forceinline__ void k2_quads(A (&w)[NQ][4], A (&wp)[NQ][4], A (&wm)[NQ][4],
                                         const uint64_t (&idx)[NQ], const int (&cnt)[NQ],
                                         const K2Params &P,
                                         ZgenScratch<NQ *((UPD ? 4 : 0) + (PERT ? 4 : 0))> &sc) {
  constexpr int PER = (UPD ? 4 : 0) + (PERT ? 4 : 0);
  constexpr int OFF = UPD ? 4 : 0;
#if ZO2_K2_TWO_PHASE
  if (UPD && PERT) {
    // two warp-cooperative passes of 4 draws per quad (update, then perturb):
    // half the live f64 state, more resident warps
    ZgenScratch<NQ * 4> &s4 = *reinterpret_cast<ZgenScratch<NQ * 4> *>(&sc);
    double u[NQ * 4], z[NQ * 4];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      uint64_t r[4];
      if (cnt[q] > 0) zo2_raw4(P.lrs_seed, ZO2_PERTURB_STREAM, P.base + idx[q], r);
#pragma unroll
      for (int j = 0; j < 4; ++j) u[q * 4 + j] = j < cnt[q] ? zo2_u53(r[j]) : 0.5;
    }
    warp_ndtri<NQ * 4>(u, z, s4);
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < cnt[q]) w[q][j] = axpy1(w[q][j], P.ucoef, z[q * 4 + j]);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      uint64_t r[4];
      if (cnt[q] > 0) zo2_raw4(P.rs_seed, ZO2_PERTURB_STREAM, P.base + idx[q], r);
#pragma unroll
      for (int j = 0; j < 4; ++j) u[q * 4 + j] = j < cnt[q] ? zo2_u53(r[j]) : 0.5;
    }
    warp_ndtri<NQ * 4>(u, z, s4);
    const double m2 = -2.0 * P.eps;
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= cnt[q]) continue;
        const double zr = z[q * 4 + j];
        wp[q][j] = axpy1(w[q][j], P.eps, zr);
        wm[q][j] = axpy1(wp[q][j], m2, zr);
        w[q][j] = axpy1(wm[q][j], P.eps, zr);
      }
    return;
  }
#endif
  double u[NQ * PER], z[NQ * PER];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    uint64_t r[4];
    if (UPD) {
      if (cnt[q] > 0) zo2_raw4(P.lrs_seed, ZO2_PERTURB_STREAM, P.base + idx[q], r);
#pragma unroll
      for (int j = 0; j < 4; ++j) u[q * PER + j] = j < cnt[q] ? zo2_u53(r[j]) : 0.5;
    }
    if (PERT) {
      if (cnt[q] > 0) zo2_raw4(P.rs_seed, ZO2_PERTURB_STREAM, P.base + idx[q], r);
#pragma unroll
      for (int j = 0; j < 4; ++j) u[q * PER + OFF + j] = j < cnt[q] ? zo2_u53(r[j]) : 0.5;
    }
  }
  warp_ndtri<NQ * PER>(u, z, sc);
  const double m2 = -2.0 * P.eps;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= cnt[q]) continue;
      A x = w[q][j];
      if (UPD) x = axpy1(x, P.ucoef, z[q * PER + j]);
      if (PERT) {
        const double zr = z[q * PER + OFF + j];
        wp[q][j] = axpy1(x, P.eps, zr);
        wm[q][j] = axpy1(wp[q][j], m2, zr);
        x = axpy1(wm[q][j], P.eps, zr);
      } else {
        wp[q][j] = wm[q][j] = x;
      }
      w[q][j] = x;
    }
  }
}

__device__ __forceinline__ void split_bf16(float x, __nv_bfloat16 &hi, __nv_bfloat16 &lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

template <typename A>
__device__ __forceinline__ void emit_linear(const zo2_segment_desc &sg, uint64_t li,
                                            const A wp[4], const A wm[4], int cnt) {
  // li: element index within the segment (same layout)
  switch (sg.out_kind) {
    case ZO2_OUT_F32:
      for (int j = 0; j < cnt; ++j) {
        ((float *)sg.out_plus)[li + j] = (float)wp[j];
        ((float *)sg.out_minus)[li + j] = (float)wm[j];
      }
      break;
    case ZO2_OUT_BF16:
      for (int j = 0; j < cnt; ++j) {
        ((__nv_bfloat16 *)sg.out_plus)[li + j] = __float2bfloat16_rn((float)wp[j]);
        ((__nv_bfloat16 *)sg.out_minus)[li + j] = __float2bfloat16_rn((float)wm[j]);
      }
      break;
    case ZO2_OUT_SPLIT:
      for (int j = 0; j < cnt; ++j) {
        __nv_bfloat16 h, l;
        split_bf16((float)wp[j], h, l);
        ((__nv_bfloat16 *)sg.out_plus)[li + j] = h;
        ((__nv_bfloat16 *)sg.out_plus_lo)[li + j] = l;
        split_bf16((float)wm[j], h, l);
        ((__nv_bfloat16 *)sg.out_minus)[li + j] = h;
        ((__nv_bfloat16 *)sg.out_minus_lo)[li + j] = l;
      }
      break;
    default:
      break;
  }
}

#ifndef ZO2_K2_TWO_PHASE
#define ZO2_K2_TWO_PHASE 0
#endif
#ifndef ZO2_K2_MINBLOCKS
#define ZO2_K2_MINBLOCKS 2
#endif
#define ZO2_MAX_SEGS 16
// quads (4 columns) per lane in the transposing K2: warp tile = 32 rows x 4*TQ cols
constexpr int TQ = 1;
struct SegTable {
  zo2_segment_desc s[ZO2_MAX_SEGS];
  uint64_t quad_start[ZO2_MAX_SEGS + 1];  // prefix of 4-element chunks (linear kernel)
  uint64_t tile_start[ZO2_MAX_SEGS + 1];  // prefix of 64x64 tiles (transpose kernel)
  int n;
};

// update: 0 = none, 1 = deferred update gated on g != 0 (PendingGradient.valid,
// zo2_engine.py:45-47), 2 = ungated (naive update-after-forward, :254-255).
__device__ __forceinline__ double resolve_ucoef(const double *d_g, double lr, int &upd) {
  if (!upd) return 0.0;
  const double g = *d_g;
  if (upd == 1 && g == 0.0) {
    upd = 0;
    return 0.0;
  }
  return -(lr * g);
}

// Linear (same-layout) segments: one thread = 4 consecutive elements; the loop
// advances whole warps so warp_ndtri always sees 32 converged lanes.
template <int FMT, bool UPD, bool PERT>
__device__ __forceinline__ void k2_linear_body(void *arena, const SegTable &T, const K2Params &P,
                                               unsigned &nn, unsigned &ns, uint8_t *raw) {
  typedef typename Wire<FMT>::A A;
  constexpr int PER = (UPD ? 4 : 0) + (PERT ? 4 : 0);
  ZgenScratch<PER> &sc = ((ZgenScratch<PER> *)raw)[threadIdx.x / 32];
  const uint64_t total = T.quad_start[T.n];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t qb = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); qb < total;
       qb += stride) {
    const uint64_t q = qb + (threadIdx.x & 31u);
    int si = 0;
    uint64_t li = 0, i = 0;
    int cnt[1] = {0};
    if (q < total) {
      while (q >= T.quad_start[si + 1]) ++si;
      const uint64_t seg_n = (uint64_t)T.s[si].rows * T.s[si].cols;
      li = (q - T.quad_start[si]) * 4;
      i = T.s[si].offset + li;
      cnt[0] = (int)min((uint64_t)4, seg_n - li);
    }
    A w[1][4], wp[1][4], wm[1][4];
    const uint64_t idx[1] = {i};
    const bool vec = cnt[0] == 4 && (i & 3) == 0;
    if (vec) Wire<FMT>::load4(arena, i, w[0]);
    else
      for (int j = 0; j < cnt[0]; ++j) w[0][j] = Wire<FMT>::load1(arena, i + j);
    k2_quads<A, 1, UPD, PERT>(w, wp, wm, idx, cnt, P, sc);
    if (cnt[0] == 0) continue;
    if (vec) Wire<FMT>::store4(arena, i, w[0], nn, ns);
    else
      for (int j = 0; j < cnt[0]; ++j) Wire<FMT>::store1(arena, i + j, w[0][j], nn, ns);
    if (PERT) emit_linear<A>(T.s[si], li, wp[0], wm[0], cnt[0]);
  }
}

template <int FMT>
__global__ void __launch_bounds__(256, ZO2_K2_MINBLOCKS) k_update_perturb_linear(
    void *arena, SegTable T, K2Params P, const double *d_g, double lr, uint64_t *counts) {
  int upd = P.do_update;
  P.ucoef = resolve_ucoef(d_g, lr, upd);
  unsigned nn = 0, ns = 0;
  __shared__ __align__(16) uint8_t raw[8 * sizeof(ZgenScratch<8>)];
  if (upd && P.do_perturb) k2_linear_body<FMT, true, true>(arena, T, P, nn, ns, raw);
  else if (upd) k2_linear_body<FMT, true, false>(arena, T, P, nn, ns, raw);
  else if (P.do_perturb) k2_linear_body<FMT, false, true>(arena, T, P, nn, ns, raw);
  if (FMT != ZO2_F32 && FMT != ZO2_F64) add_counts(counts, nn, ns);
}

// Transposed segments ([rows=K, cols=N] -> operand [N, K]), shared-memory
// free so it co-resides with the persistent GEMM on the same SMs (the GEMM
// keeps the tensor pipe busy, this kernel the FP64/INT pipes).  Warp tile =
// 32 rows x 8 cols: lane t owns row r0+t, cols c0..c0+7 (two Philox blocks
// per stream); for each column the warp writes operand row n = c0+j over
// K = r0..r0+31 as one coalesced 64-byte store.
template <int FMT, bool UPD, bool PERT>
__device__ __forceinline__ void k2_transpose_body(void *arena, const SegTable &T,
                                                  const K2Params &P, unsigned &nn, unsigned &ns,
                                                  uint8_t *raw) {
  typedef typename Wire<FMT>::A A;
  constexpr int PER = (UPD ? 4 : 0) + (PERT ? 4 : 0);
  ZgenScratch<TQ * PER> &sc = ((ZgenScratch<TQ * PER> *)raw)[threadIdx.x / 32];
  const int lane = threadIdx.x & 31;
  const uint64_t total = T.tile_start[T.n];
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x / 32);
  for (uint64_t t = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; t < total;
       t += nwarps) {  // warp-uniform: one tile per warp
    int si = 0;
    while (t >= T.tile_start[si + 1]) ++si;
    const zo2_segment_desc &sg = T.s[si];
    const uint32_t tiles_c = (sg.cols + 4 * TQ - 1) / (4 * TQ);
    const uint64_t lt = t - T.tile_start[si];
    const uint32_t r = (uint32_t)(lt / tiles_c) * 32 + lane, c0 = (uint32_t)(lt % tiles_c) * (4 * TQ);
    const bool split = sg.out_kind == ZO2_OUT_SPLIT_T;
    A w[TQ][4], wp[TQ][4], wm[TQ][4];
    uint64_t idx[TQ];
    int cnt[TQ];
    bool vec[TQ];
#pragma unroll
    for (int q = 0; q < TQ; ++q) {
      const uint32_t c = c0 + 4 * q;
      cnt[q] = (r < sg.rows && c < sg.cols) ? (int)min(4u, sg.cols - c) : 0;
      idx[q] = sg.offset + (uint64_t)r * sg.cols + c;
      vec[q] = cnt[q] == 4 && (idx[q] & 3) == 0;
      if (vec[q]) Wire<FMT>::load4(arena, idx[q], w[q]);
      else
        for (int j = 0; j < cnt[q]; ++j) w[q][j] = Wire<FMT>::load1(arena, idx[q] + j);
    }
    k2_quads<A, TQ, UPD, PERT>(w, wp, wm, idx, cnt, P, sc);
#pragma unroll
    for (int q = 0; q < TQ; ++q) {
      if (vec[q]) Wire<FMT>::store4(arena, idx[q], w[q], nn, ns);
      else
        for (int j = 0; j < cnt[q]; ++j) Wire<FMT>::store1(arena, idx[q] + j, w[q][j], nn, ns);
      if (!PERT) continue;
      const uint32_t c = c0 + 4 * q;
      for (int j = 0; j < cnt[q]; ++j) {
        const uint64_t o = (uint64_t)(c + j) * sg.rows + r;
        if (split) {
          __nv_bfloat16 h, l;
          split_bf16((float)wp[q][j], h, l);
          ((__nv_bfloat16 *)sg.out_plus)[o] = h;
          ((__nv_bfloat16 *)sg.out_plus_lo)[o] = l;
          split_bf16((float)wm[q][j], h, l);
          ((__nv_bfloat16 *)sg.out_minus)[o] = h;
          ((__nv_bfloat16 *)sg.out_minus_lo)[o] = l;
        } else {
          ((__nv_bfloat16 *)sg.out_plus)[o] = __float2bfloat16_rn((float)wp[q][j]);
          ((__nv_bfloat16 *)sg.out_minus)[o] = __float2bfloat16_rn((float)wm[q][j]);
        }
      }
    }
  }
}

template <int FMT>
__global__ void __launch_bounds__(256, ZO2_K2_MINBLOCKS) k_update_perturb_transpose(
    void *arena, SegTable T, K2Params P, const double *d_g, double lr, uint64_t *counts) {
  int upd = P.do_update;
  P.ucoef = resolve_ucoef(d_g, lr, upd);
  unsigned nn = 0, ns = 0;
  __shared__ __align__(16) uint8_t raw[8 * sizeof(ZgenScratch<TQ * 8>)];
  if (upd && P.do_perturb) k2_transpose_body<FMT, true, true>(arena, T, P, nn, ns, raw);
  else if (upd) k2_transpose_body<FMT, true, false>(arena, T, P, nn, ns, raw);
  else if (P.do_perturb) k2_transpose_body<FMT, false, true>(arena, T, P, nn, ns, raw);
  if (FMT != ZO2_F32 && FMT != ZO2_F64) add_counts(counts, nn, ns);
}

template <int FMT>
static int launch_k2(void *arena, const SegTable &lin, const SegTable &tr, const K2Params &P,
                     const double *d_g, double lr, uint64_t *counts, cudaStream_t s) {
  if (lin.n > 0 && lin.quad_start[lin.n] > 0) {
    // grid: multiple of 148 SMs, every thread a full loop trip
    const uint64_t q = lin.quad_start[lin.n];
    unsigned g = zo2_grid_for(q, 256, 148u * g_k2_ctas_per_sm);
    k_update_perturb_linear<FMT><<<g, 256, 0, s>>>(arena, lin, P, d_g, lr, counts);
    zo2_count_launch();
    ZO2_CHECK_LAUNCH();
  }
  if (tr.n > 0 && tr.tile_start[tr.n] > 0) {
    unsigned g = zo2_grid_for(tr.tile_start[tr.n], 8, 148u * g_k2_ctas_per_sm);
    k_update_perturb_transpose<FMT><<<g, 256, 0, s>>>(arena, tr, P, d_g, lr, counts);
    zo2_count_launch();
    ZO2_CHECK_LAUNCH();
  }
  return ZO2_OK;
}

extern "C" int zo2_update_perturb(void *arena, int wire_fmt, uint64_t n, uint64_t base,
                                  int update, const double *d_g, double lr,
                                  uint64_t lrs_seed, int perturb, double eps,
                                  uint64_t rs_seed, const zo2_segment_desc *segs,
                                  int n_segs, uint64_t *counts, void *cs) {
  if (n == 0) return ZO2_OK;
  if (!arena) return zo2_set_error(ZO2_E_ARG, "zo2_update_perturb: null arena");
  if (update && !d_g) return zo2_set_error(ZO2_E_ARG, "zo2_update_perturb: update needs d_g");
  if (n_segs < 1 || n_segs > ZO2_MAX_SEGS)
    return zo2_set_error(ZO2_E_ARG, "zo2_update_perturb: 1..16 segments required");
  SegTable lin, tr;
  memset(&lin, 0, sizeof(lin));
  memset(&tr, 0, sizeof(tr));
  uint64_t covered = 0;
  for (int k = 0; k < n_segs; ++k) {
    const zo2_segment_desc &sg = segs[k];
    const uint64_t sn = (uint64_t)sg.rows * sg.cols;
    if (sg.offset != covered)
      return zo2_set_error(ZO2_E_ARG, "zo2_update_perturb: segments must tile the bucket in order");
    covered += sn;
    const bool t = sg.out_kind == ZO2_OUT_BF16_T || sg.out_kind == ZO2_OUT_SPLIT_T;
    if (perturb && sg.out_kind != ZO2_OUT_NONE && (!sg.out_plus || !sg.out_minus))
      return zo2_set_error(ZO2_E_ARG, "zo2_update_perturb: operand outputs missing");
    if (perturb && (sg.out_kind == ZO2_OUT_SPLIT || sg.out_kind == ZO2_OUT_SPLIT_T) &&
        (!sg.out_plus_lo || !sg.out_minus_lo))
      return zo2_set_error(ZO2_E_ARG, "zo2_update_perturb: split lo planes missing");
    if (t && perturb) {
      tr.s[tr.n] = sg;
      tr.tile_start[tr.n + 1] =
          tr.tile_start[tr.n] + (uint64_t)((sg.rows + 31) / 32) * ((sg.cols + 4 * TQ - 1) / (4 * TQ));
      ++tr.n;
    } else {
      lin.s[lin.n] = sg;
      if (!perturb) lin.s[lin.n].out_kind = ZO2_OUT_NONE;
      lin.quad_start[lin.n + 1] = lin.quad_start[lin.n] + (sn + 3) / 4;
      ++lin.n;
    }
  }
  if (covered != n) return zo2_set_error(ZO2_E_ARG, "zo2_update_perturb: segments do not cover n");
  K2Params P;
  P.base = base;
  P.do_update = update;
  P.ucoef = 0.0;
  P.lrs_seed = lrs_seed;
  P.do_perturb = perturb;
  P.eps = eps;
  P.rs_seed = rs_seed;
  cudaStream_t s = S(cs);
  switch (wire_fmt) {
    case ZO2_F64: return launch_k2<ZO2_F64>(arena, lin, tr, P, d_g, lr, counts, s);
    case ZO2_F32: return launch_k2<ZO2_F32>(arena, lin, tr, P, d_g, lr, counts, s);
    case ZO2_BF16: return launch_k2<ZO2_BF16>(arena, lin, tr, P, d_g, lr, counts, s);
    case ZO2_F16: return launch_k2<ZO2_F16>(arena, lin, tr, P, d_g, lr, counts, s);
    case ZO2_F8E4M3: return launch_k2<ZO2_F8E4M3>(arena, lin, tr, P, d_g, lr, counts, s);
    default: return zo2_set_error(ZO2_E_ARG, "zo2_update_perturb: bad wire format");
  }
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
