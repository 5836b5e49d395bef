// zo2_wire.cuh -- wire-format codecs (numerics.py:204-311) and arena access
// for the element-wise kernels; shared by zo2_elementwise.cu and zo2_k2.cu.
#pragma once
#include "zo2_common.cuh"
#include <math.h>

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

