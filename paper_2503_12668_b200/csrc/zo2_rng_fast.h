/*
 * zo2_rng_fast.h -- the "fast" Gaussian direction z (rng = "fast"), shared by
 * host C++ and sm_100a device code.
 *
 * The reference-exact z (zo2_rng.h: numpy Philox4x64-10 + Cephes ndtri in
 * IEEE double, numerics.py:161-182) costs ~200 instructions per draw and
 * dominates the fused update/perturb kernel.  This is the north star's
 * "counter-based Philox stream keyed on (seed, param offset)" at GPU cost
 * (~45 instructions per draw):
 *
 *   block b = pos / 4 of (seed, stream):  Philox4x32-10 with key
 *     (lo32 seed, hi32 seed) and counter (lo32 b, hi32 b, lo32 stream,
 *     hi32 stream); lane pos % 4 of the output.
 *   u = ((r >> 9) + 1/2) * 2^-23 in (0, 1), exact in binary32.
 *   z = sqrt(2) * erfinv(2u - 1) with M. Giles' single-precision erfinv
 *     ("Approximating the erfinv function", GPU Computing Gems, 2011),
 *     w = -log(4u(1-u)) from an exponent split + atanh series.
 *
 * Every operation is a single correctly rounded IEEE binary32 add / mul /
 * div / sqrt in a fixed order (no FMA contraction: device code uses the
 * __f*_rn intrinsics, the host build uses -ffp-contract=off), so the CPU
 * restatement (oracle/zo2_oracle.py fast_gauss) reproduces it bit for bit.
 * Same (seed, stream, position) -> same z in every kernel (update, perturb,
 * restore, embedding), which is all ZO-SGD needs: E[z] = 0, E[z z^T] = I.
 */
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define ZO2F_HD __host__ __device__ __forceinline__
#else
#define ZO2F_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define ZO2F_MUL(a, b) __fmul_rn((a), (b))
#define ZO2F_ADD(a, b) __fadd_rn((a), (b))
#define ZO2F_SUB(a, b) __fsub_rn((a), (b))
#define ZO2F_DIV(a, b) __fdiv_rn((a), (b))
#define ZO2F_SQRT(a) __fsqrt_rn((a))
#else
#include <math.h>
#define ZO2F_MUL(a, b) ((float)((a) * (b)))
#define ZO2F_ADD(a, b) ((float)((a) + (b)))
#define ZO2F_SUB(a, b) ((float)((a) - (b)))
#define ZO2F_DIV(a, b) ((float)((a) / (b)))
#define ZO2F_SQRT(a) sqrtf((a))
#endif

ZO2F_HD uint32_t zo2f_as_u32(float x) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(x);
#else
  union { float f; uint32_t u; } c; c.f = x; return c.u;
#endif
}
ZO2F_HD float zo2f_as_f32(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  union { float f; uint32_t u; } c; c.u = u; return c.f;
#endif
}

ZO2F_HD void zo2f_mulhilo32(uint32_t a, uint32_t b, uint32_t *hi, uint32_t *lo) {
#if defined(__CUDA_ARCH__)
  /* one IMAD.WIDE.U32; the 64-bit C form left an add of zero per multiply */
  uint64_t p;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
#else
  const uint64_t p = (uint64_t)a * b;
#endif
  *hi = (uint32_t)(p >> 32);
  *lo = (uint32_t)p;
}

/* Philox4x32-10 of counter (b, stream) under key seed. */
ZO2F_HD void zo2f_philox(uint64_t seed, uint64_t stream, uint64_t b, uint32_t out[4]) {
  uint32_t c0 = (uint32_t)b, c1 = (uint32_t)(b >> 32), c2 = (uint32_t)stream,
           c3 = (uint32_t)(stream >> 32);
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    zo2f_mulhilo32(0xD2511F53u, c0, &hi0, &lo0);
    zo2f_mulhilo32(0xCD9E8D57u, c2, &hi1, &lo1);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* natural log of a in (0, 1]: a = m 2^e with m in [sqrt(1/2), sqrt(2)),
 * log m = 2 atanh(s), s = (m - 1) / (m + 1), |s| < 0.1716 (odd series to s^9). */
ZO2F_HD float zo2f_log(float a) {
  uint32_t ia = zo2f_as_u32(a);
  int e = (int)((ia >> 23) & 0xFF) - 127;
  uint32_t im = (ia & 0x007FFFFFu) | 0x3F800000u; /* m in [1, 2) */
  if (im > 0x3FB504F3u) { /* m > sqrt(2): use m / 2 */
    im -= 0x00800000u;
    e += 1;
  }
  const float m = zo2f_as_f32(im);
  const float s = ZO2F_DIV(ZO2F_SUB(m, 1.0f), ZO2F_ADD(m, 1.0f));
  const float s2 = ZO2F_MUL(s, s);
  float p = 0.11111111f;                              /* 1/9 */
  p = ZO2F_ADD(ZO2F_MUL(p, s2), 0.14285715f);         /* 1/7 */
  p = ZO2F_ADD(ZO2F_MUL(p, s2), 0.2f);                /* 1/5 */
  p = ZO2F_ADD(ZO2F_MUL(p, s2), 0.33333334f);         /* 1/3 */
  p = ZO2F_ADD(ZO2F_MUL(p, s2), 1.0f);
  const float lm = ZO2F_MUL(ZO2F_MUL(2.0f, s), p);
  return ZO2F_ADD(ZO2F_MUL((float)e, 0.6931472f), lm);
}

/* z from one raw 32-bit draw. */
ZO2F_HD float zo2f_gauss(uint32_t r) {
  const float u = ZO2F_MUL(ZO2F_ADD((float)(r >> 9), 0.5f), 1.1920929e-07f); /* 2^-23: exact, u < 1 */
  const float x = ZO2F_SUB(ZO2F_MUL(2.0f, u), 1.0f);                        /* exact */
  const float a = ZO2F_MUL(ZO2F_MUL(4.0f, u), ZO2F_SUB(1.0f, u));
  float w = ZO2F_SUB(0.0f, zo2f_log(a));
  float p;
  if (w < 5.0f) {
    w = ZO2F_SUB(w, 2.5f);
    p = 2.81022636e-08f;
    p = ZO2F_ADD(3.43273939e-07f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(-3.5233877e-06f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(-4.39150654e-06f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(0.00021858087f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(-0.00125372503f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(-0.00417768164f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(0.246640727f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(1.50140941f, ZO2F_MUL(p, w));
  } else {
    w = ZO2F_SUB(ZO2F_SQRT(w), 3.0f);
    p = -0.000200214257f;
    p = ZO2F_ADD(0.000100950558f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(0.00134934322f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(-0.00367342844f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(0.00573950773f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(-0.0076224613f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(0.00943887047f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(1.00167406f, ZO2F_MUL(p, w));
    p = ZO2F_ADD(2.83297682f, ZO2F_MUL(p, w));
  }
  return ZO2F_MUL(1.4142135f, ZO2F_MUL(p, x));
}

/* z at absolute position pos of (seed, stream). */
ZO2F_HD float zo2f_gauss_at(uint64_t seed, uint64_t stream, uint64_t pos) {
  uint32_t r[4];
  zo2f_philox(seed, stream, pos >> 2, r);
  return zo2f_gauss(r[pos & 3]);
}
