// zo2_zapprox.cuh -- a cheap binary32 approximation of the reference's z with
// a verified error bound, for K2's certified path (zo2_k2.cu, K2c).
//
// The reference's z (numerics.py:171-182: Philox4x64-10, u = ((r>>11)+0.5)
// 2^-53, Cephes ndtri in IEEE double with glibc log) costs ~55 FP64 ops per
// draw plus the branch compaction K2 needs for ndtri's two branches.  But the
// kernel's OUTPUTS are narrow roundings of w + c z: the arena is re-encoded
// to bf16 / f16 / e4m3 (the AMP wire, runtime.py:145-199), the GEMM operands
// are bf16.  A z~ with |z~ - z| <= tau(z~) decides those roundings unless the
// pre-rounding value sits within a few f32 ulps of a rounding boundary of the
// output format (probability ~1e-3 per element at the model's weight scales),
// and then the kernel recomputes the element with the exact z.  The result
// is the reference's bits either way.
//
// z~ is a function of one float only: y = min(u, 1-u) rounded to binary32
// (from the 53-bit integer, one rounding) -> g(y) = -ndtri(y) >= 0 with
// M. Giles' single-precision erfinv polynomials ("Approximating the erfinv
// function", GPU Computing Gems Jade, 2011) over MUFU log2 / sqrt, signed by
// the side of 1/2 that u is on.  Because z~ depends on y alone and the exact
// z is monotone in the 53-bit integer, zo2_zapprox_bound_probe() checks the
// bound EXHAUSTIVELY: for every binary32 y in [2^-24, 1/2] it evaluates the
// exact z at both ends of the integer interval that rounds to y, on both
// sides of 1/2 (tests/test_gpu_kernels.py::test_zapprox_bound_exhaustive).
// y < 2^-24 (probability 2^-23) is outside Giles' range: always exact.
#pragma once
#include <stdint.h>

// tau(z~) = ZA_TAU_ABS + ZA_TAU_REL |z~|.  The probe is exhaustive, so the
// bound is proven for every input; the test still demands max |err| / tau
// <= 0.5 (measured 0.44 with these constants: 1.8e-6 worst absolute error).
#define ZA_TAU_ABS 7.0e-7f
#define ZA_TAU_REL 7.0e-7f
#define ZA_Y_MIN 0x1p-24f

__device__ __forceinline__ float za_lg2(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float za_sqrt(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// y of a raw draw: m = r >> 11 (numerics.py:181), upper = u > 1/2,
// y53 = upper ? 2^53 - 1 - m : m, y = fl32((2 y53 + 1) 2^-54) (exact scaling).
// 2 y53 + 1 = ((upper ? ~r : r) >> 10) | 1 (upper = bit 63 of r).
__device__ __forceinline__ float za_y(uint64_t r, bool &upper) {
  upper = (int64_t)r < 0;
  const uint64_t f = r ^ (uint64_t)((int64_t)r >> 63);
  return __fmul_rn(__ull2float_rn((f >> 10) | 1ull), 0x1p-54f);
}

// Giles' two polynomials: central in w - 2.5 (w < 5), tail in sqrt(w) - 3.
__device__ __forceinline__ float za_central(float w) {
  float p = 2.81022636e-08f;
  p = __fmaf_rn(p, w, 3.43273939e-07f);
  p = __fmaf_rn(p, w, -3.5233877e-06f);
  p = __fmaf_rn(p, w, -4.39150654e-06f);
  p = __fmaf_rn(p, w, 0.00021858087f);
  p = __fmaf_rn(p, w, -0.00125372503f);
  p = __fmaf_rn(p, w, -0.00417768164f);
  p = __fmaf_rn(p, w, 0.246640727f);
  return __fmaf_rn(p, w, 1.50140941f);
}
__device__ __forceinline__ float za_tailp(float w) {
  float p = -0.000200214257f;
  p = __fmaf_rn(p, w, 0.000100950558f);
  p = __fmaf_rn(p, w, 0.00134934322f);
  p = __fmaf_rn(p, w, -0.00367342844f);
  p = __fmaf_rn(p, w, 0.00573950773f);
  p = __fmaf_rn(p, w, -0.0076224613f);
  p = __fmaf_rn(p, w, 0.00943887047f);
  p = __fmaf_rn(p, w, 1.00167406f);
  return __fmaf_rn(p, w, 2.83297682f);
}

// g(y) = -ndtri(y) for y in [2^-24, 1/2]; every operation explicit (no
// contraction choices left to the compiler), so the probe and K2 evaluate
// the same operations (K2's za_z4 is this function unrolled over 4 draws).
__device__ __forceinline__ float za_g(float y) {
  const float x = __fmaf_rn(-2.0f, y, 1.0f);                    // 1 - 2y
  const float a = __fmul_rn(__fmul_rn(4.0f, y), __fsub_rn(1.0f, y));
  const float w = __fmul_rn(za_lg2(a), -0.69314718056f);       // -log(4y(1-y))
  const float p = w < 5.0f ? za_central(__fsub_rn(w, 2.5f))
                           : za_tailp(__fsub_rn(za_sqrt(w), 3.0f));
  return __fmul_rn(1.41421356237f, __fmul_rn(p, x));
}

// z~ of a raw draw and its bound; tau = +inf where the approximation is not
// used (y < 2^-24, which includes u == 1.0 -> z = +inf).
__device__ __forceinline__ float za_z(uint64_t r, float &tau) {
  bool upper;
  const float y = za_y(r, upper);
  if (!(y >= ZA_Y_MIN)) {
    tau = __int_as_float(0x7f800000);
    return 0.0f;
  }
  const float g = za_g(y);
  tau = __fmaf_rn(ZA_TAU_REL, g, ZA_TAU_ABS);
  return upper ? g : -g;
}
