/*
 * zo2_oracle.c -- TEST INFRASTRUCTURE ONLY (CPU parity oracle).
 *
 * Plain-C restatement of the reference's element-wise arithmetic on the ZO2
 * hot path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library; the product
 * (paper_2503_12668_b200) never does.
 *
 * What it restates (reference = /root/reference/pkg/src/zo2lab):
 *   - raw_uint64            numerics.py:161-168   numpy Philox4x64-10, key =
 *                           (stream<<64)|seed, position p -> counter block
 *                           p//4 (numpy pre-increments: block+1), lane p%4.
 *                           Third-party algorithm: numpy 2.3.5
 *                           numpy.random.Philox (Random123 Philox4x64-10).
 *   - gaussian_fill         numerics.py:171-182   u = ((r>>11)+0.5)*2^-53,
 *                           z = ndtri(u).  Third-party algorithm: scipy 1.18.1
 *                           scipy.special.ndtri (Cephes ndtri), restated in
 *                           plain IEEE double with no FMA contraction
 *                           (compile with -ffp-contract=off).
 *   - derive_step_seed      numerics.py:185-190   splitmix64 finaliser.
 *   - axpy                  model.py:227-233      flat += coef*z with an f64
 *                           product, f64 sum, one final rounding to storage.
 *   - codecs                numerics.py:204-311   bf16 / f16 / e4m3 encode
 *                           (RNE, saturation, NaN tallies) and exact decode.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- Philox */
static const uint64_t PHILOX_M0 = 0xD2E7470EE14C6C93ULL;
static const uint64_t PHILOX_M1 = 0xCA5A826395121157ULL;
static const uint64_t PHILOX_W0 = 0x9E3779B97F4A7C15ULL;
static const uint64_t PHILOX_W1 = 0xBB67AE8584CAA73BULL;

/* One Philox4x64-10 block: ctr (4 words, little-endian 256-bit) + key (2). */
static void philox_block(const uint64_t ctr_in[4], uint64_t k0, uint64_t k1,
                         uint64_t out[4]) {
  uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  for (int r = 0; r < 10; ++r) {
    u128 p0 = (u128)PHILOX_M0 * c0;
    u128 p1 = (u128)PHILOX_M1 * c2;
    uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += PHILOX_W0;
    k1 += PHILOX_W1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Draw at absolute position p of the (seed, stream) sequence. numpy's
 * Philox(counter=b) increments the 256-bit counter before each block, so
 * position p uses counter value (p/4 + 1) as a 256-bit integer. */
static void philox_at_block(uint64_t blk, uint64_t seed, uint64_t stream,
                            uint64_t out[4]) {
  uint64_t ctr[4] = {blk + 1, 0, 0, 0};
  if (ctr[0] == 0) ctr[1] = 1; /* carry (blk == 2^64-1) */
  philox_block(ctr, seed, stream, out);
}

void oracle_raw_u64(uint64_t seed, uint64_t stream, uint64_t counter,
                    uint64_t n, uint64_t *out) {
  uint64_t blk = counter >> 2, lane = counter & 3, buf[4];
  philox_at_block(blk, seed, stream, buf);
  for (uint64_t i = 0; i < n; ++i) {
    out[i] = buf[lane];
    if (++lane == 4) {
      lane = 0;
      ++blk;
      if (i + 1 < n) philox_at_block(blk, seed, stream, buf);
    }
  }
}

/* ------------------------------------------------------- Cephes ndtri */
static const double S2PI = 2.50662827463100050242E0;
static const double EXPM2 = 0.13533528323661269189; /* exp(-2) */
static const double P0[5] = {
    -5.99633501014107895267E1, 9.80010754185999661536E1,
    -5.66762857469070293439E1, 1.39312609387279679503E1,
    -1.23916583867381258016E0};
static const double Q0[8] = {
    1.95448858338141759834E0,  4.67627912898881538453E0,
    8.63602421390890590575E1,  -2.25462687854119370527E2,
    2.00260212380060660359E2,  -8.20372256168333339912E1,
    1.59056225126211695515E1,  -1.18331621121330003142E0};
static const double P1[9] = {
    4.05544892305962419923E0,   3.15251094599893866154E1,
    5.71628192246421288162E1,   4.40805073893200834700E1,
    1.46849561928858024014E1,   2.18663306850790267539E0,
    -1.40256079171354495875E-1, -3.50424626827848203418E-2,
    -8.57456785154685413611E-4};
static const double Q1[8] = {
    1.57799883256466749731E1,   4.53907635128879210584E1,
    4.13172038254672030440E1,   1.50425385692907503408E1,
    2.50464946208309415979E0,   -1.42182922854787788574E-1,
    -3.80806407691578277194E-2, -9.33259480895457427372E-4};
static const double P2[9] = {
    3.23774891776946035970E0,  6.91522889068984211695E0,
    3.93881025292474443415E0,  1.33303460815807542389E0,
    2.01485389549179081538E-1, 1.23716634817820021358E-2,
    3.01581553508235416007E-4, 2.65806974686737550832E-6,
    6.23974539184983293730E-9};
static const double Q2[8] = {
    6.02427039364742014255E0,  3.67983563856160859403E0,
    1.37702099489081330271E0,  2.16236993594496635890E-1,
    1.34204006088543189037E-2, 3.28014464682127739104E-4,
    2.89247864745380683936E-6, 6.79019408009981274425E-9};

static double polevl(double x, const double *c, int n) {
  double a = c[0];
  for (int i = 1; i <= n; ++i) a = a * x + c[i];
  return a;
}
static double p1evl(double x, const double *c, int n) {
  double a = x + c[0];
  for (int i = 1; i < n; ++i) a = a * x + c[i];
  return a;
}

double oracle_ndtri(double y0) {
  if (y0 == 0.0) return -INFINITY;
  if (y0 == 1.0) return INFINITY;
  if (y0 < 0.0 || y0 > 1.0) return NAN;
  int code = 1;
  double y = y0;
  if (y > 1.0 - EXPM2) {
    y = 1.0 - y;
    code = 0;
  }
  if (y > EXPM2) {
    y = y - 0.5;
    double y2 = y * y;
    double x = y + y * (y2 * polevl(y2, P0, 4) / p1evl(y2, Q0, 8));
    return x * S2PI;
  }
  double x = sqrt(-2.0 * log(y));
  double x0 = x - log(x) / x;
  double z = 1.0 / x;
  double x1;
  if (x < 8.0)
    x1 = z * polevl(z, P1, 8) / p1evl(z, Q1, 8);
  else
    x1 = z * polevl(z, P2, 8) / p1evl(z, Q2, 8);
  x = x0 - x1;
  if (code != 0) x = -x;
  return x;
}

static double u53(uint64_t r) {
  return ((double)(r >> 11) + 0.5) * 0x1p-53;
}

void oracle_gaussian_fill(uint64_t seed, uint64_t stream, uint64_t counter,
                          uint64_t n, double *out) {
  uint64_t blk = counter >> 2, lane = counter & 3, buf[4];
  philox_at_block(blk, seed, stream, buf);
  for (uint64_t i = 0; i < n; ++i) {
    out[i] = oracle_ndtri(u53(buf[lane]));
    if (++lane == 4) {
      lane = 0;
      ++blk;
      if (i + 1 < n) philox_at_block(blk, seed, stream, buf);
    }
  }
}

/* z at arbitrary stream positions counter + idx[i] (sampled checks of
 * whole-block kernels; same Philox block + lane + ndtri as the fill). */
void oracle_gauss_at(uint64_t seed, uint64_t stream, uint64_t counter,
                     const uint64_t *idx, uint64_t n, double *out) {
  uint64_t buf[4];
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t pos = counter + idx[i];
    philox_at_block(pos >> 2, seed, stream, buf);
    out[i] = oracle_ndtri(u53(buf[pos & 3]));
  }
}

uint64_t oracle_derive_step_seed(uint64_t base, uint64_t j) {
  uint64_t x = base ^ (j * 0x9E3779B97F4A7C15ULL);
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

/* axpy with regenerated z: flat[i] = store(f64(flat[i]) + coef*z[i]). */
void oracle_axpy_z_f32(float *flat, uint64_t n, double coef, uint64_t seed,
                       uint64_t stream, uint64_t counter) {
  uint64_t blk = counter >> 2, lane = counter & 3, buf[4];
  philox_at_block(blk, seed, stream, buf);
  for (uint64_t i = 0; i < n; ++i) {
    double z = oracle_ndtri(u53(buf[lane]));
    double t = coef * z;
    flat[i] = (float)((double)flat[i] + t);
    if (++lane == 4) {
      lane = 0;
      ++blk;
      if (i + 1 < n) philox_at_block(blk, seed, stream, buf);
    }
  }
}

void oracle_axpy_z_f64(double *flat, uint64_t n, double coef, uint64_t seed,
                       uint64_t stream, uint64_t counter) {
  uint64_t blk = counter >> 2, lane = counter & 3, buf[4];
  philox_at_block(blk, seed, stream, buf);
  for (uint64_t i = 0; i < n; ++i) {
    double z = oracle_ndtri(u53(buf[lane]));
    double t = coef * z;
    flat[i] = flat[i] + t;
    if (++lane == 4) {
      lane = 0;
      ++blk;
      if (i + 1 < n) philox_at_block(blk, seed, stream, buf);
    }
  }
}

/* ---------------------------------------------------------------- codecs */
static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* bf16 (numerics.py:232-245): RNE by u + 0x7FFF + lsb, saturate exp=0xFF
 * results to 0x7F7F, NaN -> sign|0x7FC0. */
void oracle_encode_bf16(const float *x, uint64_t n, uint16_t *out,
                        uint64_t *nan_count, uint64_t *sat_count) {
  uint64_t nn = 0, ns = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t u = f2u(x[i]);
    uint16_t r = (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
    uint16_t sign = r & 0x8000u;
    int isnan_ = isnan(x[i]);
    if (isnan_) {
      r = sign | 0x7FC0u;
      ++nn;
    } else if ((r & 0x7FFFu) >= 0x7F80u) {
      r = sign | 0x7F7Fu;
      ++ns;
    }
    out[i] = r;
  }
  if (nan_count) *nan_count += nn;
  if (sat_count) *sat_count += ns;
}

void oracle_decode_bf16(const uint16_t *x, uint64_t n, float *out) {
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t u = (uint32_t)x[i] << 16;
    memcpy(&out[i], &u, 4);
  }
}

/* f16 (numerics.py:220-229): IEEE RNE cast, finite overflow -> +-65504. */
void oracle_encode_f16(const float *x, uint64_t n, uint16_t *out,
                       uint64_t *nan_count, uint64_t *sat_count) {
  uint64_t nn = 0, ns = 0;
  for (uint64_t i = 0; i < n; ++i) {
    _Float16 h = (_Float16)x[i];
    uint16_t b;
    memcpy(&b, &h, 2);
    if (isnan(x[i])) ++nn;
    else if (isinf((float)h) && isfinite(x[i])) {
      b = (uint16_t)((b & 0x8000u) | 0x7BFFu);
      ++ns;
    }
    out[i] = b;
  }
  if (nan_count) *nan_count += nn;
  if (sat_count) *sat_count += ns;
}

void oracle_decode_f16(const uint16_t *x, uint64_t n, float *out) {
  for (uint64_t i = 0; i < n; ++i) {
    _Float16 h;
    memcpy(&h, &x[i], 2);
    out[i] = (float)h;
  }
}

/* e4m3 (numerics.py:248-270): saturate at 448, binade exponent clamped at
 * -6, mantissa step 2^(e-3), rint ties-to-even, roll-over bumps the binade,
 * NaN -> 0x7F, sign bit from the source (also for NaN / -0). */
void oracle_encode_e4m3(const float *x, uint64_t n, uint8_t *out,
                        uint64_t *nan_count, uint64_t *sat_count) {
  uint64_t nn = 0, ns = 0;
  for (uint64_t i = 0; i < n; ++i) {
    double v = (double)x[i];
    int nan_ = isnan(v);
    int neg = signbit(v) ? 1 : 0;
    double mag = nan_ ? 0.0 : fabs(v);
    if (mag > 448.0) { ++ns; mag = 448.0; }
    int ex;
    (void)frexp(mag, &ex);
    int e = ex - 1;
    if (e < -6) e = -6;
    double step = ldexp(1.0, e - 3);
    double q = nearbyint(mag / step);
    if (q >= 16.0) { e += 1; q = 8.0; }
    long qi = (long)q;
    uint8_t code = (qi >= 8) ? (uint8_t)(((e + 7) << 3) + (qi - 8)) : (uint8_t)qi;
    if (nan_) { code = 0x7F; ++nn; }
    if (neg) code |= 0x80;
    out[i] = code;
  }
  if (nan_count) *nan_count += nn;
  if (sat_count) *sat_count += ns;
}

void oracle_decode_e4m3(const uint8_t *x, uint64_t n, float *out) {
  for (uint64_t i = 0; i < n; ++i) {
    uint8_t c = x[i];
    int expf_ = (c >> 3) & 0xF;
    double mant = (double)(c & 7);
    double v = (expf_ == 0) ? ldexp(mant, -9) : ldexp(8.0 + mant, expf_ - 10);
    if (expf_ == 15 && (c & 7) == 7) v = NAN;
    if (c >= 0x80) v = -v;
    out[i] = (float)v;
  }
}
