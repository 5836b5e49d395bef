// zo2_k2.cu -- K2: fused deferred ZO-SGD update + SPSA perturbation of one
// module bucket, emitting the W+eps z / W-eps z GEMM operands (sm_100a).
//
// Reference arithmetic (bit-exact): zo2_engine.py:183-204 dual_forward,
// _update_flat :168-174, _perturb :161-166, model.py:227-233 axpy, with z from
// numerics.py:161-182 (Philox4x64-10 + Cephes ndtri).  Per element:
//   w  = st(w + (-(lr g)) z(lrs))                       (deferred update)
//   w+ = st(w + eps z(rs)); w- = st(w+ - 2eps z(rs)); w = st(w- + eps z(rs))
//
// Design (why it looks like this).  The kernel is bound by issue slots of
// the exact Gaussian transform, not by HBM: ~60 FP64 + ~45 integer
// instructions per draw, two draws per parameter.  Evaluated per lane, a
// warp executes both Cephes branches (central 73% / tail 27% of draws) for
// every draw slot.  Here one CTA processes a 1024-element tile in four
// phases, with all draws of the tile staged in shared memory:
//   P1  load mapping: vector load of 4 weights per thread into a shared W
//       tile; Philox blocks of both streams; each draw is classified and its
//       slot pushed on a CTA-wide queue -- tail draws at the front, central
//       draws at the back (warp-scanned offsets, one shared atomic per warp).
//   P2  every warp takes 32 consecutive queue entries at a time: tail
//       entries first, then central ones, so exactly one warp-chunk per tile
//       mixes the two branches; nothing else diverges.
//   P3  apply mapping (transposed for [K, N] weight segments, so the operand
//       rows [N, K] are written as 8-byte-per-lane coalesced runs): update +
//       perturb/restore chain from the staged z, outputs written, restored
//       weights back into the W tile.
//   P4  load mapping again: restored (re-encoded) weights to the arena.
// The division / square root / Philox building blocks come from
// zo2_zexact.cuh (same IEEE results, fewer instructions).
#include "zo2_common.cuh"
#include "zo2_wire.cuh"
#include "zo2_zexact.cuh"
#include "zo2_rng_fast.h"
#include "zo2_zapprox.cuh"
#include <string.h>

void zo2_count_launch(uint64_t n = 1);

namespace {

constexpr int NT = 256;          // threads per CTA
constexpr int TE = 1024;         // elements per tile (32 x 32, or 1024 linear)
constexpr int NSLOT = 8 * NT;    // draw slots per tile (update 4 + perturb 4 per thread)
constexpr int WPITCH = 33;       // W tile row pitch (conflict-free transposed reads)
constexpr int MAX_SEGS = 16;
#ifndef ZO2_K2_CENTRAL_X2
#define ZO2_K2_CENTRAL_X2 1
#endif
#ifndef ZO2_K2_TAIL_X2
#define ZO2_K2_TAIL_X2 1
#endif
#ifndef ZO2_K2_MINB
#define ZO2_K2_MINB 4  // 64 registers (a few spills in cold paths): 4 CTAs (32 warps) per SM
#endif

// 0 = grid from occupancy; n = at most n CTAs per SM (leave room for a
// concurrently running persistent GEMM)
unsigned g_k2_ctas_per_sm = 0;
// z generator: 0 = reference-exact (Philox4x64-10 + Cephes ndtri), 1 = fast
// (Philox4x32-10 + binary32 erfinv, zo2_rng_fast.h)
int g_rng_mode = 0;

struct K2Table {
  zo2_segment_desc s[MAX_SEGS];
  uint64_t tile_start[MAX_SEGS + 1];
  uint32_t tiles_c[MAX_SEGS];   // column tiles (transposed segments)
  uint8_t transposed[MAX_SEGS];
  int n;
  int any_transposed;
  // K2c warp tiles: 32 rows x 4 columns (transposed) or 128 linear elements
  uint64_t wt_start[MAX_SEGS + 1];
  uint32_t wt_c[MAX_SEGS];      // 4-column groups per row band (transposed)
};

struct K2Params {
  uint64_t base;  // module RNG offset
  int do_update;  // 0 none, 1 deferred (gated on g != 0), 2 ungated (naive)
  double ucoef;   // -(lr * g), resolved on device
  uint64_t lrs_seed;
  int do_perturb;
  double eps;
  uint64_t rs_seed;
};

template <typename A>
struct K2Smem {
  double z[NSLOT];                  // y (reflected uniform) in P1, z after P2
  double logtab[256];               // glibc log (invc, logc) table
  double ccoef[13];                 // central-branch coefficients
  double tcoef[42];                 // tail-branch coefficients (ZX_TAIL_C)
  A w[2][32 * WPITCH];              // weight tile, double-buffered across tiles
  uint16_t q[NSLOT];                // tail slots from the front, central from the back
  unsigned counts[2];               // packed (n_tail | n_central << 16), per buffer
};

// Swizzled z index of draw k of load-thread t: k*256 + 32a + (b ^ (a | (k&1)<<3))
// with t = 32a + b.  Load-mapping accesses (fixed k, t = 32a + lane) and the
// transposed apply mapping both hit every 8-byte bank pair exactly twice.
__device__ __forceinline__ int zslot(int k, int t) {
  const int a = t >> 5, b = t & 31;
  return k * NT + (a << 5) + (b ^ (a | ((k & 1) << 3)));
}


// bf16 pair (a in the low half), one cvt.rn.bf16x2.f32
__device__ __forceinline__ uint32_t bf16x2(float a, float b) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t *>(&v);
}
// hi = bf16(x), lo = bf16(x - f32(hi)) for a pair, as split_bf16
__device__ __forceinline__ void split_bf16x2(float a, float b, uint32_t &hi, uint32_t &lo) {
  hi = bf16x2(a, b);
  lo = bf16x2(a - __uint_as_float(hi << 16), b - __uint_as_float(hi & 0xFFFF0000u));
}

// Element chain without the per-op NaN checks (finite weights and z); the
// caller re-runs axpy1's exact NaN semantics when an input is not finite.
template <bool UPD, bool PERT>
__device__ __forceinline__ void chain_fast(float &w, float &wp, float &wm, double uc, double zu,
                                           double eps, double zp) {
  double x = (double)w;
  if (UPD) x = (double)__double2float_rn(__dadd_rn(x, __dmul_rn(uc, zu)));
  if (PERT) {
    const double ez = __dmul_rn(eps, zp);  // (-2 eps) z == -2 (eps z) exactly
    const float p = __double2float_rn(__dadd_rn(x, ez));
    const float m = __double2float_rn(__fma_rn(-2.0, ez, (double)p));
    wp = p;
    wm = m;
    w = __double2float_rn(__dadd_rn((double)m, ez));
  } else {
    w = (float)x;
    wp = wm = w;
  }
}
template <bool UPD, bool PERT>
__device__ __forceinline__ void chain_fast(double &w, double &wp, double &wm, double uc, double zu,
                                           double eps, double zp) {
  double x = w;
  if (UPD) x = __dadd_rn(x, __dmul_rn(uc, zu));
  if (PERT) {
    const double ez = __dmul_rn(eps, zp);
    wp = __dadd_rn(x, ez);
    wm = __fma_rn(-2.0, ez, wp);
    w = __dadd_rn(wm, ez);
  } else {
    w = x;
    wp = wm = x;
  }
}
template <typename A>
struct Chain3 {
  A w, wp, wm;
};
template <bool UPD, bool PERT, typename A>
__device__ __noinline__ Chain3<A> chain_exact(A w, double uc, double zu, double eps, double zp) {
  Chain3<A> c;
  A x = w;
  if (UPD) x = axpy1(x, uc, zu);
  if (PERT) {
    c.wp = axpy1(x, eps, zp);
    c.wm = axpy1(c.wp, -2.0 * eps, zp);
    x = axpy1(c.wm, eps, zp);
  } else {
    c.wp = c.wm = x;
  }
  c.w = x;
  return c;
}

// Operand stores for 4 consecutive output elements starting at o (same kind
// for the transposed and the linear layouts: the index already points into
// the operand).
template <typename A>
__device__ __forceinline__ void emit4(const zo2_segment_desc &sg, int kind, uint64_t o,
                                      const A (&wp)[4], const A (&wm)[4], int cnt) {
  if (kind == ZO2_OUT_F32) {
    if (cnt == 4 && (o & 3) == 0) {
      *(float4 *)((float *)sg.out_plus + o) =
          make_float4((float)wp[0], (float)wp[1], (float)wp[2], (float)wp[3]);
      *(float4 *)((float *)sg.out_minus + o) =
          make_float4((float)wm[0], (float)wm[1], (float)wm[2], (float)wm[3]);
    } else {
      for (int j = 0; j < cnt; ++j) {
        ((float *)sg.out_plus)[o + j] = (float)wp[j];
        ((float *)sg.out_minus)[o + j] = (float)wm[j];
      }
    }
  } else if (kind == ZO2_OUT_BF16 || kind == ZO2_OUT_BF16_T) {
    // one cvt.rn.bf16x2.f32 per pair (same bits as two __float2bfloat16_rn)
    const uint32_t p01 = bf16x2((float)wp[0], (float)wp[1]), p23 = bf16x2((float)wp[2], (float)wp[3]);
    const uint32_t m01 = bf16x2((float)wm[0], (float)wm[1]), m23 = bf16x2((float)wm[2], (float)wm[3]);
    if (cnt == 4 && (o & 3) == 0) {
      *(uint2 *)((__nv_bfloat16 *)sg.out_plus + o) = make_uint2(p01, p23);
      *(uint2 *)((__nv_bfloat16 *)sg.out_minus + o) = make_uint2(m01, m23);
    } else {
      const uint32_t pv[2] = {p01, p23}, mv[2] = {m01, m23};
      for (int j = 0; j < cnt; ++j) {
        ((uint16_t *)sg.out_plus)[o + j] = (uint16_t)(pv[j >> 1] >> (16 * (j & 1)));
        ((uint16_t *)sg.out_minus)[o + j] = (uint16_t)(mv[j >> 1] >> (16 * (j & 1)));
      }
    }
  } else if (kind == ZO2_OUT_SPLIT || kind == ZO2_OUT_SPLIT_T) {
    uint32_t ph[2], pl[2], mh[2], ml[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      split_bf16x2((float)wp[2 * j], (float)wp[2 * j + 1], ph[j], pl[j]);
      split_bf16x2((float)wm[2 * j], (float)wm[2 * j + 1], mh[j], ml[j]);
    }
    if (cnt == 4 && (o & 3) == 0) {
      *(uint2 *)((__nv_bfloat16 *)sg.out_plus + o) = make_uint2(ph[0], ph[1]);
      *(uint2 *)((__nv_bfloat16 *)sg.out_plus_lo + o) = make_uint2(pl[0], pl[1]);
      *(uint2 *)((__nv_bfloat16 *)sg.out_minus + o) = make_uint2(mh[0], mh[1]);
      *(uint2 *)((__nv_bfloat16 *)sg.out_minus_lo + o) = make_uint2(ml[0], ml[1]);
    } else {
      for (int j = 0; j < cnt; ++j) {
        const int w = j >> 1, sh = 16 * (j & 1);
        ((uint16_t *)sg.out_plus)[o + j] = (uint16_t)(ph[w] >> sh);
        ((uint16_t *)sg.out_plus_lo)[o + j] = (uint16_t)(pl[w] >> sh);
        ((uint16_t *)sg.out_minus)[o + j] = (uint16_t)(mh[w] >> sh);
        ((uint16_t *)sg.out_minus_lo)[o + j] = (uint16_t)(ml[w] >> sh);
      }
    }
  }
}

#ifndef ZO2_K2_CERT_UPDATE
#define ZO2_K2_CERT_UPDATE 1
#endif
// z~ of the 4 draws of one Philox block (K2c section below)
__device__ __forceinline__ void za_z4(const uint64_t r[4], float z[4], float tau[4]);
// The exact z of one raw draw (Cephes ndtri in IEEE double), out of line: the
// certified update below needs it for ~1e-4 of the elements.
__device__ __noinline__ double exact_z(uint64_t raw) { return zo2_ndtri(zo2_u53(raw)); }

// Deferred update of one f32 weight, x = f32(f64(w + f64(uc z))) (axpy1),
// decided from z~ (zo2_zapprox.cuh, |z~ - z| <= tau) when the whole interval
// of candidate values rounds to one binary32: |uc| = lr |g| is ~1e-7, so
// |uc| tau ~ 1e-13 against a binary32 ulp of ~1e-9 and almost every element
// is certified.  Margin: 1.01 |uc| tau plus 2^-50 (|w| + |uc z~|) for the two
// f64 roundings of the exact chain and of v +- m (each <= 2^-53 relative).
// Otherwise (non-finite w, y below z~'s range, or an interval straddling a
// rounding boundary) the element takes the exact z: the same bits as the
// queued exact path either way.
__device__ __forceinline__ float upd_cert(float w, double uc, float zt, float tau, uint64_t raw) {
  if (fabsf(w) <= 3.0e38f && tau < 1.0e30f) {
    const double zd = (double)zt;
    const double v = __dadd_rn((double)w, __dmul_rn(uc, zd));
    const double m = 1.01 * fabs(uc) * (double)tau + 0x1p-50 * (fabs((double)w) + fabs(uc * zd));
    const float lo = __double2float_rn(v - m), hi = __double2float_rn(v + m);
    if (__float_as_uint(lo) == __float_as_uint(hi)) return lo;
  }
  return axpy1(w, uc, exact_z(raw));
}
__device__ __forceinline__ double upd_cert(double w, double uc, float, float, uint64_t raw) {
  return axpy1(w, uc, exact_z(raw));  // not used: f64 arenas need the exact z
}

template <int FMT, bool FAST, bool UPD, bool PERT>
__device__ __forceinline__ void k2_tiles(void *arena, const K2Table &T, const K2Params &P,
                                         const ZxKeys2 &KS,
                                         K2Smem<typename Wire<FMT>::A> &sm, unsigned &nn,
                                         unsigned &ns) {
  typedef typename Wire<FMT>::A A;
  // f32 arenas: the update draw is certified from z~ in P1 (upd_cert) and only
  // the perturbation draws go through the exact queue (QU = queued update)
  constexpr bool CU = UPD && !FAST && FMT == ZO2_F32 && ZO2_K2_CERT_UPDATE;
  constexpr bool QU = UPD && !CU;
  constexpr int OFF = QU ? 4 : 0;  // first perturb slot
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const double expm2 = 0.13533528323661269189;
  const double one_m = __dsub_rn(1.0, expm2);
  const uint64_t total = T.tile_start[T.n];
  int buf = 0, si = 0;
  for (uint64_t tile = blockIdx.x; tile < total; tile += gridDim.x, buf ^= 1) {
    while (tile >= T.tile_start[si + 1]) ++si;  // tiles ascend: si never moves back
    const zo2_segment_desc &sg = T.s[si];
    const bool tr = T.transposed[si] != 0;
    const uint64_t ltile = tile - T.tile_start[si];
    A *W = sm.w[buf];

    // ---------------- P1: load mapping
    uint32_t r0 = 0, c0 = 0;
    uint64_t e0 = 0, idx;
    int cnt, widx;
    if (tr) {
      // 32-bit division: a segment has < 2^32 tiles
      const uint32_t lt = (uint32_t)ltile, tc = T.tiles_c[si], q = lt / tc;
      r0 = q * 32;
      c0 = (lt - q * tc) * 32;
      const uint32_t r = r0 + (t >> 3), c = c0 + 4 * (t & 7);
      cnt = (r < sg.rows && c < sg.cols) ? (int)min(4u, sg.cols - c) : 0;
      idx = sg.offset + (uint64_t)r * sg.cols + c;
      widx = (t >> 3) * WPITCH + 4 * (t & 7);
    } else {
      e0 = ltile * TE;
      const uint64_t seg_n = (uint64_t)sg.rows * sg.cols;
      const uint64_t e = e0 + 4 * (uint64_t)t;
      cnt = e < seg_n ? (int)min((uint64_t)4, seg_n - e) : 0;
      idx = sg.offset + e;
      widx = 4 * t;
    }
    A w[4] = {0, 0, 0, 0};
    const bool vec = cnt == 4 && (idx & 3) == 0;
    if (vec) Wire<FMT>::load4(arena, idx, w);
    else
      for (int j = 0; j < cnt; ++j) w[j] = Wire<FMT>::load1(arena, idx + j);
    if (CU) {
      // every lane (za_z4 votes across the warp); lanes past the segment end
      // draw at harmless positions and keep their zeros
      uint64_t r[4];
      float zt[4], tau[4];
      zx_raw4_k(KS.lrs, P.base + idx, r);
      za_z4(r, zt, tau);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < cnt) w[j] = upd_cert(w[j], P.ucoef, zt[j], tau[j], r[j]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) W[widx + j] = w[j];

    unsigned tmask = 0, cmask = 0, negmask = 0;
    auto classify = [&](int k, uint64_t raw, bool valid) {
      if (!valid) return;
      const double u = zx_u53(raw);
      double y = u;
      bool neg = true;
      if (y > one_m) {
        y = __dsub_rn(1.0, y);
        neg = false;
      }
      const int zi = zslot(k, t);
      if (u == 1.0) {
        sm.z[zi] = INFINITY;  // ndtri(1) = +inf (u > 0 always)
      } else if (y > expm2) {
        sm.z[zi] = y;
        cmask |= 1u << k;
      } else {
        sm.z[zi] = y;
        tmask |= 1u << k;
        if (neg) negmask |= 1u << k;
      }
    };
    if (FAST) {
      // rng = "fast": z straight from Philox4x32 + binary32 erfinv, no queue
      const uint64_t pos = P.base + idx;
      if (cnt > 0 && (pos & 3) == 0) {
        uint32_t r[4];
        if (UPD) {
          zo2f_philox(P.lrs_seed, ZO2_PERTURB_STREAM, pos >> 2, r);
#pragma unroll
          for (int j = 0; j < 4; ++j) sm.z[zslot(j, t)] = (double)zo2f_gauss(r[j]);
        }
        if (PERT) {
          zo2f_philox(P.rs_seed, ZO2_PERTURB_STREAM, pos >> 2, r);
#pragma unroll
          for (int j = 0; j < 4; ++j) sm.z[zslot(OFF + j, t)] = (double)zo2f_gauss(r[j]);
        }
      } else if (cnt > 0) {  // segment offsets not a multiple of 4 (toy widths)
        for (int j = 0; j < cnt; ++j) {
          if (UPD) sm.z[zslot(j, t)] = (double)zo2f_gauss_at(P.lrs_seed, ZO2_PERTURB_STREAM, pos + j);
          if (PERT) sm.z[zslot(OFF + j, t)] = (double)zo2f_gauss_at(P.rs_seed, ZO2_PERTURB_STREAM, pos + j);
        }
      }
      __syncthreads();
    } else {
    if (cnt > 0) {
      uint64_t r[4];
      if (QU) {
        zx_raw4_k(KS.lrs, P.base + idx, r);
#pragma unroll
        for (int j = 0; j < 4; ++j) classify(j, r[j], j < cnt);
      }
      if (PERT) {
        zx_raw4_k(KS.rs, P.base + idx, r);
#pragma unroll
        for (int j = 0; j < 4; ++j) classify(OFF + j, r[j], j < cnt);
      }
    }
    // queue offsets: warp-inclusive scan of packed (tails | centrals << 16)
    {
      const unsigned mine = (unsigned)__popc(tmask) | ((unsigned)__popc(cmask) << 16);
      unsigned incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      unsigned base = 0;
      if (lane == 31) base = atomicAdd(&sm.counts[buf], incl);
      base = __shfl_sync(0xffffffffu, base, 31);
      const unsigned excl = base + incl - mine;
      unsigned tp = excl & 0xffffu, cp = NSLOT - 1 - (excl >> 16);
      const int zb0 = zslot(0, t), zb1 = zslot(1, t) - NT;  // even / odd k bases
#pragma unroll
      for (int k = 0; k < (QU ? 4 : 0) + (PERT ? 4 : 0); ++k) {
        const int zi = ((k & 1) ? zb1 : zb0) + k * NT;
        if ((tmask >> k) & 1u) sm.q[tp++] = (uint16_t)(zi | (((negmask >> k) & 1u) << 15));
        if ((cmask >> k) & 1u) sm.q[cp--] = (uint16_t)zi;
      }
    }
    __syncthreads();

    // ---------------- P2: queue (tails, then centrals), 32 entries per warp
    {
      const unsigned cnts = sm.counts[buf];
      const int nt = (int)(cnts & 0xffffu), nc = (int)(cnts >> 16), ntot = nt + nc;
      int i0 = warp * 32;
#if ZO2_K2_TAIL_X2
      // two pure-tail chunks per trip: two independent FP64 chains per lane
      for (; i0 + NT + 32 <= nt; i0 += 2 * NT) {
        const unsigned ea = sm.q[i0 + lane], eb = sm.q[i0 + NT + lane];
        const int za = (int)(ea & 0x7FFFu), zb = (int)(eb & 0x7FFFu);
        const double ra = zx_ndtri_tail(sm.z[za], (ea >> 15) != 0, sm.logtab, sm.tcoef);
        const double rb = zx_ndtri_tail(sm.z[zb], (eb >> 15) != 0, sm.logtab, sm.tcoef);
        sm.z[za] = ra;
        sm.z[zb] = rb;
      }
#endif
      // chunks holding tail entries (the last one may also hold centrals)
      for (; i0 < nt; i0 += NT) {
        const int i = i0 + lane;
        if (i < nt) {
          const unsigned e = sm.q[i];
          const int zi = (int)(e & 0x7FFFu);
          sm.z[zi] = zx_ndtri_tail(sm.z[zi], (e >> 15) != 0, sm.logtab, sm.tcoef);
        } else if (i < ntot) {
          const int zi = sm.q[NSLOT - nc + (i - nt)];
          sm.z[zi] = zx_ndtri_central(sm.z[zi], zx_central_coef(ZX_CENTRAL_C));
        }
      }
      if (i0 < ntot) {
        // pure central chunks: coefficients held in registers across the loop
        const ZxCentral cc = zx_central_coef(sm.ccoef);
#if ZO2_K2_CENTRAL_X2
        // two entries per lane per trip: two independent FP64 chains in flight
        for (; i0 + NT < ntot; i0 += 2 * NT) {
          const int ia = i0 + lane, ib = i0 + NT + lane;
          const int za = sm.q[NSLOT - nc + (ia - nt)];
          const bool vb = ib < ntot;
          const int zb = vb ? sm.q[NSLOT - nc + (ib - nt)] : za;
          const double ra = zx_ndtri_central(sm.z[za], cc);
          const double rb = zx_ndtri_central(sm.z[zb], cc);
          sm.z[za] = ra;
          if (vb) sm.z[zb] = rb;
        }
#endif
        for (; i0 < ntot; i0 += NT) {
          const int i = i0 + lane;
          if (i < ntot) {
            const int zi = sm.q[NSLOT - nc + (i - nt)];
            sm.z[zi] = zx_ndtri_central(sm.z[zi], cc);
          }
        }
      }
    }
    __syncthreads();
    }  // !FAST

    // ---------------- P3: apply mapping
    if (t == 0) sm.counts[buf ^ 1] = 0;  // next tile's queue
    {
      const int kind = PERT ? sg.out_kind : ZO2_OUT_NONE;
      int acnt, wi0, wstep, za[4];
      uint64_t o;
      if (tr) {
        const int c = t >> 3, rb = 4 * (t & 7);
        const bool cok = c0 + c < sg.cols;
        acnt = cok ? (int)min(4u, sg.rows > r0 + rb ? sg.rows - (r0 + rb) : 0u) : 0;
        wi0 = rb * WPITCH + c;
        wstep = WPITCH;
#pragma unroll
        for (int i = 0; i < 4; ++i) za[i] = zslot(c & 3, (rb + i) * 8 + (c >> 2));
        o = (uint64_t)(c0 + c) * sg.rows + r0 + rb;
      } else {
        acnt = cnt;
        wi0 = 4 * t;
        wstep = 1;
#pragma unroll
        for (int i = 0; i < 4; ++i) za[i] = zslot(i, t);
        o = e0 + 4 * (uint64_t)t;
      }
      // straight-line chain; zslot(OFF + j, t) = zslot(j, t) + OFF * NT (same parity)
      A a[4], ap[4], am[4];
      bool bad = false;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = W[wi0 + i * wstep];
        const double zu = QU ? sm.z[za[i]] : 0.0;
        const double zp = PERT ? sm.z[za[i] + OFF * NT] : 0.0;
        chain_fast<QU, PERT>(a[i], ap[i], am[i], P.ucoef, zu, P.eps, zp);
        // a NaN anywhere in the chain (NaN weight, inf - inf) reaches the
        // restored weight: redo those elements with axpy1's exact NaN rules
        bad |= (i < acnt) && (a[i] != a[i]);
      }
      if (bad) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i >= acnt || a[i] == a[i]) continue;
          const double zu = QU ? sm.z[za[i]] : 0.0;
          const double zp = PERT ? sm.z[za[i] + OFF * NT] : 0.0;
          const Chain3<A> c = chain_exact<QU, PERT, A>(W[wi0 + i * wstep], P.ucoef, zu, P.eps, zp);
          a[i] = c.w;
          ap[i] = c.wp;
          am[i] = c.wm;
        }
      }
      if (acnt == 4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) W[wi0 + i * wstep] = a[i];
      } else {
        for (int i = 0; i < acnt; ++i) W[wi0 + i * wstep] = a[i];
      }
      if (kind != ZO2_OUT_NONE && acnt > 0) emit4<A>(sg, kind, o, ap, am, acnt);
    }
    __syncthreads();

    // ---------------- P4: load mapping, restored weights to the arena
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = W[widx + j];
    if (vec) Wire<FMT>::store4(arena, idx, w, nn, ns);
    else
      for (int j = 0; j < cnt; ++j) Wire<FMT>::store1(arena, idx + j, w[j], nn, ns);
    // the W buffer read here is rewritten two tiles later, after two barriers
  }
}

__device__ __forceinline__ double resolve_ucoef(const double *d_g, double lr, int &upd) {
  if (!upd) return 0.0;
  const double g = *d_g;
  if (upd == 1 && g == 0.0) {
    upd = 0;
    return 0.0;
  }
  return -(lr * g);
}

template <int FMT, bool FAST>
__global__ void __launch_bounds__(NT, ZO2_K2_MINB) k_update_perturb(void *arena, K2Table T, K2Params P,
                                                          const __grid_constant__ ZxKeys2 KS,
                                                          const double *d_g, double lr,
                                                          uint64_t *counts) {
  typedef typename Wire<FMT>::A A;
  __shared__ __align__(16) K2Smem<A> sm;
  for (int i = threadIdx.x; i < 256; i += NT) sm.logtab[i] = ZO2_LOG_TAB_D[i];
  if (threadIdx.x < 13) sm.ccoef[threadIdx.x] = ZX_CENTRAL_C[threadIdx.x];
  if (threadIdx.x < 42) sm.tcoef[threadIdx.x] = ZX_TAIL_C[threadIdx.x];
  if (threadIdx.x < 2) sm.counts[threadIdx.x] = 0;
  __syncthreads();
  int upd = P.do_update;
  P.ucoef = resolve_ucoef(d_g, lr, upd);
  unsigned nn = 0, ns = 0;
  if (upd && P.do_perturb) k2_tiles<FMT, FAST, true, true>(arena, T, P, KS, sm, nn, ns);
  else if (upd) k2_tiles<FMT, FAST, true, false>(arena, T, P, KS, sm, nn, ns);
  else if (P.do_perturb) k2_tiles<FMT, FAST, false, true>(arena, T, P, KS, sm, nn, ns);
  else k2_tiles<FMT, FAST, false, false>(arena, T, P, KS, sm, nn, ns);
  if (FMT != ZO2_F32 && FMT != ZO2_F64) add_counts(counts, nn, ns);
}

// ============================================================================
// K2c: the certified path for codec arenas (bf16 / f16 / e4m3 wire) whose
// matrix operands are bf16 -- the AMP configurations 3-5.  Every output of
// the element chain is a narrow rounding (arena code, bf16 operand), so the
// chain runs in binary32 on z~ (zo2_zapprox.cuh) and an output is kept only
// if the whole interval [v - M, v + M] that provably contains the exact
// chain's value encodes to one code (the encoders are monotone).  Elements
// that fail (~1e-3 at the model's weight scales) are appended to a per-stream
// fix-up list and recomputed with the exact z (Philox4x64 + Cephes in IEEE
// double, axpy1 NaN rules) by a second kernel on the same stream, 32 per
// warp, so the rare exact element costs a lane, not a diverged warp.  The
// result is the reference's bits either way.  Vector segments (f32 operands
// for LN / bias epilogues) always take the exact chain inline.
//
// Error bound.  Exact chain (chain_exact): x = f32(w + f64(uc zu));
// ez = f64(eps zp); p = f32(x + ez); m = f32(p - 2 ez); w' = f32(m + ez).
// Here: x~ = fma32(uc, z~u, w), e = f32(eps z~p), p~ = f32(x~ + e),
// m~ = fma32(-2, e, p~), w~' = f32(m~ + e).  With Du = x~ - x - r0 and
// D = e - ez (the same D enters all three steps, it is one number):
//   p~ - p  = (x~ - x) + D + r1
//   m~ - m  = (p~ - p) - 2D + r2 = (x~ - x) - D + r1 + r2
//   w~' - w' = (m~ - m) + D + r3 = (x~ - x) + r1 + r2 + r3
// |ri| <= 2^-24 |vi| (round to nearest), |x~ - x| <= |uc| tau_u + 2^-24
// (|uc z~u| + 2|x|), |D| <= eps tau_p + 2^-23 |e|; the f64 roundings of the
// exact chain are 2^-29 of these.  So with A = max |x|, |p|, |m|, |w'|:
//   M_pm = |uc| tau_u + eps tau_p + 2^-22 (A + |uc z~u| + |e|)
//   M_w  = |uc| tau_u + 2^-22 (A + |uc z~u|)        (z~p cancels in w')
// (times 1.01), so the restored arena weight almost never needs the exact z.
// ============================================================================
// elements recomputed with the exact z (diagnostics: zo2_k2c_fallbacks)
__device__ unsigned long long g_k2c_redo = 0;

struct K2cEntry {
  uint64_t idx;  // element index in the module bucket
  float w0;      // decoded arena value before the chain
  uint32_t pad;
};
struct K2cList {
  unsigned long long *count;  // device counter, zeroed before every K2c launch
  unsigned long long cap;
  K2cEntry *e;
};

// the codec's code of a finite value below cert_lim (no NaN / saturation
// cases): bf16 RNE on the bits (numerics.py:232-245), f16 cvt.rn (numpy's
// cast), e4m3 the full encoder
template <int FMT>
__device__ __forceinline__ uint32_t code_of(float v) {
  if (FMT == ZO2_BF16) {
    const uint32_t u = __float_as_uint(v);
    return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
  }
  if (FMT == ZO2_F16) return __half_as_ushort(__float2half_rn(v));
  unsigned a = 0, b = 0;
  return enc_e4m3(v, a, b);
}
template <int FMT>
__device__ __forceinline__ void store1_cert(void *arena, uint64_t i, float w) {
  if (FMT == ZO2_F8E4M3) ((uint8_t *)arena)[i] = (uint8_t)code_of<FMT>(w);
  else ((uint16_t *)arena)[i] = (uint16_t)code_of<FMT>(w);
}
// store 4 certified values (codes as code_of), or fall back to the codec
template <int FMT>
__device__ __forceinline__ void store4_cert(void *arena, uint64_t i, const float w[4], unsigned &nn,
                                            unsigned &ns) {
  if (FMT == ZO2_BF16) {
    uint2 v;
    v.x = code_of<FMT>(w[0]) | (code_of<FMT>(w[1]) << 16);
    v.y = code_of<FMT>(w[2]) | (code_of<FMT>(w[3]) << 16);
    *(uint2 *)((uint16_t *)arena + i) = v;
  } else if (FMT == ZO2_F16) {
    uint2 v;
    v.x = code_of<FMT>(w[0]) | (code_of<FMT>(w[1]) << 16);
    v.y = code_of<FMT>(w[2]) | (code_of<FMT>(w[3]) << 16);
    *(uint2 *)((uint16_t *)arena + i) = v;
  } else {
    Wire<FMT>::store4(arena, i, w, nn, ns);
  }
}
// below these magnitudes no value of the interval saturates (so the codec's
// saturation counter cannot differ between the two chains)
template <int FMT> __device__ __forceinline__ float cert_lim() {
  return FMT == ZO2_BF16 ? 1e38f : FMT == ZO2_F16 ? 32768.0f : 256.0f;
}

__device__ __forceinline__ uint64_t raw_at(const ZxKeys &K, uint64_t pos) {
  uint64_t b[4];
  zx_philox_block_k(K, pos >> 2, b);
  const unsigned l = (unsigned)(pos & 3);
  return l == 0 ? b[0] : l == 1 ? b[1] : l == 2 ? b[2] : b[3];
}

// the exact element: Philox4x64 + Cephes (zo2_rng.h) + axpy1 chain
template <bool UPD, bool PERT>
__device__ __noinline__ Chain3<float> cert_exact(float w, const ZxKeys2 &KS, uint64_t pos,
                                                  double uc, double eps) {
  const double zu = UPD ? zo2_ndtri(zo2_u53(raw_at(KS.lrs, pos))) : 0.0;
  const double zp = PERT ? zo2_ndtri(zo2_u53(raw_at(KS.rs, pos))) : 0.0;
  return chain_exact<UPD, PERT, float>(w, uc, zu, eps, zp);
}

// z~ for the 4 draws of one Philox block, warp-converged: Giles' central
// polynomial for every draw, the tail one only when some lane needs it
// (same operations as za_g, so the same values the bound probe checked).
__device__ __forceinline__ void za_z4(const uint64_t r[4], float z[4], float tau[4]) {
  float w[4], x[4];
  bool up[4], tail = false;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float y = za_y(r[j], up[j]);
    x[j] = __fmaf_rn(-2.0f, y, 1.0f);
    const float a = __fmul_rn(__fmul_rn(4.0f, y), __fsub_rn(1.0f, y));
    w[j] = __fmul_rn(za_lg2(a), -0.69314718056f);
    tau[j] = y >= ZA_Y_MIN ? 0.0f : __int_as_float(0x7f800000);
    tail |= !(w[j] < 5.0f);
  }
  float p[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) p[j] = za_central(__fsub_rn(w[j], 2.5f));
  if (__any_sync(0xffffffffu, tail)) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (!(w[j] < 5.0f)) p[j] = za_tailp(__fsub_rn(za_sqrt(w[j]), 3.0f));
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float g = __fmul_rn(1.41421356237f, __fmul_rn(p[j], x[j]));
    tau[j] = __fadd_rn(tau[j], __fmaf_rn(ZA_TAU_REL, g, ZA_TAU_ABS));
    z[j] = up[j] ? g : -g;
  }
}

template <int FMT, bool UPD, bool PERT>
__device__ void k2c_exact_inline(void *arena, uint64_t idx, float w0, const ZxKeys2 &KS,
                                 const K2Params &P, float &w, float &op, float &om) {
  const Chain3<float> c = cert_exact<UPD, PERT>(w0, KS, P.base + idx, P.ucoef, P.eps);
  w = c.w;
  op = c.wp;
  om = c.wm;
}

// Coordinates of warp tile `wt`: lane = row (transposed: 32 rows x 4 columns,
// the lane's 4 elements are one Philox block of its row) or 4 consecutive
// elements (linear: 128 per warp).  Operand rows [N, K] of a transposed
// segment are then written as 32 consecutive bf16 per column: coalesced,
// without a shared-memory transpose or a barrier.
struct K2cTile {
  uint64_t idx, o;  // first element in the bucket; first operand index
  int si, cnt, ostride;
};
__device__ __forceinline__ void k2c_coords(const K2Table &T, uint64_t wt, int &si, int lane,
                                           K2cTile &c) {
  while (wt >= T.wt_start[si + 1]) ++si;  // tiles ascend: si never moves back
  const zo2_segment_desc &sg = T.s[si];
  const uint64_t lt = wt - T.wt_start[si];
  c.si = si;
  if (T.transposed[si]) {
    const uint32_t l = (uint32_t)lt, q = l / T.wt_c[si];
    const uint32_t r = q * 32 + lane, col = (l - q * T.wt_c[si]) * 4;
    c.cnt = (r < sg.rows) ? (int)min(4u, sg.cols - col) : 0;
    c.idx = sg.offset + (uint64_t)r * sg.cols + col;
    c.o = (uint64_t)col * sg.rows + r;  // operand [cols][rows]
    c.ostride = (int)sg.rows;
  } else {
    const uint64_t seg_n = (uint64_t)sg.rows * sg.cols;
    const uint64_t e = lt * 128 + 4 * (uint64_t)lane;
    c.cnt = e < seg_n ? (int)min((uint64_t)4, seg_n - e) : 0;
    c.idx = sg.offset + e;
    c.o = e;
    c.ostride = 1;
  }
}

template <int FMT>
__device__ __forceinline__ void k2c_load(const void *arena, const K2cTile &c, float w[4]) {
  w[0] = w[1] = w[2] = w[3] = 0.f;
  if (c.cnt == 4 && (c.idx & 3) == 0) Wire<FMT>::load4(arena, c.idx, w);
  else
    for (int j = 0; j < c.cnt; ++j) w[j] = Wire<FMT>::load1(arena, c.idx + j);
}

template <int FMT, bool UPD, bool PERT>
__device__ __forceinline__ void k2c_tiles(void *arena, const K2Table &T, const K2Params &P,
                                          const ZxKeys2 &KS, K2cList L, unsigned &nn,
                                          unsigned &ns) {
  const int lane = threadIdx.x & 31;
  const float ucf = (float)P.ucoef, epsf = (float)P.eps;
  const float auc = fabsf(ucf), aeps = fabsf(epsf);
  const uint64_t total = T.wt_start[T.n];
  const uint64_t stride = (uint64_t)gridDim.x * (NT / 32);
  uint64_t wt = (uint64_t)blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
  int si = 0;
  K2cTile cur;
  for (; wt < total; wt += stride) {
    // (prefetching the next tile's weights here measured 5% slower: spills)
    k2c_coords(T, wt, si, lane, cur);
    float w[4], op[4], om[4];
    k2c_load<FMT>(arena, cur, w);
    const K2cTile c = cur;
    const zo2_segment_desc &sg = T.s[c.si];
    const int kind = PERT ? sg.out_kind : ZO2_OUT_NONE;
    const int cnt = c.cnt;
    const uint64_t idx = c.idx;
    const bool vec = cnt == 4 && (idx & 3) == 0;
    unsigned inl = 0;  // elements computed by the exact chain here (codec-encoded)
    if (kind == ZO2_OUT_F32) {
      // vector segment (warp-uniform): f32 operands need the exact chain
      inl = cnt > 0 ? (1u << cnt) - 1u : 0u;
      for (int j = 0; j < cnt; ++j)
        k2c_exact_inline<FMT, UPD, PERT>(arena, idx + j, w[j], KS, P, w[j], op[j], om[j]);
    } else {
      // the warp stays converged here (lanes past a segment edge compute
      // unused values): za_z4 votes across the warp
      float zu[4], tu[4], zp[4], tp[4];
      uint64_t r[4];
      if (UPD) {
        zx_raw4_k(KS.lrs, P.base + idx, r);
        za_z4(r, zu, tu);
      }
      if (PERT) {
        zx_raw4_k(KS.rs, P.base + idx, r);
        za_z4(r, zp, tp);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float x0 = w[j];
        float x = x0, e = 0.f, p, m, wn;
        float Mu = 0.f, R = 0.f;
        if (UPD) {
          x = __fmaf_rn(ucf, zu[j], x0);
          Mu = __fmul_rn(auc, tu[j]);
          R = __fmul_rn(auc, fabsf(zu[j]));
        }
        if (PERT) {
          e = __fmul_rn(epsf, zp[j]);
          p = __fadd_rn(x, e);
          m = __fmaf_rn(-2.0f, e, p);
          wn = __fadd_rn(m, e);
        } else {
          p = m = wn = x;
        }
        const float A = fmaxf(fmaxf(fabsf(x0), fabsf(x)), fmaxf(fabsf(p), fabsf(m)));
        // R: magnitudes the roundings scale with (+ eps tau_p, so that an
        // unusable z~p, tau = inf, also voids the arena check)
        float Mp = Mu;
        R = __fadd_rn(R, A);
        if (PERT) {
          const float et = __fmul_rn(aeps, tp[j]);
          R = __fadd_rn(R, __fadd_rn(fabsf(e), et));
          Mp = __fadd_rn(Mp, et);
        }
        const float Mw = __fmul_rn(__fmaf_rn(0x1p-22f, R, Mu), 1.01f);
        bool ok = (A < cert_lim<FMT>()) && (Mw < 1e30f) &&
                  code_of<FMT>(__fsub_rd(wn, Mw)) == code_of<FMT>(__fadd_ru(wn, Mw));
        if (kind != ZO2_OUT_NONE) {
          Mp = __fmul_rn(__fmaf_rn(0x1p-22f, R, Mp), 1.01f);
          ok = ok && bf16x2(__fsub_rd(p, Mp), __fsub_rd(m, Mp)) ==
                         bf16x2(__fadd_ru(p, Mp), __fadd_ru(m, Mp));
        }
        op[j] = p;
        om[j] = m;
        w[j] = wn;
        if (!ok && j < cnt) {
          const unsigned long long slot = atomicAdd(L.count, 1ull);
          atomicAdd(&g_k2c_redo, 1ull);
          if (slot < L.cap) {
            L.e[slot].idx = idx + j;
            L.e[slot].w0 = x0;
            w[j] = 0.0f;  // placeholder code (no codec counts); fix-up rewrites it
          } else {       // list full: this element inline
            k2c_exact_inline<FMT, UPD, PERT>(arena, idx + j, x0, KS, P, w[j], op[j], om[j]);
            inl |= 1u << j;
          }
        }
      }
    }
    // restored (updated) weights, re-encoded, straight back to the arena;
    // exact-chain elements (NaN / saturation possible) through the codec
    if (vec && !inl) store4_cert<FMT>(arena, idx, w, nn, ns);
    else
      for (int j = 0; j < cnt; ++j) {
        if ((inl >> j) & 1u) Wire<FMT>::store1(arena, idx + j, w[j], nn, ns);
        else store1_cert<FMT>(arena, idx + j, w[j]);
      }
    if (kind == ZO2_OUT_F32) {
      for (int j = 0; j < cnt; ++j) {
        ((float *)sg.out_plus)[c.o + j] = op[j];
        ((float *)sg.out_minus)[c.o + j] = om[j];
      }
    } else if (kind == ZO2_OUT_BF16) {
      if (vec) {
        *(uint2 *)((__nv_bfloat16 *)sg.out_plus + c.o) = make_uint2(bf16x2(op[0], op[1]), bf16x2(op[2], op[3]));
        *(uint2 *)((__nv_bfloat16 *)sg.out_minus + c.o) = make_uint2(bf16x2(om[0], om[1]), bf16x2(om[2], om[3]));
      } else {
        for (int j = 0; j < cnt; ++j) {
          ((__nv_bfloat16 *)sg.out_plus)[c.o + j] = __float2bfloat16_rn(op[j]);
          ((__nv_bfloat16 *)sg.out_minus)[c.o + j] = __float2bfloat16_rn(om[j]);
        }
      }
    } else if (kind == ZO2_OUT_BF16_T) {
      // column j of the tile -> operand row (col + j), this lane's K position:
      // 32 lanes write 32 consecutive bf16 (64 B) per column and sign
      const uint32_t pp01 = bf16x2(op[0], op[1]), pp23 = bf16x2(op[2], op[3]);
      const uint32_t mm01 = bf16x2(om[0], om[1]), mm23 = bf16x2(om[2], om[3]);
      const uint32_t pv[2] = {pp01, pp23}, mv[2] = {mm01, mm23};
      uint16_t *P_ = (uint16_t *)sg.out_plus + c.o, *M_ = (uint16_t *)sg.out_minus + c.o;
      const uint64_t os = (uint64_t)c.ostride;
      if (cnt == 4) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          P_[j * os] = (uint16_t)(pv[j >> 1] >> (16 * (j & 1)));
          M_[j * os] = (uint16_t)(mv[j >> 1] >> (16 * (j & 1)));
        }
      } else {
        for (int j = 0; j < cnt; ++j) {
          P_[j * os] = (uint16_t)(pv[j >> 1] >> (16 * (j & 1)));
          M_[j * os] = (uint16_t)(mv[j >> 1] >> (16 * (j & 1)));
        }
      }
    }
  }
}

#ifndef ZO2_K2C_MINB
#define ZO2_K2C_MINB 3
#endif
template <int FMT>
__global__ void __launch_bounds__(NT, ZO2_K2C_MINB) k_update_perturb_cert(void *arena, K2Table T, K2Params P,
                                                            const __grid_constant__ ZxKeys2 KS,
                                                            const double *d_g, double lr,
                                                            uint64_t *counts, K2cList L) {
  int upd = P.do_update;
  P.ucoef = resolve_ucoef(d_g, lr, upd);
  unsigned nn = 0, ns = 0;
  if (upd && P.do_perturb) k2c_tiles<FMT, true, true>(arena, T, P, KS, L, nn, ns);
  else if (upd) k2c_tiles<FMT, true, false>(arena, T, P, KS, L, nn, ns);
  else if (P.do_perturb) k2c_tiles<FMT, false, true>(arena, T, P, KS, L, nn, ns);
  else k2c_tiles<FMT, false, false>(arena, T, P, KS, L, nn, ns);
  add_counts(counts, nn, ns);
}

// Fix-up of the listed elements (stream-ordered after k_update_perturb_cert):
// exact chain, arena code and operands rewritten at their positions.
template <int FMT>
__global__ void __launch_bounds__(128) k_k2c_fixup(void *arena, K2Table T, K2Params P,
                                                   const __grid_constant__ ZxKeys2 KS,
                                                   const double *d_g, double lr,
                                                   uint64_t *counts, K2cList L) {
  int upd = P.do_update;
  P.ucoef = resolve_ucoef(d_g, lr, upd);
  const uint64_t n = min(*L.count, L.cap);
  unsigned nn = 0, ns = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const K2cEntry en = L.e[i];
    Chain3<float> c;
    if (upd && P.do_perturb) c = cert_exact<true, true>(en.w0, KS, P.base + en.idx, P.ucoef, P.eps);
    else if (upd) c = cert_exact<true, false>(en.w0, KS, P.base + en.idx, P.ucoef, P.eps);
    else if (P.do_perturb) c = cert_exact<false, true>(en.w0, KS, P.base + en.idx, P.ucoef, P.eps);
    else c = cert_exact<false, false>(en.w0, KS, P.base + en.idx, P.ucoef, P.eps);
    Wire<FMT>::store1(arena, en.idx, c.w, nn, ns);
    if (!P.do_perturb) continue;
    int k = 0;
    while (k + 1 < T.n && en.idx >= T.s[k + 1].offset) ++k;
    const zo2_segment_desc &sg = T.s[k];
    const uint64_t rel = en.idx - sg.offset;
    uint64_t o = rel;
    if (T.transposed[k]) o = (rel % sg.cols) * sg.rows + rel / sg.cols;
    if (sg.out_kind == ZO2_OUT_BF16 || sg.out_kind == ZO2_OUT_BF16_T) {
      ((__nv_bfloat16 *)sg.out_plus)[o] = __float2bfloat16_rn(c.wp);
      ((__nv_bfloat16 *)sg.out_minus)[o] = __float2bfloat16_rn(c.wm);
    }
  }
  // all lanes reach this point (no early return): warp-collective counts
  add_counts(counts, nn, ns);
}

// 0 = certified path where it applies (default), 1 = always the queued exact kernel
int g_k2_variant = 0;

// fix-up lists, one per CUDA stream (K2c launches on one stream are ordered)
struct K2cSlot {
  cudaStream_t s;
  void *buf;
  unsigned long long cap;
};
K2cSlot g_k2c_slots[16];
int g_k2c_nslots = 0;

int k2c_list_for(cudaStream_t s, uint64_t n, K2cList &L) {
  const unsigned long long want = n >> 9 > (1ull << 18) ? n >> 9 : (1ull << 18);
  K2cSlot *sl = nullptr;
  for (int i = 0; i < g_k2c_nslots; ++i)
    if (g_k2c_slots[i].s == s) sl = &g_k2c_slots[i];
  if (!sl) {
    if (g_k2c_nslots == 16) sl = &g_k2c_slots[15];  // recycle (synchronised below)
    else sl = &g_k2c_slots[g_k2c_nslots++];
    sl->s = s;
    sl->buf = nullptr;
    sl->cap = 0;
  }
  if (sl->cap < want) {
    if (sl->buf) {
      ZO2_CUDA_TRY(cudaDeviceSynchronize());
      ZO2_CUDA_TRY(cudaFree(sl->buf));
    }
    ZO2_CUDA_TRY(cudaMalloc(&sl->buf, 16 + want * sizeof(K2cEntry)));
    sl->cap = want;
  }
  L.count = (unsigned long long *)sl->buf;
  L.cap = sl->cap;
  L.e = (K2cEntry *)((char *)sl->buf + 16);
  return ZO2_OK;
}

template <int FMT>
int launch_k2c(void *arena, const K2Table &T, const K2Params &P, const double *d_g, double lr,
               uint64_t *counts, cudaStream_t s) {
  const uint64_t tiles = (T.wt_start[T.n] + NT / 32 - 1) / (NT / 32);  // CTA-sized groups
  if (tiles == 0) return ZO2_OK;
  static int occ = 0;
  if (occ == 0) {
    ZO2_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update_perturb_cert<FMT>, NT, 0));
    if (occ < 1) occ = 1;
  }
  unsigned per_sm = (unsigned)occ;
  if (g_k2_ctas_per_sm && g_k2_ctas_per_sm < per_sm) per_sm = g_k2_ctas_per_sm;
  const uint64_t cap = 148ull * per_sm;
  const unsigned g = (unsigned)(tiles < cap ? tiles : cap);
  ZxKeys2 KS;
  zx_round_keys(P.lrs_seed, ZO2_PERTURB_STREAM, KS.lrs);
  zx_round_keys(P.rs_seed, ZO2_PERTURB_STREAM, KS.rs);
  K2cList L;
  const int rc = k2c_list_for(s, T.wt_start[T.n] * 128, L);
  if (rc != ZO2_OK) return rc;
  ZO2_CUDA_TRY(cudaMemsetAsync(L.count, 0, sizeof(unsigned long long), s));
  k_update_perturb_cert<FMT><<<g, NT, 0, s>>>(arena, T, P, KS, d_g, lr, counts, L);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  k_k2c_fixup<FMT><<<148, 128, 0, s>>>(arena, T, P, KS, d_g, lr, counts, L);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

// ---------------------------------------------------------------- bound probe
// For every binary32 y in [2^-24, 1/2]: the 53-bit integers y53 whose
// fl32((2 y53 + 1) 2^-54) is y form one interval; z is monotone in the raw
// integer, so the exact z at the interval ends (both sides of 1/2) bracket
// every exact z that shares this z~.  out[0] = max |z~ - z| / tau(z~),
// out[1] = max |z~ - z|, out[2] = za_y mismatches at the ends (must be 0),
// out[3 + b] = max |z~ - z| / (1 + |z~|) in binade b of y (2^(b-24)).
__device__ __forceinline__ void atomic_max_pos(float *a, float v) {
  atomicMax((int *)a, __float_as_int(v));
}
__global__ void k_zapprox_probe(float *out) {
  const uint32_t lo = 0x33800000u, hi = 0x3F000000u;  // 2^-24 .. 0.5
  float mr = 0.f, ma = 0.f, mismatch = 0.f;
  for (uint32_t b = lo + blockIdx.x * blockDim.x + threadIdx.x; b <= hi;
       b += gridDim.x * blockDim.x) {
    const float f = __uint_as_float(b);
    const float fu = __uint_as_float(b + 1), fd = __uint_as_float(b - 1);
    const uint64_t F = (uint64_t)((double)f * 0x1p54);
    const uint64_t hu = (uint64_t)(((double)fu - (double)f) * 0x1p53);
    const uint64_t hd = (uint64_t)(((double)f - (double)fd) * 0x1p53);
    uint64_t nlo = F - hd + 1, nhi = F + hu - 1;
    if (nhi > (1ull << 53) - 1) nhi = (1ull << 53) - 1;
    const float g = za_g(f);
    const float tau = __fmaf_rn(ZA_TAU_REL, g, ZA_TAU_ABS);
    float mrel = 0.f;
    for (int end = 0; end < 2; ++end) {
      const uint64_t y53 = ((end ? nhi : nlo) - 1) >> 1;
      for (int side = 0; side < 2; ++side) {
        const uint64_t m = side ? ((1ull << 53) - 1 - y53) : y53;
        bool upper;
        if (za_y(m << 11, upper) != f || upper != (side != 0)) mismatch += 1.f;
        const double z = zo2_ndtri(zo2_u53(m << 11));
        const float za = side ? g : -g;
        const float err = (float)fabs((double)za - z);
        mr = fmaxf(mr, err / tau);
        ma = fmaxf(ma, err);
        mrel = fmaxf(mrel, err / (1.f + g));
      }
    }
    const int bin = (int)((b >> 23) & 0xFF) - (127 - 24);
    atomic_max_pos(&out[3 + bin], mrel);
  }
  atomic_max_pos(&out[0], mr);
  atomic_max_pos(&out[1], ma);
  if (mismatch > 0.f) atomicAdd(&out[2], mismatch);
}

template <int FMT, bool FAST>
int launch_k2(void *arena, const K2Table &T, const K2Params &P, const double *d_g, double lr,
              uint64_t *counts, cudaStream_t s) {
  const uint64_t tiles = T.tile_start[T.n];
  if (tiles == 0) return ZO2_OK;
  static int occ = 0;
  if (occ == 0) {
    // maximum shared-memory carveout: an SM configured for this kernel can
    // also host the persistent GEMM CTA (co-residence on the prepare lane)
    ZO2_CUDA_TRY(cudaFuncSetAttribute(k_update_perturb<FMT, FAST>,
                                      cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    ZO2_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update_perturb<FMT, FAST>, NT, 0));
    if (occ < 1) occ = 1;
  }
  unsigned per_sm = (unsigned)occ;
  if (g_k2_ctas_per_sm && g_k2_ctas_per_sm < per_sm) per_sm = g_k2_ctas_per_sm;
  const uint64_t cap = 148ull * per_sm;
  const unsigned g = (unsigned)(tiles < cap ? tiles : cap);
  ZxKeys2 KS;
  zx_round_keys(P.lrs_seed, ZO2_PERTURB_STREAM, KS.lrs);
  zx_round_keys(P.rs_seed, ZO2_PERTURB_STREAM, KS.rs);
  k_update_perturb<FMT, FAST><<<g, NT, 0, s>>>(arena, T, P, KS, d_g, lr, counts);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

}  // namespace

extern "C" int zo2_set_k2_ctas_per_sm(int n) {
  if (n < 0 || n > 32) return zo2_set_error(ZO2_E_ARG, "zo2_set_k2_ctas_per_sm: 0..32");
  g_k2_ctas_per_sm = (unsigned)n;
  return ZO2_OK;
}

extern "C" int zo2_set_k2_variant(int v) {
  if (v != 0 && v != 1) return zo2_set_error(ZO2_E_ARG, "zo2_set_k2_variant: 0 (certified where valid) or 1 (queued exact)");
  g_k2_variant = v;
  return ZO2_OK;
}

extern "C" int zo2_k2c_fallbacks(uint64_t *out, int reset) {
  if (!out) return zo2_set_error(ZO2_E_ARG, "zo2_k2c_fallbacks: null output");
  unsigned long long v = 0;
  ZO2_CUDA_TRY(cudaMemcpyFromSymbol(&v, g_k2c_redo, sizeof(v)));
  *out = v;
  if (reset) {
    v = 0;
    ZO2_CUDA_TRY(cudaMemcpyToSymbol(g_k2c_redo, &v, sizeof(v)));
  }
  return ZO2_OK;
}

extern "C" int zo2_zapprox_bound_probe(float *d_out, void *cs) {
  if (!d_out) return zo2_set_error(ZO2_E_ARG, "zo2_zapprox_bound_probe: null output");
  ZO2_CUDA_TRY(cudaMemsetAsync(d_out, 0, 32 * sizeof(float), (cudaStream_t)cs));
  k_zapprox_probe<<<148 * 8, 256, 0, (cudaStream_t)cs>>>(d_out);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

extern "C" int zo2_set_rng_mode(int mode) {
  if (mode != 0 && mode != 1) return zo2_set_error(ZO2_E_ARG, "zo2_set_rng_mode: 0 (exact) or 1 (fast)");
  g_rng_mode = mode;
  return ZO2_OK;
}
extern "C" int zo2_rng_mode(void) { return g_rng_mode; }

extern "C" int zo2_update_perturb(void *arena, int wire_fmt, uint64_t n, uint64_t base,
                                  int update, const double *d_g, double lr,
                                  uint64_t lrs_seed, int perturb, double eps,
                                  uint64_t rs_seed, const zo2_segment_desc *segs,
                                  int n_segs, uint64_t *counts, void *cs) {
  if (n == 0) return ZO2_OK;
  if (!arena) return zo2_set_error(ZO2_E_ARG, "zo2_update_perturb: null arena");
  if (update && !d_g) return zo2_set_error(ZO2_E_ARG, "zo2_update_perturb: update needs d_g");
  if (n_segs < 1 || n_segs > MAX_SEGS)
    return zo2_set_error(ZO2_E_ARG, "zo2_update_perturb: 1..16 segments required");
  K2Table T;
  memset(&T, 0, sizeof(T));
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
    T.s[k] = sg;
    if (!perturb) T.s[k].out_kind = ZO2_OUT_NONE;
    T.transposed[k] = (t && perturb) ? 1 : 0;
    T.any_transposed |= T.transposed[k];
    uint64_t tiles;
    if (T.transposed[k]) {
      T.tiles_c[k] = (sg.cols + 31) / 32;
      tiles = (uint64_t)((sg.rows + 31) / 32) * T.tiles_c[k];
    } else {
      tiles = (sn + TE - 1) / TE;
    }
    T.tile_start[k + 1] = T.tile_start[k] + tiles;
    uint64_t wt;
    if (T.transposed[k]) {
      T.wt_c[k] = (sg.cols + 3) / 4;
      wt = (uint64_t)((sg.rows + 31) / 32) * T.wt_c[k];
    } else {
      wt = (sn + 127) / 128;
    }
    T.wt_start[k + 1] = T.wt_start[k] + wt;
  }
  T.n = n_segs;
  if (covered != n) return zo2_set_error(ZO2_E_ARG, "zo2_update_perturb: segments do not cover n");
  K2Params P;
  P.base = base;
  P.do_update = update;
  P.ucoef = 0.0;
  P.lrs_seed = lrs_seed;
  P.do_perturb = perturb;
  P.eps = eps;
  P.rs_seed = rs_seed;
  cudaStream_t s = (cudaStream_t)cs;
  const bool fast = g_rng_mode == 1;
  bool cert = !fast && g_k2_variant == 0 &&
              (wire_fmt == ZO2_BF16 || wire_fmt == ZO2_F16 || wire_fmt == ZO2_F8E4M3);
  for (int k = 0; k < n_segs && cert; ++k) {
    const int kd = T.s[k].out_kind;
    cert = kd == ZO2_OUT_NONE || kd == ZO2_OUT_BF16 || kd == ZO2_OUT_BF16_T ||
           (kd == ZO2_OUT_F32 && !T.transposed[k]);
  }
  if (cert) {
    switch (wire_fmt) {
      case ZO2_BF16: return launch_k2c<ZO2_BF16>(arena, T, P, d_g, lr, counts, s);
      case ZO2_F16: return launch_k2c<ZO2_F16>(arena, T, P, d_g, lr, counts, s);
      default: return launch_k2c<ZO2_F8E4M3>(arena, T, P, d_g, lr, counts, s);
    }
  }
  switch (wire_fmt) {
    case ZO2_F64: return fast ? launch_k2<ZO2_F64, true>(arena, T, P, d_g, lr, counts, s)
                          : launch_k2<ZO2_F64, false>(arena, T, P, d_g, lr, counts, s);
    case ZO2_F32: return fast ? launch_k2<ZO2_F32, true>(arena, T, P, d_g, lr, counts, s)
                          : launch_k2<ZO2_F32, false>(arena, T, P, d_g, lr, counts, s);
    case ZO2_BF16: return fast ? launch_k2<ZO2_BF16, true>(arena, T, P, d_g, lr, counts, s)
                          : launch_k2<ZO2_BF16, false>(arena, T, P, d_g, lr, counts, s);
    case ZO2_F16: return fast ? launch_k2<ZO2_F16, true>(arena, T, P, d_g, lr, counts, s)
                          : launch_k2<ZO2_F16, false>(arena, T, P, d_g, lr, counts, s);
    case ZO2_F8E4M3: return fast ? launch_k2<ZO2_F8E4M3, true>(arena, T, P, d_g, lr, counts, s)
                          : launch_k2<ZO2_F8E4M3, false>(arena, T, P, d_g, lr, counts, s);
    default: return zo2_set_error(ZO2_E_ARG, "zo2_update_perturb: bad wire format");
  }
}
