// zgen_warp.cuh -- (tools only) the previous, warp-cooperative evaluation of
// z = ndtri(u), kept for A/B against the CTA-queue kernel in zo2_k2.cu.
//
// Cephes ndtri has a cheap central branch (73% of draws) and an expensive tail
// branch (2 logs, sqrt, 2 divisions, degree-8 rationals).  Evaluated per lane,
// nearly every warp executes BOTH branches for every draw slot.  Here each
// lane evaluates its central draws in place, tail draws are compacted into a
// per-warp queue in shared memory and evaluated 32 at a time by all lanes,
// then returned to their owners.  Results are bit-identical to zo2_ndtri()
// (same scalar routines, same operation order) -- only the lane that computes
// a given draw changes.
#pragma once
#include "../paper_2503_12668_b200/csrc/zo2_rng.h"
#ifndef ZO2_CENTRAL_BRANCHLESS
#define ZO2_CENTRAL_BRANCHLESS 0
#endif

// Per-warp scratch: N*32 doubles (values / results) + N*32 queue entries.
template <int N>
struct ZgenScratch {
  double val[N * 32];
  uint16_t q[N * 32];
};

#ifndef ZO2_RAW4_NOINLINE
#define ZO2_RAW4_NOINLINE 1
#endif
// Positions not aligned to a Philox block (never on the hot path: segment
// offsets are multiples of 4 when d % 4 == 0) -- kept out of line so the hot
// loop's code stays small enough for the instruction cache.
#if ZO2_RAW4_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
void zo2_raw4_unaligned(uint64_t seed, uint64_t stream, uint64_t pos, uint64_t *r) {
  for (int j = 0; j < 4; ++j) {
    uint64_t b[4];
    zo2_raw_block(seed, stream, (pos + j) >> 2, b);
    r[j] = b[(pos + j) & 3];
  }
}

// Raw draws for positions pos..pos+3 of (seed, stream).
__device__ __forceinline__ void zo2_raw4(uint64_t seed, uint64_t stream, uint64_t pos,
                                         uint64_t r[4]) {
  if ((pos & 3) == 0) zo2_raw_block(seed, stream, pos >> 2, r);
  else zo2_raw4_unaligned(seed, stream, pos, r);
}

#ifndef ZO2_CENTRAL_ROLLED
#define ZO2_CENTRAL_ROLLED 0
#endif

// All 32 lanes of the warp must call this together (convergent).
template <int N>
__device__ __forceinline__ void warp_ndtri(const double (&u)[N], double (&z)[N],
                                           ZgenScratch<N> &sc) {
  const double expm2 = 0.13533528323661269189;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned lt = (1u << lane) - 1u;
  unsigned qn = 0;
  unsigned tail_bits = 0;     // slots of this lane that went to the tail queue
  unsigned special_bits = 0;  // u == 0 or u == 1 (z = -inf / +inf)
#pragma unroll
  for (int s = 0; s < N; ++s) {
    const double y0 = u[s];
    double y = y0;
    int neg = 1;
    if (y > ZO2_DSUB(1.0, expm2)) {
      y = ZO2_DSUB(1.0, y);
      neg = 0;
    }
    const bool special = (y0 == 1.0) || (y0 == 0.0);
    const bool tail = !special && !(y > expm2);
    if (special) special_bits |= 1u << s;
    const unsigned m = __ballot_sync(0xffffffffu, tail);
    if (tail) {
      const unsigned pos = qn + __popc(m & lt);
      sc.q[pos] = (uint16_t)((s * 32 + lane) | (neg ? 0x8000u : 0u));
      tail_bits |= 1u << s;
    }
    qn += __popc(m);
#if ZO2_CENTRAL_ROLLED
    sc.val[s * 32 + lane] = y;
#else
    if (special) z[s] = (y0 == 1.0) ? INFINITY : -INFINITY;
    else if (!tail) z[s] = zo2_ndtri_central(y);
    if (tail) sc.val[s * 32 + lane] = y;
#endif
  }
#if ZO2_CENTRAL_ROLLED
  // central branch in a rolled loop over the staged values: one copy of the
  // rational evaluation in the instruction stream instead of N
#pragma unroll 1
  for (int s = 0; s < N; ++s) {
    if (((tail_bits | special_bits) >> s) & 1u) continue;
    sc.val[s * 32 + lane] = zo2_ndtri_central(sc.val[s * 32 + lane]);
  }
#endif
  __syncwarp();
  for (unsigned base = 0; base < qn; base += 32) {
    const unsigned i = base + lane;
    if (i < qn) {
      const unsigned e = sc.q[i];
      const unsigned idx = e & 0x7FFFu;
      sc.val[idx] = zo2_ndtri_tail(sc.val[idx], (e & 0x8000u) ? 1 : 0);
    }
  }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < N; ++s) {
#if ZO2_CENTRAL_ROLLED
    z[s] = ((special_bits >> s) & 1u) ? ((u[s] == 1.0) ? INFINITY : -INFINITY)
                                      : sc.val[s * 32 + lane];
#else
    if (tail_bits & (1u << s)) z[s] = sc.val[s * 32 + lane];
#endif
  }
  __syncwarp();
}
