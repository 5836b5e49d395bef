// zo2_gemm_sm100.cu -- K3: the dual-forward GEMMs on 5th-gen tensor cores.
//
//   C[M,N] = A[M,K] . B[N,K]^T     A, B bf16 K-major, fp32 accumulation in TMEM
//
// Persistent, warp-specialised kernel (one CTA per SM):
//   warp 0      TMA producer (cp.async.bulk.tensor, 128B swizzle, mbarrier tx)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> fused epilogue
// Two TMEM accumulators let the epilogue of tile i overlap the MMAs of i+1.
// The +eps and -eps problems of the dual forward are one launch (batch = 2).
//
// SPLIT (f32 arithmetic, model.py f32 path): operands carry a bf16 hi and a
// bf16 lo plane (x = hi + lo to ~2^-16) and every k-step issues
// hi.hi + hi.lo + lo.hi, all into the same fp32 TMEM accumulator.
//
// Epilogues (model.py:272-301): bias store (qkv), bias + residual (attention
// out-proj, MLP out), bias + erf-GELU emitted as the next GEMM's A operand
// (mlp_in), and the cross-entropy partials of the LM head (model.py:304-313)
// so the [T, V] logits never reach HBM.
#include "zo2_common.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>
#include <unordered_map>
#include <string.h>
#include <stdio.h>

void zo2_count_launch(uint64_t n = 1);

#ifndef ZO2_GEMM_SMEM_KB
#define ZO2_GEMM_SMEM_KB 200  // operand staging budget per CTA
#endif
// Smaller budgets (2 split / 5 bf16 stages) leave room for K2 CTAs beside a
// GEMM CTA; they used to hang the CTA-pair kernel's TMEM allocation (fixed by
// the cluster barrier before tcgen05.alloc.cta_group::2 in k_gemm2).

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = one 128-byte swizzle row
constexpr int NUM_THREADS = 192;

struct alignas(64) GemmArgs {
  CUtensorMap tm[2][4];  // [problem][a_hi, a_lo, b_hi, b_lo]
  const float *bias[2];
  void *c[2];
  void *c_lo[2];
  const int64_t *targets[2];
  float *ce_part[2];
  uint32_t M, N, K;
  int batch;
  uint32_t group_m;        // raster group height in M tiles (tile_mn)
  unsigned int *tile_ctr;  // [0] next tile, [1] CTAs finished (self-resetting)
};

// ---------------------------------------------------------------- PTX glue
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
#ifdef ZO2_MBAR_WATCHDOG
// diagnostic build (tools/build_variant.py ... -DZO2_MBAR_WATCHDOG): a wait
// that has not completed after 5 s reports where it is stuck and traps
__device__ __forceinline__ uint64_t wd_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __noinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  uint32_t ok = 0;
  const uint64_t t0 = wd_now();
  for (uint64_t it = 0; !ok; ++it) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (!ok && (it & 1023) == 1023 && wd_now() - t0 > 5000000000ull) {
      printf("ZO2 mbarrier watchdog: block (%d,%d,%d) thread %d smem 0x%x parity %u\n",
             blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x, smem_u32(b), parity);
      __trap();
    }
  }
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
#endif
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *tm, uint64_t *bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)tm), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
        "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// L2-aware tile raster.  Tile r of a problem -> (mt, nt), visiting groups of
// `gm` M-tiles n-major inside a group: the ~#SM tiles in flight at any time
// then touch about gm A panels and in_flight / gm B panels, instead of one
// or two A panels and EVERY B panel of the problem (row-major order).  With
// production shapes both operands exceed L2 (OPT-30B mlp_out: 32 x 28 tiles
// of 14.7 MB panels), so what L2 saves is exactly this in-flight sharing.
__device__ __forceinline__ void tile_mn(uint32_t r, uint32_t tiles_m, uint32_t tiles_n,
                                        uint32_t gm, uint32_t &mt, uint32_t &nt) {
  const uint32_t per_group = gm * tiles_n;
  const uint32_t g = r / per_group, first = g * gm;
  const uint32_t rows = tiles_m - first < gm ? tiles_m - first : gm;
  const uint32_t q = r - g * per_group;
  mt = first + q % rows;
  nt = q / rows;
}
#ifndef ZO2_GEMM_GROUP_M
#define ZO2_GEMM_GROUP_M 12  // 1-CTA kernel: 148 tiles in flight ~ 12 x 12
#endif
#ifndef ZO2_GEMM2_DYNAMIC
#define ZO2_GEMM2_DYNAMIC 1  // CTA-pair kernel: dynamic tile scheduler (k_gemm2)
#endif
#ifndef ZO2_GEMM2_GROUP_M
#define ZO2_GEMM2_GROUP_M 8  // CTA-pair kernel: 74 tiles in flight ~ 8 x 9
#endif
// raster group heights ([0] 1-CTA, [1] pair); 0 = automatic (group_auto),
// zo2_set_gemm_raster overrides
uint32_t g_group_m[2] = {0, 0};
#ifndef ZO2_GEMM_B_RESIDENT_MB
#define ZO2_GEMM_B_RESIDENT_MB 80
#endif
// Automatic group height: when the whole B operand (weights, N x K x 2 B x
// planes) fits in L2 with room to spare, row-major order (height 1) streams
// A once and keeps B resident (OPT-1.3B mlp_out, bf16x3: 1.66 -> 1.38 GB of
// DRAM per launch); otherwise the square-window height.
inline uint32_t group_auto(uint32_t set, uint32_t N, uint32_t K, bool split, uint32_t square) {
  if (set) return set;
  const uint64_t b_bytes = (uint64_t)N * K * 2u * (split ? 2u : 1u);
  return b_bytes <= ((uint64_t)ZO2_GEMM_B_RESIDENT_MB << 20) ? 1u : square;
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// Instruction descriptor: bf16 x bf16 -> f32, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752440f));
}

template <int BN, bool SPLIT>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = (SPLIT ? 2 : 1) * (A_BYTES + B_BYTES);
  static constexpr int STAGES = (ZO2_GEMM_SMEM_KB * 1024) / STAGE_BYTES > 6 ? 6 : (ZO2_GEMM_SMEM_KB * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

// Cross-entropy partials are emitted per CE_W output columns whatever the
// tile width, so the partial count ceil(N / CE_W) is kernel independent.
constexpr int CE_W = 128;

// Epilogue of one accumulator row segment: this thread owns output row `row`
// and columns [n0, n0 + BN) held in TMEM at column offset tbase.
template <int BN, bool SPLIT, int EPI>
__device__ __forceinline__ void epilogue_tile(const GemmArgs &args, uint32_t p, uint32_t row,
                                              uint32_t n0, uint32_t tbase) {
  const uint32_t M = args.M, N = args.N;
  float run_max = -INFINITY, run_sum = 0.f, tgt = -INFINITY;
  int64_t target = -1;
  if (EPI == ZO2_EPI_CE && row < M) target = args.targets[p][row];
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t v[32];
    tmem_ld32(tbase + (uint32_t)c0, v);  // warp-collective: every lane executes it
    const uint32_t col0 = n0 + (uint32_t)c0;
    if (row < M && col0 < N) {
      if (EPI == ZO2_EPI_CE) {
        float cm = -INFINITY;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < N) cm = fmaxf(cm, __uint_as_float(v[j]));
        const float nm = fmaxf(run_max, cm);
        float s = run_sum * expf(run_max - nm);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < N) s += expf(__uint_as_float(v[j]) - nm);
        run_sum = s;
        run_max = nm;
        if (target >= (int64_t)col0 && target < (int64_t)col0 + 32 && target < (int64_t)N) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if ((int64_t)col0 + j == target) tgt = __uint_as_float(v[j]);
        }
      } else {
        const float *bias = args.bias[p];
        float x[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          x[j] = __uint_as_float(v[j]);
          if (bias && col0 + j < N) x[j] += bias[col0 + j];
        }
        const bool full_chunk = (col0 + 32 <= N) && (N % 4 == 0);
        if (EPI == ZO2_EPI_STORE || EPI == ZO2_EPI_RESIDUAL) {
          float *cp = (float *)args.c[p] + (uint64_t)row * N + col0;
          if (full_chunk) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              float4 o = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
              if (EPI == ZO2_EPI_RESIDUAL) {
                const float4 h = *(const float4 *)(cp + j);
                o.x += h.x; o.y += h.y; o.z += h.z; o.w += h.w;
              }
              *(float4 *)(cp + j) = o;
            }
          } else {
            for (int j = 0; j < 32 && col0 + j < N; ++j)
              cp[j] = (EPI == ZO2_EPI_RESIDUAL) ? cp[j] + x[j] : x[j];
          }
        } else {  // GELU / OPERAND -> bf16 operand planes
          __nv_bfloat16 *hp = (__nv_bfloat16 *)args.c[p] + (uint64_t)row * N + col0;
          __nv_bfloat16 *lp =
              SPLIT ? (__nv_bfloat16 *)args.c_lo[p] + (uint64_t)row * N + col0 : nullptr;
          __align__(16) __nv_bfloat16 hv[32], lv[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float g = EPI == ZO2_EPI_GELU ? gelu_erf(x[j]) : x[j];
            hv[j] = __float2bfloat16_rn(g);
            lv[j] = __float2bfloat16_rn(g - __bfloat162float(hv[j]));
          }
          if (full_chunk && (N % 8 == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              *(uint4 *)(hp + j) = *(const uint4 *)(hv + j);
              if (SPLIT) *(uint4 *)(lp + j) = *(const uint4 *)(lv + j);
            }
          } else {
            for (int j = 0; j < 32 && col0 + j < N; ++j) {
              hp[j] = hv[j];
              if (SPLIT) lp[j] = lv[j];
            }
          }
        }
      }
    }
    // end of a CE_W-column chunk that holds at least one valid column
    if (EPI == ZO2_EPI_CE && ((c0 + 32) % CE_W == 0) && row < M &&
        col0 + 32 - CE_W < N) {
      const uint32_t n_ce = (N + CE_W - 1) / CE_W;
      float *o = args.ce_part[p] + ((uint64_t)row * n_ce + (col0 / CE_W)) * 3;
      o[0] = run_max;
      o[1] = run_sum;
      o[2] = tgt;
      run_max = -INFINITY;
      run_sum = 0.f;
      tgt = -INFINITY;
    }
  }
}

template <int BN, bool SPLIT, int EPI>
__global__ void __launch_bounds__(NUM_THREADS, 1) k_gemm(const __grid_constant__ GemmArgs args) {
  using C = Cfg<BN, SPLIT>;
  extern __shared__ uint8_t smem_raw[];
  // aligned by offset, not through an integer cast: the pointer stays in the
  // shared window, so plain loads/stores through it compile to LDS/STS
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *full = (uint64_t *)(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *empty = full + C::STAGES;
  uint64_t *tfull = empty + C::STAGES;
  uint64_t *tempty = tfull + 2;
  uint64_t *qfull = tempty + 2;   // tile-id ring (dynamic scheduler -> MMA/epilogue)
  uint64_t *qempty = qfull + 4;
  uint32_t *qtile = (uint32_t *)(qempty + 4);
  uint32_t *tmem_slot = qtile + 4;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t M = args.M, N = args.N, K = args.K;
  const uint32_t tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const uint32_t tiles = tiles_m * tiles_n * (uint32_t)args.batch;
  const uint32_t kblocks = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    for (int q = 0; q < 4; ++q) {
      mbar_init(&qfull[q], 1);
      mbar_init(&qempty[q], 5);  // MMA warp + 4 epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    for (int p = 0; p < args.batch; ++p)
      for (int j = 0; j < 4; ++j)
        if (SPLIT || (j & 1) == 0)
          asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&args.tm[p][j]) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"((uint32_t)C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      // dynamic tile scheduler: CTAs that start late (SM shared with the
      // prepare lane's K2) simply take fewer tiles
      int stage = 0;
      uint32_t phase = 0;
      for (uint32_t it = 0;; ++it) {
        const int qs = it & 3;
        mbar_wait(&qempty[qs], ((it >> 2) & 1) ^ 1);
        const uint32_t t = atomicAdd(args.tile_ctr, 1u);
        qtile[qs] = t;
        mbar_arrive(&qfull[qs]);
        if (t >= tiles) break;
        const uint32_t p = t / (tiles_m * tiles_n);
        uint32_t mt, nt;
        tile_mn(t % (tiles_m * tiles_n), tiles_m, tiles_n, args.group_m, mt, nt);
        const int m0 = (int)(mt * BM), n0 = (int)(nt * BN);
        for (uint32_t kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t *st = smem + stage * C::STAGE_BYTES;
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          const int kx = (int)(kb * BK);
          tma_load_2d(st, &args.tm[p][0], &full[stage], kx, m0);
          tma_load_2d(st + C::A_BYTES, &args.tm[p][2], &full[stage], kx, n0);
          if (SPLIT) {
            tma_load_2d(st + C::A_BYTES + C::B_BYTES, &args.tm[p][1], &full[stage], kx, m0);
            tma_load_2d(st + 2 * C::A_BYTES + C::B_BYTES, &args.tm[p][3], &full[stage], kx, n0);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_bf16(BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (uint32_t it = 0;; ++it) {
      const int qs = it & 3;
      mbar_wait(&qfull[qs], (it >> 2) & 1);
      const uint32_t t = qtile[qs];
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[qs]);
      if (t >= tiles) break;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + (uint32_t)(acc * BN);
      for (uint32_t kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
          const uint32_t sal = sb + C::B_BYTES;
          const uint32_t sbl = sal + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint32_t koff = (uint32_t)k * 32;
            const uint64_t da = sw128_desc(sa + koff), db = sw128_desc(sb + koff);
            tc_mma(d, da, db, idesc, (kb | (uint32_t)k) != 0);
            if (SPLIT) {
              tc_mma(d, da, sw128_desc(sbl + koff), idesc, 1u);
              tc_mma(d, sw128_desc(sal + koff), db, idesc, 1u);
            }
          }
          tc_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) tc_commit(&tfull[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..5)
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (uint32_t it = 0;; ++it) {
      const int qs = it & 3;
      mbar_wait(&qfull[qs], (it >> 2) & 1);
      const uint32_t t = qtile[qs];
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[qs]);
      if (t >= tiles) break;
      const uint32_t p = t / (tiles_m * tiles_n);
      uint32_t mt, nt;
      tile_mn(t % (tiles_m * tiles_n), tiles_m, tiles_n, args.group_m, mt, nt);
      const uint32_t m0 = mt * BM, n0 = nt * BN;
      const uint32_t row = m0 + quad * 32 + lane;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * BN);
      epilogue_tile<BN, SPLIT, EPI>(args, p, row, n0, tbase);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // the producer (thread 0) made its last tile fetch before this point; the
    // last CTA out resets the counter pair for the next launch on this slot
    __threadfence();
    if (atomicAdd(args.tile_ctr + 1, 1u) == gridDim.x - 1) {
      atomicExch(args.tile_ctr, 0u);
      atomicExch(args.tile_ctr + 1, 0u);
    }
  }
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)C::TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------- 2-SM variant
// A CTA pair (cluster of 2 on one TPC) computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2: each CTA stages its own 128 rows of A and 128
// rows of B, the leader issues the MMAs for the pair and each CTA's TMEM holds
// its 128 output rows.  Per SM this moves 32 KB of operands per 64-deep
// k-block instead of 48 KB for the same MMA work, which is what lifts the
// GEMM off the L2->SM bandwidth ceiling of the 1-CTA 128x256 tile.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void *dst, const CUtensorMap *tm, uint64_t *bar,
                                                 int x, int y) {
  // completion bytes go to the leader CTA's barrier (peer bit cleared)
  const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)tm), "r"(mbar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tc_mma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit2_mc(uint64_t *bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t *bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_rank(uint64_t *bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
__device__ __forceinline__ void st_rank_u32(uint32_t *p, uint32_t v, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(p)), "r"(rank));
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(remote), "r"(v) : "memory");
}
// parity wait with cluster-scope acquire (the phase was completed by, or
// orders data written by, the other CTA of the pair)
__device__ __forceinline__ void mbar_wait_cl(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__host__ __device__ constexpr uint32_t idesc_bf16_m256(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

template <bool SPLIT>
struct Cfg2 {
  static constexpr int BN = 256;          // pair tile N (each CTA stages BN/2 rows of B)
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;
  static constexpr int STAGE_BYTES = (SPLIT ? 2 : 1) * (A_BYTES + B_BYTES);
  static constexpr int STAGES = (ZO2_GEMM_SMEM_KB * 1024) / STAGE_BYTES > 6 ? 6 : (ZO2_GEMM_SMEM_KB * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <bool SPLIT, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    k_gemm2(const __grid_constant__ GemmArgs args) {
  using C = Cfg2<SPLIT>;
  constexpr int BN = C::BN;
  extern __shared__ uint8_t smem_raw[];
  // aligned by offset, not through an integer cast: the pointer stays in the
  // shared window, so plain loads/stores through it compile to LDS/STS
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *full = (uint64_t *)(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *empty = full + C::STAGES;
  uint64_t *tfull = empty + C::STAGES;
  uint64_t *tempty = tfull + 2;
  uint64_t *qfull = tempty + 2;   // tile-id ring, written by the leader's producer
  uint64_t *qempty = qfull + 4;   // (leader's copy is the one used)
  uint32_t *qtile = (uint32_t *)(qempty + 4);
  uint32_t *tmem_slot = qtile + 4;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const uint32_t M = args.M, N = args.N, K = args.K;
  const uint32_t tiles_m = (M + 2 * BM - 1) / (2 * BM), tiles_n = (N + BN - 1) / BN;
  const uint32_t tiles = tiles_m * tiles_n * (uint32_t)args.batch;
  const uint32_t kblocks = (K + BK - 1) / BK;
#if !ZO2_GEMM2_DYNAMIC
  const uint32_t cid = blockIdx.x / 2, ncl = gridDim.x / 2;
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps in each of the 2 CTAs
    }
    for (int q = 0; q < 4; ++q) {
      mbar_init(&qfull[q], 1);
      // consumers of a tile id: the leader's MMA warp, the peer's producer
      // and the 4 epilogue warps of each CTA
      mbar_init(&qempty[q], 10);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    for (int p = 0; p < args.batch; ++p)
      for (int j = 0; j < 4; ++j)
        if (SPLIT || (j & 1) == 0)
          asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&args.tm[p][j]) : "memory");
  }
  // Both CTAs of the pair meet BEFORE the pair allocation (and relinquish
  // after it, below).  Without this barrier a peer whose warps start late --
  // its SM still shared with K2 CTAs, which only fit beside a GEMM CTA with a
  // staging budget below ~190 KB -- issued its tcgen05.alloc.cta_group::2
  // after the leader's had completed, and that alloc never returned: cuda-gdb
  // on the hung step showed the leader at the post-alloc cluster barrier,
  // the peer's warp 1 spinning inside tcgen05.alloc and no other CTA on
  // either SM (tools/gpu_r2_hang_gdb.sh).
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"((uint32_t)C::TMEM_COLS)
                 : "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  // Relinquish only once BOTH CTAs of the pair have allocated.  The pair's
  // relinquish_alloc_permit.cta_group::2 issued while the peer's alloc is
  // still pending leaves that alloc waiting forever: with a smaller staging
  // budget K2 CTAs share the SMs, the peer's warps start late, and the
  // leader used to get there first (cuda-gdb on the hung step: leader at the
  // cluster barrier, peer warp 1 spinning inside tcgen05.alloc,
  // tools/gpu_r2_hang_gdb.sh).
  if (warp == 1)
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  // Tile sequence.  Dynamic (default): the leader's producer takes tiles from
  // a global counter in raster order and hands each id to both CTAs through
  // a 4-deep ring (qtile/qfull in each CTA, qempty in the leader), so the
  // ~74 tiles in flight stay a contiguous window of the L2-aware raster even
  // when pairs start late (SMs still running K2) or run at different speeds;
  // a static round-robin assignment let those drifts accumulate over the
  // ~100 tile waves of the OPT-175B GEMMs and lost the L2 reuse.
#if ZO2_GEMM2_DYNAMIC
  auto fetch_tile = [&](uint32_t it) -> uint32_t {  // leader producer (one thread)
    const int qs = (int)(it & 3u);
    mbar_wait_cl(&qempty[qs], ((it >> 2) & 1u) ^ 1u);
    const uint32_t t = atomicAdd(args.tile_ctr, 1u);
    qtile[qs] = t;
    st_rank_u32(&qtile[qs], t, 1);
    mbar_arrive(&qfull[qs]);
    mbar_arrive_rank(&qfull[qs], 1);
    return t;
  };
  auto take_tile = [&](uint32_t it, bool warp_wide) -> uint32_t {  // every consumer
    const int qs = (int)(it & 3u);
    mbar_wait_cl(&qfull[qs], (it >> 2) & 1u);
    const uint32_t t = qtile[qs];
    if (warp_wide) __syncwarp();
    if (!warp_wide || lane == 0) mbar_arrive_rank(&qempty[qs], 0);
    return t;
  };
#endif

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
#if ZO2_GEMM2_DYNAMIC
      for (uint32_t it = 0;; ++it) {
        const uint32_t t = leader ? fetch_tile(it) : take_tile(it, false);
        if (t >= tiles) break;
#else
      for (uint32_t t = cid; t < tiles; t += ncl) {
#endif
        const uint32_t p = t / (tiles_m * tiles_n);
        uint32_t mt, nt;
        tile_mn(t % (tiles_m * tiles_n), tiles_m, tiles_n, args.group_m, mt, nt);
        const int m0 = (int)(mt * 2 * BM + rank * BM);
        const int n0 = (int)(nt * BN + rank * (BN / 2));
        for (uint32_t kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t *st = smem + stage * C::STAGE_BYTES;
          if (leader) mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
          const int kx = (int)(kb * BK);
          tma_load_2d_pair(st, &args.tm[p][0], &full[stage], kx, m0);
          tma_load_2d_pair(st + C::A_BYTES, &args.tm[p][2], &full[stage], kx, n0);
          if (SPLIT) {
            tma_load_2d_pair(st + C::A_BYTES + C::B_BYTES, &args.tm[p][1], &full[stage], kx, m0);
            tma_load_2d_pair(st + 2 * C::A_BYTES + C::B_BYTES, &args.tm[p][3], &full[stage], kx,
                             n0);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader CTA only)
    if (leader) {
      constexpr uint32_t idesc = idesc_bf16_m256(BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
#if ZO2_GEMM2_DYNAMIC
      for (uint32_t it = 0;; ++it) {
        const uint32_t t = take_tile(it, true);
        if (t >= tiles) break;
#else
      for (uint32_t t = cid; t < tiles; t += ncl) {
#endif
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * BN);
        for (uint32_t kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
            const uint32_t sb = sa + C::A_BYTES;
            const uint32_t sal = sb + C::B_BYTES;
            const uint32_t sbl = sal + C::A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint32_t koff = (uint32_t)k * 32;
              const uint64_t da = sw128_desc(sa + koff), db = sw128_desc(sb + koff);
              tc_mma2(d, da, db, idesc, (kb | (uint32_t)k) != 0);
              if (SPLIT) {
                tc_mma2(d, da, sw128_desc(sbl + koff), idesc, 1u);
                tc_mma2(d, sw128_desc(sal + koff), db, idesc, 1u);
              }
            }
            tc_commit2_mc(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) tc_commit2_mc(&tfull[acc], 0x3);
        __syncwarp();
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------ epilogue (both CTAs, own 128 rows)
    const int quad = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
#if ZO2_GEMM2_DYNAMIC
    for (uint32_t it = 0;; ++it) {
      const uint32_t t = take_tile(it, true);
      if (t >= tiles) break;
#else
    for (uint32_t t = cid; t < tiles; t += ncl) {
#endif
      const uint32_t p = t / (tiles_m * tiles_n);
      uint32_t mt, nt;
      tile_mn(t % (tiles_m * tiles_n), tiles_m, tiles_n, args.group_m, mt, nt);
      const uint32_t m0 = mt * 2 * BM + rank * BM, n0 = nt * BN;
      const uint32_t row = m0 + quad * 32 + lane;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * BN);
      epilogue_tile<BN, SPLIT, EPI>(args, p, row, n0, tbase);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  __syncthreads();
#if ZO2_GEMM2_DYNAMIC
  if (threadIdx.x == 0) {
    // every leader fetched its last tile id before its CTA got here: the last
    // CTA out resets the counter pair for the next launch on this slot
    __threadfence();
    if (atomicAdd(args.tile_ctr + 1, 1u) == gridDim.x - 1) {
      atomicExch(args.tile_ctr, 0u);
      atomicExch(args.tile_ctr + 1, 0u);
    }
  }
#endif
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)C::TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::mutex g_mu;

struct MapKey {
  const void *p;
  uint32_t rows, k, box_rows;
  bool operator==(const MapKey &o) const {
    return p == o.p && rows == o.rows && k == o.k && box_rows == o.box_rows;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey &k) const {
    return std::hash<const void *>()(k.p) ^ ((size_t)k.rows * 1315423911u) ^
           ((size_t)k.k << 20) ^ k.box_rows;
  }
};
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

int get_encoder() {
  if (g_encode) return ZO2_OK;
  cudaDriverEntryPointQueryResult q;
  void *fn = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
    return zo2_set_error(ZO2_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  return ZO2_OK;
}

int make_map(const void *ptr, uint32_t rows, uint32_t k, uint32_t box_rows, CUtensorMap *out) {
  MapKey key{ptr, rows, k, box_rows};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return ZO2_OK;
    }
  }
  int rc = get_encoder();
  if (rc) return rc;
  cuuint64_t dims[2] = {k, rows};
  cuuint64_t strides[1] = {(cuuint64_t)k * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char msg[160];
    snprintf(msg, sizeof(msg), "cuTensorMapEncodeTiled failed (%d) rows=%u k=%u", (int)r, rows, k);
    return zo2_set_error(ZO2_E_ARG, msg);
  }
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_maps.size() > 4096) g_maps.clear();
  g_maps[key] = *out;
  return ZO2_OK;
}

int g_num_sms = 0;
constexpr unsigned kCtrSlots = 256;

// One self-resetting (next tile, CTAs finished) counter pair per launch,
// rotating over kCtrSlots pairs per device: a pair is reused 256 GEMM
// launches later, long after the stream-ordered launch that used it ended.
int tile_counter(unsigned int **out) {
  static unsigned int *ctrs[64] = {nullptr};
  static unsigned seq[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return zo2_set_error(ZO2_E_ARG, "zo2_gemm: device id out of range");
  std::lock_guard<std::mutex> lk(g_mu);
  if (!ctrs[dev]) {
    cudaError_t e = cudaMalloc(&ctrs[dev], 2 * kCtrSlots * sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaMemset(ctrs[dev], 0, 2 * kCtrSlots * sizeof(unsigned int));
    if (e != cudaSuccess) return zo2_set_cuda_error(e);
  }
  *out = ctrs[dev] + 2 * (seq[dev]++ % kCtrSlots);
  return ZO2_OK;
}

template <int BN, bool SPLIT, int EPI>
int launch(const GemmArgs &a, cudaStream_t s) {
  using C = Cfg<BN, SPLIT>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm<BN, SPLIT, EPI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return zo2_set_cuda_error(e);
    attr_set = true;
  }
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  const uint32_t tiles = ((a.M + BM - 1) / BM) * ((a.N + BN - 1) / BN) * (uint32_t)a.batch;
  const unsigned grid = tiles < (uint32_t)g_num_sms ? tiles : (unsigned)g_num_sms;
  GemmArgs b = a;
  if (int rc = tile_counter(&b.tile_ctr)) return rc;
  b.group_m = group_auto(g_group_m[0], a.N, a.K, SPLIT, ZO2_GEMM_GROUP_M);
  k_gemm<BN, SPLIT, EPI><<<grid, NUM_THREADS, C::SMEM, s>>>(b);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

template <int BN, bool SPLIT>
int dispatch_epi(const GemmArgs &a, int epi, cudaStream_t s) {
  switch (epi) {
    case ZO2_EPI_STORE: return launch<BN, SPLIT, ZO2_EPI_STORE>(a, s);
    case ZO2_EPI_RESIDUAL: return launch<BN, SPLIT, ZO2_EPI_RESIDUAL>(a, s);
    case ZO2_EPI_GELU: return launch<BN, SPLIT, ZO2_EPI_GELU>(a, s);
    case ZO2_EPI_CE: return launch<BN, SPLIT, ZO2_EPI_CE>(a, s);
    case ZO2_EPI_OPERAND: return launch<BN, SPLIT, ZO2_EPI_OPERAND>(a, s);
    default: return zo2_set_error(ZO2_E_ARG, "zo2_gemm: unknown epilogue");
  }
}

template <bool SPLIT, int EPI>
int launch2(const GemmArgs &a, cudaStream_t s) {
  using C = Cfg2<SPLIT>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm2<SPLIT, EPI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return zo2_set_cuda_error(e);
    attr_set = true;
  }
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  const uint32_t tiles =
      ((a.M + 2 * BM - 1) / (2 * BM)) * ((a.N + C::BN - 1) / C::BN) * (uint32_t)a.batch;
  const uint32_t pairs = tiles < (uint32_t)(g_num_sms / 2) ? tiles : (uint32_t)(g_num_sms / 2);
  GemmArgs b = a;
  if (int rc = tile_counter(&b.tile_ctr)) return rc;
  b.group_m = group_auto(g_group_m[1], a.N, a.K, SPLIT, ZO2_GEMM2_GROUP_M);
  k_gemm2<SPLIT, EPI><<<2 * pairs, NUM_THREADS, C::SMEM, s>>>(b);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

template <bool SPLIT>
int dispatch_epi2(const GemmArgs &a, int epi, cudaStream_t s) {
  switch (epi) {
    case ZO2_EPI_STORE: return launch2<SPLIT, ZO2_EPI_STORE>(a, s);
    case ZO2_EPI_RESIDUAL: return launch2<SPLIT, ZO2_EPI_RESIDUAL>(a, s);
    case ZO2_EPI_GELU: return launch2<SPLIT, ZO2_EPI_GELU>(a, s);
    case ZO2_EPI_CE: return launch2<SPLIT, ZO2_EPI_CE>(a, s);
    case ZO2_EPI_OPERAND: return launch2<SPLIT, ZO2_EPI_OPERAND>(a, s);
    default: return zo2_set_error(ZO2_E_ARG, "zo2_gemm: unknown epilogue");
  }
}

int g_variant = 0;  // 0 auto, 1 single-CTA only, 2 CTA pair whenever legal


// ====================================================================== K5 (tcgen05)
// Causal attention of one (q-tile of 128 queries, head, batch) on the 5th-gen
// tensor cores (model.py:273-283):  S = Q K^T -> softmax(S / sqrt(hd)) -> P V.
//   * Q, K, V tiles come straight from the QKV GEMM's bf16 planes ([T, 3d]:
//     q | k | v column blocks) by TMA (128-byte swizzle, 64-column panels);
//     V is consumed MN-major (hd contiguous), so it is never transposed.
//   * S (128 x 128 f32) and O (128 x hd f32) live in TMEM; 4 warps own 32
//     TMEM lanes (= query rows) each and run the softmax from tcgen05.ld.
//   * two passes over the causal key tiles: the first takes the row max (of
//     Qhi Khi in split mode, within ~2^-8 of the full S: exp stays <= ~1), the
//     second computes the full S, writes P = exp(S - max) to shared
//     memory (bf16, swizzled K-major A operand) and accumulates O += P V, so O
//     is never rescaled.  Split (f32-faithful) mode: S = Qh Kh + Qh Kl + Ql Kh,
//     O += Ph Vh + Ph Vl + Pl Vh (~2^-16 relative per product, as the GEMMs).
//   * one thread issues TMA and MMAs; completion is tracked with mbarriers.
struct AttnTcArgs {
  CUtensorMap tq[2];  // qkv hi / lo planes, [T, 3d], box 64 x 128 (query tile)
  CUtensorMap tk[2];  // same planes, box 64 x 64 (key / value tile)
  __nv_bfloat16 *out_hi, *out_lo;
  uint32_t seq, n_heads, dim;
  float scale_log2;   // log2(e) / sqrt(hd)
};

constexpr int ATT_Q = 128;  // queries per CTA (TMEM lanes)
constexpr int ATT_K = 64;   // keys per tile
constexpr int ATT_T = ATT_Q;

// Instruction descriptor: bf16 x bf16 -> f32, M = 128, N = n; b_mn: B MN-major.
__host__ __device__ constexpr uint32_t idesc_bf16_b(int n, bool b_mn) {
  return idesc_bf16(n) | (b_mn ? (1u << 16) : 0u);
}
// MN-major 128B-swizzle descriptor: 8-row K groups 1024 B apart (SBO), 64-element
// MN groups `lbo` bytes apart (LBO).
__device__ __forceinline__ uint64_t sw128_desc_mn(uint32_t saddr, uint32_t lbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int HD, bool SPLIT>
struct AttnTcCfg {
  static constexpr int PL = SPLIT ? 2 : 1;               // planes
  static constexpr int PAN = HD / 64;                    // 64-column panels of hd
  static constexpr int QTILE = ATT_Q * 128;              // one 128-row panel, bytes
  static constexpr int KTILE = ATT_K * 128;              // one 64-row panel
  static constexpr int KV = PL * PAN * KTILE;            // K (or V) tile, all planes
  static constexpr int NS = 2;                           // K/V ring stages
  static constexpr int Q_OFF = 0;
  static constexpr int KV_OFF = Q_OFF + PL * PAN * QTILE;  // stage s: K at +2s*KV, V at +(2s+1)*KV
  static constexpr int BAR_OFF = KV_OFF + NS * 2 * KV;
  static constexpr int SMEM = BAR_OFF + 256 + 6 * 128 * 4 + 1024;
  // TMEM columns (256 per CTA, two CTAs per SM): two S buffers of 64 columns,
  // then O.  P(g) (bf16 pairs: hi in columns 0-31, lo in 32-63) overwrites
  // S(g) in its own buffer, so P is double-buffered along with S.
  static constexpr int SB = 2;
  static constexpr uint32_t T_O = SB * ATT_K;
  static constexpr uint32_t TMEM_COLS = 256;
  static_assert(T_O + HD <= TMEM_COLS, "TMEM budget");
};

__device__ __forceinline__ void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 lanes x 16 consecutive 32-bit columns from 16 registers per thread
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15])
      : "memory");
}

// 8 softmax warps (warp w and w + 4 share TMEM lane quadrant w % 4 = 32 query
// rows and split the 64 columns of S and the hd columns of O) + 1 warp that
// issues TMA and tcgen05.mma; the two sides meet only on mbarriers.  P goes
// to TMEM (tcgen05.st) and is the A operand of P.V straight from there, so
// a CTA needs no P staging in shared memory: two CTAs per SM.
constexpr int ATT_SOFT = 256;
// online softmax: the running max moves only when a row's tile max exceeds it
// by more than 2^ATT_TAU (P values stay <= 2^ATT_TAU, O is rescaled rarely)
constexpr float ATT_TAU = 8.0f;
template <int HD, bool SPLIT>
__global__ void __launch_bounds__(ATT_SOFT + 32, 2) k_attn_tc(const __grid_constant__ AttnTcArgs a) {
  using C = AttnTcCfg<HD, SPLIT>;
  constexpr int NS = C::NS, SB = C::SB;
  extern __shared__ uint8_t smem_raw[];
  // aligned by offset, not through an integer cast: the pointer stays in the
  // shared window, so plain loads/stores through it compile to LDS/STS
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *bar_kv = (uint64_t *)(smem + C::BAR_OFF);  // [NS] tile loaded (TMA)
  uint64_t *bar_s = bar_kv + NS;                       // [SB] S written (MMA commit)
  uint64_t *bar_p = bar_s + SB;                        // [SB] P written into its S buffer (256 arrivals)
  uint64_t *bar_o = bar_p + SB;                        // P.V done (MMA commit)
  uint64_t *bar_kvfree = bar_o + 1;                    // [NS] ring stage read by its MMAs
  uint64_t *bar_done = bar_kvfree + NS;                // every P.V done (one phase)
  uint32_t *tmem_slot = (uint32_t *)(bar_done + 1);
  float *xch = (float *)(smem + C::BAR_OFF + 256);     // [2][2][128] row max, then [2][128] row sum
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // heavy (late) query tiles first
  const uint32_t qt = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int row0 = (int)(b * a.seq + qt * ATT_Q);
  const uint32_t n_kt = (qt + 1) * (ATT_Q / ATT_K);  // causal: key tiles up to the diagonal
  const uint32_t d = a.dim;

  if (threadIdx.x == ATT_SOFT) {
    for (int i = 0; i < NS; ++i) mbar_init(&bar_kv[i], 1);
    for (int i = 0; i < SB; ++i) {
      mbar_init(&bar_s[i], 1);
      mbar_init(&bar_p[i], ATT_SOFT);
    }
    mbar_init(bar_o, 1);
    for (int i = 0; i < NS; ++i) mbar_init(&bar_kvfree[i], 1);
    mbar_init(bar_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int p = 0; p < C::PL; ++p) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&a.tq[p]) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&a.tk[p]) : "memory");
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_o = tmem + C::T_O;

  // Barrier phases.  Every wait below is on a phase that cannot be two ahead
  // of it (a parity wait trailing its barrier by two phases would hang):
  //   bar_s[g%2] phase g/2: S(g+2) is issued only after P.V(g) completed,
  //     which needs P(g), which the softmax writes after reading S(g);
  //   bar_p[g%2] phase g/2: P(g+2) needs S(g+2), issued after the MMA thread
  //     saw P(g) (P.V(g) issued) and P.V(g) completed;
  //   bar_o phase j, waited at tile j+1 (softmax, only to rescale O) and
  //     before S(j+2) (MMA thread): P.V(j-1) is complete by then (S(j+1)
  //     waited for it) and P.V(j+1) needs P(j+1), not yet written.  The
  //     epilogue cannot wait on bar_o (P.V(n-2) may still run, so a parity
  //     wait for phase n-1 could be satisfied by phase n-3): it waits for
  //     bar_done, committed once after the last P.V.
  if (warp == ATT_SOFT / 32) {
    // ================================================ TMA + MMA issue (one thread)
    if (lane == 0) {
      const uint32_t sq = smem_u32(smem + C::Q_OFF), skv = smem_u32(smem + C::KV_OFF);
      auto load_tile = [&](uint32_t g) {
        const bool with_q = g == 0;
        const int st = (int)(g % NS);
        const uint32_t bytes = 2u * (uint32_t)C::KV +
                               (with_q ? (uint32_t)(C::PL * C::PAN * C::QTILE) : 0u);
        mbar_expect_tx(&bar_kv[st], bytes);
        const int krow = (int)(b * a.seq + g * ATT_K);
        uint8_t *kb = smem + C::KV_OFF + 2 * st * C::KV;
        for (int p = 0; p < C::PL; ++p)
          for (int c = 0; c < C::PAN; ++c) {
            const int o = (p * C::PAN + c) * C::KTILE;
            if (with_q)
              tma_load_2d(smem + C::Q_OFF + (p * C::PAN + c) * C::QTILE, &a.tq[p], &bar_kv[st],
                          (int)(h * HD + 64 * c), row0);
            tma_load_2d(kb + o, &a.tk[p], &bar_kv[st], (int)(d + h * HD + 64 * c), krow);
            tma_load_2d(kb + C::KV + o, &a.tk[p], &bar_kv[st], (int)(2 * d + h * HD + 64 * c),
                        krow);
          }
      };
      // S[g % SB] = Q K(g)^T (3 passes split); K-major A and B
      auto issue_qk = [&](uint32_t g) {
        constexpr uint32_t id = idesc_bf16_b(ATT_K, false);
        const uint32_t ts = tmem + (g % SB) * ATT_K;
        const uint32_t sk = skv + (uint32_t)(2 * (int)(g % NS) * C::KV);
        for (int ks = 0; ks < HD / 16; ++ks) {
          const uint32_t qo = (uint32_t)((ks / 4) * C::QTILE + (ks % 4) * 32);
          const uint32_t ko = (uint32_t)((ks / 4) * C::KTILE + (ks % 4) * 32);
          const uint64_t qa = sw128_desc(sq + qo), kd = sw128_desc(sk + ko);
          tc_mma(ts, qa, kd, id, ks != 0);
          if (SPLIT) {
            tc_mma(ts, qa, sw128_desc(sk + C::PAN * C::KTILE + ko), id, 1u);
            tc_mma(ts, sw128_desc(sq + C::PAN * C::QTILE + qo), kd, id, 1u);
          }
        }
        tc_commit(&bar_s[g % SB]);
      };
      // O += P(g) V(g): A = P [128 q x 64 keys] in S buffer g % SB (hi columns
      // 0-31, lo 32-63), B = V [64 keys x hd] MN-major
      auto issue_pv = [&](uint32_t g) {
        constexpr uint32_t id = idesc_bf16_b(HD, true);
        constexpr uint32_t vlbo = (uint32_t)C::KTILE;  // next 64 hd columns: next panel
        const uint32_t sv = skv + (uint32_t)((2 * (int)(g % NS) + 1) * C::KV);
        const uint32_t tp = tmem + (g % SB) * ATT_K;
        for (int ks = 0; ks < ATT_K / 16; ++ks) {
          const uint32_t voff = (uint32_t)(ks * 16 * 128);  // 16 keys x 128 B
          const uint32_t pa = tp + (uint32_t)(ks * 8);       // 16 keys = 8 columns
          const uint64_t vb = sw128_desc_mn(sv + voff, vlbo);
          tc_mma_ts(t_o, pa, vb, id, (g | (uint32_t)ks) != 0);
          if (SPLIT) {
            tc_mma_ts(t_o, pa, sw128_desc_mn(sv + C::PAN * C::KTILE + voff, vlbo), id, 1u);
            tc_mma_ts(t_o, pa + ATT_K / 2, vb, id, 1u);
          }
        }
        tc_commit(bar_o);
      };

      for (uint32_t g = 0; g < (uint32_t)NS && g < n_kt; ++g) load_tile(g);
      mbar_wait(&bar_kv[0], 0);
      tc_fence_after();
      issue_qk(0);
      for (uint32_t g = 0; g < n_kt; ++g) {
        // refill the ring stage of tile g - 1 (read by S(g - 1) and P.V(g - 1))
        if (g >= 1 && g - 1 + NS < n_kt) {
          const uint32_t gp = g - 1;
          mbar_wait(&bar_kvfree[gp % NS], (gp / NS) & 1u);
          load_tile(gp + NS);
        }
        // S(g + 1) next: needs K(g + 1) and its buffer free of P(g - 1)
        if (g + 1 < n_kt) {
          const uint32_t gn = g + 1;
          mbar_wait(&bar_kv[gn % NS], (gn / NS) & 1u);
          if (gn >= (uint32_t)SB) mbar_wait(bar_o, (gn - SB) & 1u);
          tc_fence_after();
          issue_qk(gn);
        } else if (g >= 1) {
          // last tile: observe phase g - 1 of bar_o before committing phase g,
          // so no phase of the barrier completes unobserved by this thread
          // (compute-sanitizer synccheck "missing wait"); P.V(g - 1) and P.V(g)
          // accumulate into the same TMEM columns and serialise anyway
          mbar_wait(bar_o, (g - 1) & 1u);
        }
        // P.V(g) once the softmax stored P(g)
        mbar_wait(&bar_p[g % SB], (g / SB) & 1u);
        tc_fence_after();
        issue_pv(g);
        tc_commit(&bar_kvfree[g % NS]);
      }
      tc_commit(bar_done);
    }
  } else {
    // ================================================ softmax warps
    const int quad = warp & 3, half = warp >> 2;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const int r = quad * 32 + lane;  // query row within the tile (TMEM lane)
    const int c0 = 32 * half;        // this warp's 32 columns of S
    float mscaled = -INFINITY, lsum = 0.f;
    for (uint32_t g = 0; g < n_kt; ++g) {
      const int lim = (int)(qt * ATT_Q) + r - (int)(g * ATT_K) - c0;  // visible: i <= lim
      const uint32_t ts = tmem + (g % SB) * ATT_K;
      mbar_wait(&bar_s[g % SB], (g / SB) & 1u);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(ts + lane_base + (uint32_t)c0, v);
      float mt = -INFINITY;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i <= lim) mt = fmaxf(mt, __uint_as_float(v[i]));
      // the two warps of a quadrant hold the halves of the same rows; the
      // barrier also orders both warps' S reads before either overwrites the
      // buffer with P
      float *slot = xch + (g & 1u) * 256;
      slot[half * 128 + r] = mt;
      asm volatile("bar.sync %0, 64;" ::"r"(2 + quad) : "memory");
      mt = fmaxf(slot[r], slot[128 + r]) * a.scale_log2;
      float alpha = 1.f;  // O and l rescale of this row
      if (mt > mscaled + ATT_TAU) {
        alpha = ex2f(mscaled - mt);
        mscaled = mt;
        lsum *= alpha;
      }
      float pv[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float e = (i <= lim) ? ex2f(__uint_as_float(v[i]) * a.scale_log2 - mscaled) : 0.f;
        pv[i] = e;
        lsum += e;
      }
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const __nv_bfloat162 hv = __floats2bfloat162_rn(pv[2 * e], pv[2 * e + 1]);
        hi[e] = *reinterpret_cast<const uint32_t *>(&hv);
        if (SPLIT) {
          const __nv_bfloat162 lv = __floats2bfloat162_rn(pv[2 * e] - __low2float(hv),
                                                          pv[2 * e + 1] - __high2float(hv));
          lo[e] = *reinterpret_cast<const uint32_t *>(&lv);
        }
      }
      // a row's max moved: O(g - 1) must be final before it is rescaled (and
      // P.V(g) is not issued before this warp's P(g) arrives)
      if (g >= 1 && __any_sync(0xffffffffu, alpha != 1.f)) {
        mbar_wait(bar_o, (g - 1) & 1u);
        tc_fence_after();
#pragma unroll 1
        for (int o0 = half * (HD / 2); o0 < (half + 1) * (HD / 2); o0 += 32) {
          uint32_t w[32];
          tmem_ld32(t_o + lane_base + (uint32_t)o0, w);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            uint32_t x[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] = __float_as_uint(__uint_as_float(w[16 * q + e]) * alpha);
            tmem_st16(t_o + lane_base + (uint32_t)(o0 + 16 * q), x);
          }
        }
      }
      tmem_st16(ts + lane_base + (uint32_t)(c0 / 2), hi);
      if (SPLIT) tmem_st16(ts + lane_base + (uint32_t)(ATT_K / 2 + c0 / 2), lo);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&bar_p[g % SB]);
    }
    // ---------------------------------------------- epilogue: O / l -> bf16 planes
    xch[512 + half * 128 + r] = lsum;
    mbar_wait(bar_done, 0);  // every P.V done
    tc_fence_after();
    asm volatile("bar.sync 1, %0;" ::"n"(ATT_SOFT) : "memory");
    const float inv = 1.0f / (xch[512 + r] + xch[640 + r]);
    __nv_bfloat16 *oh = a.out_hi + (uint64_t)(row0 + r) * d + h * HD;
    __nv_bfloat16 *ol = SPLIT ? a.out_lo + (uint64_t)(row0 + r) * d + h * HD : nullptr;
#pragma unroll 1
    for (int o0 = half * (HD / 2); o0 < (half + 1) * (HD / 2); o0 += 32) {
      uint32_t w[32];
      tmem_ld32(t_o + lane_base + (uint32_t)o0, w);
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const float x0 = __uint_as_float(w[2 * e]) * inv, x1 = __uint_as_float(w[2 * e + 1]) * inv;
        const __nv_bfloat162 hv = __floats2bfloat162_rn(x0, x1);
        hi[e] = *reinterpret_cast<const uint32_t *>(&hv);
        const __nv_bfloat162 lv = __floats2bfloat162_rn(x0 - __low2float(hv), x1 - __high2float(hv));
        lo[e] = *reinterpret_cast<const uint32_t *>(&lv);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        *(uint4 *)(oh + o0 + 8 * q) = make_uint4(hi[4 * q], hi[4 * q + 1], hi[4 * q + 2], hi[4 * q + 3]);
        if (SPLIT)
          *(uint4 *)(ol + o0 + 8 * q) = make_uint4(lo[4 * q], lo[4 * q + 1], lo[4 * q + 2], lo[4 * q + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(C::TMEM_COLS)
                 : "memory");
}

template <int HD, bool SPLIT>
int launch_attn_tc(const void *qh, const void *ql, uint32_t batch, uint32_t seq, uint32_t nh,
                   void *oh, void *ol, cudaStream_t s) {
  using C = AttnTcCfg<HD, SPLIT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_attn_tc<HD, SPLIT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return zo2_set_cuda_error(e);
    attr = true;
  }
  AttnTcArgs a;
  memset(&a, 0, sizeof(a));
  const uint32_t d = nh * HD, T = batch * seq;
  int rc = make_map(qh, T, 3 * d, (uint32_t)ATT_Q, &a.tq[0]);
  if (!rc) rc = make_map(qh, T, 3 * d, (uint32_t)ATT_K, &a.tk[0]);
  if (!rc && SPLIT) rc = make_map(ql, T, 3 * d, (uint32_t)ATT_Q, &a.tq[1]);
  if (!rc && SPLIT) rc = make_map(ql, T, 3 * d, (uint32_t)ATT_K, &a.tk[1]);
  if (rc) return rc;
  a.out_hi = (__nv_bfloat16 *)oh;
  a.out_lo = (__nv_bfloat16 *)ol;
  a.seq = seq;
  a.n_heads = nh;
  a.dim = d;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  dim3 grid(seq / ATT_Q, nh, batch);
  k_attn_tc<HD, SPLIT><<<grid, ATT_SOFT + 32, C::SMEM, s>>>(a);
  return ZO2_OK;
}
}  // namespace


// tcgen05 attention (K5) for seq % 128 == 0 and head_dim 64 (split or bf16) or
// 128 (bf16); returns ZO2_E_UNSUPPORTED otherwise (the caller falls back).
extern "C" int zo2_attention_tc(const void *qkv_hi, const void *qkv_lo, uint32_t batch,
                                uint32_t seq, uint32_t n_heads, uint32_t head_dim, void *ctx_hi,
                                void *ctx_lo, void *cs) {
  const bool split = qkv_lo != nullptr;
  if (seq % ATT_T != 0 || seq == 0) return ZO2_E_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)cs;
  if (head_dim == 64)
    return split ? launch_attn_tc<64, true>(qkv_hi, qkv_lo, batch, seq, n_heads, ctx_hi, ctx_lo, s)
                 : launch_attn_tc<64, false>(qkv_hi, qkv_lo, batch, seq, n_heads, ctx_hi, ctx_lo, s);
  if (head_dim == 128 && !split)
    return launch_attn_tc<128, false>(qkv_hi, qkv_lo, batch, seq, n_heads, ctx_hi, ctx_lo, s);
  return ZO2_E_UNSUPPORTED;
}

extern "C" int zo2_gemm_tile_n(int split) {
  (void)split;
  return CE_W;  // CE partials are per CE_W columns for every kernel variant
}

extern "C" int zo2_set_gemm_raster(int group_m_cta, int group_m_pair) {
  if (group_m_cta < 0 || group_m_cta > 1024 || group_m_pair < 0 || group_m_pair > 1024)
    return zo2_set_error(ZO2_E_ARG, "zo2_set_gemm_raster: group heights 0 (automatic) or 1..1024");
  g_group_m[0] = (uint32_t)group_m_cta;
  g_group_m[1] = (uint32_t)group_m_pair;
  return ZO2_OK;
}

extern "C" int zo2_set_gemm_variant(int v) {
  if (v < 0 || v > 2) return zo2_set_error(ZO2_E_ARG, "zo2_set_gemm_variant: 0, 1 or 2");
  g_variant = v;
  return ZO2_OK;
}

extern "C" int zo2_gemm(const zo2_gemm_problem *probs, int batch, uint32_t M, uint32_t N,
                        uint32_t K, int epi, void *cs) {
  if (batch < 1 || batch > 2) return zo2_set_error(ZO2_E_ARG, "zo2_gemm: batch must be 1 or 2");
  if (M == 0 || N == 0) return ZO2_OK;
  if (K == 0 || K % 8 != 0) return zo2_set_error(ZO2_E_UNSUPPORTED, "zo2_gemm: K must be a positive multiple of 8");
  const bool split = probs[0].a_lo != nullptr;
  // CTA pair (256 x 256 tiles) for production shapes; single CTA for small ones
  // auto: the CTA pair for production shapes; the single-CTA kernel for
  // K <= 1024 (OPT-125M, cfg1), where a tile's mainloop is too short to
  // amortise the pair's prologue (measured +1.8 % on the cfg1 step)
  const bool pair = g_variant == 2 ? (M >= 2 * BM && N >= 256)
                                   : g_variant != 1 && M >= 2 * BM && N >= 256 && K > 1024;
  const int BROWS = pair ? 128 : (split ? 128 : 256);  // B rows staged per CTA
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = M;
  a.N = N;
  a.K = K;
  a.batch = batch;
  for (int p = 0; p < batch; ++p) {
    const zo2_gemm_problem &q = probs[p];
    if (!q.a_hi || !q.b_hi) return zo2_set_error(ZO2_E_ARG, "zo2_gemm: null operand");
    if (split != (q.a_lo != nullptr) || split != (q.b_lo != nullptr))
      return zo2_set_error(ZO2_E_ARG, "zo2_gemm: split planes must be given for A and B together");
    int rc = make_map(q.a_hi, M, K, BM, &a.tm[p][0]);
    if (!rc) rc = make_map(q.b_hi, N, K, (uint32_t)BROWS, &a.tm[p][2]);
    if (!rc && split) rc = make_map(q.a_lo, M, K, BM, &a.tm[p][1]);
    if (!rc && split) rc = make_map(q.b_lo, N, K, (uint32_t)BROWS, &a.tm[p][3]);
    if (rc) return rc;
    a.bias[p] = q.bias;
    a.c[p] = q.c;
    a.c_lo[p] = q.c_lo;
    a.targets[p] = q.targets;
    a.ce_part[p] = q.ce_part;
    if (epi == ZO2_EPI_CE && (!q.targets || !q.ce_part))
      return zo2_set_error(ZO2_E_ARG, "zo2_gemm: CE epilogue needs targets and ce_part");
    if (epi != ZO2_EPI_CE && !q.c) return zo2_set_error(ZO2_E_ARG, "zo2_gemm: null output");
    if ((epi == ZO2_EPI_GELU || epi == ZO2_EPI_OPERAND) && split && !q.c_lo)
      return zo2_set_error(ZO2_E_ARG, "zo2_gemm: split GELU needs c_lo");
  }
  cudaStream_t s = (cudaStream_t)cs;
  if (pair) return split ? dispatch_epi2<true>(a, epi, s) : dispatch_epi2<false>(a, epi, s);
  return split ? dispatch_epi<128, true>(a, epi, s) : dispatch_epi<256, false>(a, epi, s);
}
