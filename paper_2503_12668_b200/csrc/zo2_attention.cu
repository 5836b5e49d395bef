// zo2_attention.cu -- K5: causal softmax attention of the dual forward
// (model.py:273-283: split heads, q k^T / sqrt(hd), causal -inf mask,
// max-subtracted softmax, w @ v) on tensor cores.
//
// Inputs are the bf16 planes the QKV GEMM epilogue writes ([B*S, 3d]: q, k, v
// column blocks; hi, plus lo in split/f32 mode), so nothing is converted here.
// CTA = 128 queries (8 warps x 16 rows) of one (batch, head).  K / V tiles of
// 64 keys stream through shared memory with cp.async double buffering; B
// fragments come from ldmatrix (K) and ldmatrix.trans (V); the online softmax
// runs in f32 registers and P stays in registers as the A operand of P.V
// (mma.sync m16n8k16 bf16 -> f32).  In split mode every product is
// hi.hi + hi.lo + lo.hi (~2^-16 relative), as in the GEMMs.
#include "zo2_common.cuh"

void zo2_count_launch(uint64_t n = 1);
extern "C" int zo2_attention_tc(const void *qkv_hi, const void *qkv_lo, uint32_t batch,
                                uint32_t seq, uint32_t n_heads, uint32_t head_dim, void *ctx_hi,
                                void *ctx_lo, void *cs);
static int g_attn_variant = 0;  // 0: tcgen05 kernel where eligible, 1: mma.sync kernel only
extern "C" int zo2_set_attention_variant(int v) {
  if (v < 0 || v > 1) return zo2_set_error(ZO2_E_ARG, "zo2_set_attention_variant: 0 or 1");
  g_attn_variant = v;
  return ZO2_OK;
}

namespace {

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t *>(&v);
}
__device__ __forceinline__ void split2(float a, float b, uint32_t &hi, uint32_t &lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  hi = *reinterpret_cast<const uint32_t *>(&h);
  lo = pack_bf16(a - __low2float(h), b - __high2float(h));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2,
                                        uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1,
                                          uint32_t &r2, uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, bool valid) {
  const int n = valid ? 16 : 0;  // zero-fill rows past the sequence end
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

constexpr int KB = 64;        // keys per tile
constexpr int WARPS = 8;      // 16 query rows each
constexpr int QB = 16 * WARPS;

template <int HD, bool SPLIT>
struct AttnCfg {
  static constexpr int P = HD + 8;                       // padded row (bf16): ldmatrix conflict-free
  static constexpr int TILE = KB * P;                    // elements per plane tile
  static constexpr int PLANES = SPLIT ? 4 : 2;           // K hi, V hi (+ K lo, V lo)
  static constexpr int STAGE = PLANES * TILE;
  static constexpr int SMEM = 2 * STAGE * 2;             // 2 stages, bytes
};

#ifndef ZO2_ATTN_MINB
#define ZO2_ATTN_MINB 1
#endif
template <int HD, bool SPLIT>
__global__ void __launch_bounds__(32 * WARPS, ZO2_ATTN_MINB) k_attn(
    const __nv_bfloat16 *__restrict__ qkv_hi, const __nv_bfloat16 *__restrict__ qkv_lo,
    uint32_t seq, uint32_t n_heads, __nv_bfloat16 *__restrict__ out_hi,
    __nv_bfloat16 *__restrict__ out_lo) {
  using C = AttnCfg<HD, SPLIT>;
  constexpr int NKS = HD / 16;   // k-steps of q.k^T
  constexpr int NOT = HD / 8;    // n-tiles of O
  extern __shared__ __align__(128) __nv_bfloat16 sm[];
  const uint32_t dim = n_heads * HD, ld = 3 * dim;
  const uint32_t b = blockIdx.z, h = blockIdx.y;
  const uint32_t n_qt = (seq + QB - 1) / QB;
  const uint32_t qt = n_qt - 1 - blockIdx.x;  // heavy (late) query tiles first
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = lane / 4, c = lane % 4;
  const uint64_t tok0 = (uint64_t)b * seq;
  const uint32_t wrow0 = qt * QB + warp * 16;          // first row of this warp
  const uint32_t r0 = wrow0 + g, r1 = r0 + 8;
  const float scale = 1.0f / sqrtf((float)HD);

  // Q fragments straight from the planes (A operand, row-major 16 x 16)
  uint32_t qh[NKS][4], ql[NKS][4];
#pragma unroll
  for (int ks = 0; ks < NKS; ++ks)
#pragma unroll
    for (int part = 0; part < 4; ++part) {
      const uint32_t row = (part & 1) ? r1 : r0;
      const uint32_t col = h * HD + ks * 16 + (part >> 1) * 8 + 2 * c;
      const uint64_t off = (tok0 + row) * ld + col;
      qh[ks][part] = row < seq ? *(const uint32_t *)(qkv_hi + off) : 0u;
      if (SPLIT) ql[ks][part] = row < seq ? *(const uint32_t *)(qkv_lo + off) : 0u;
    }

  // async tile loader: rows = keys, 16-byte chunks of HD dims, 4 (or 2) planes
  auto load_tile = [&](int stage, uint32_t k0) {
    __nv_bfloat16 *base = sm + stage * C::STAGE;
    constexpr int CH = HD / 8;  // 16-byte chunks per row
    for (int e = threadIdx.x; e < KB * CH; e += 32 * WARPS) {
      const int kr = e / CH, ch = e % CH;
      const uint32_t key = k0 + kr;
      const bool ok = key < seq;
      const uint64_t row = (tok0 + (ok ? key : 0)) * ld + h * HD + ch * 8;
      const uint32_t so = (uint32_t)(kr * C::P + ch * 8) * 2;
      const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(base);
      cp_async16(s0 + so, qkv_hi + row + dim, ok);                              // K hi
      cp_async16(s0 + C::TILE * 2 + so, qkv_hi + row + 2 * dim, ok);           // V hi
      if (SPLIT) {
        cp_async16(s0 + 2 * C::TILE * 2 + so, qkv_lo + row + dim, ok);         // K lo
        cp_async16(s0 + 3 * C::TILE * 2 + so, qkv_lo + row + 2 * dim, ok);     // V lo
      }
    }
  };

  float o[NOT][4];
#pragma unroll
  for (int i = 0; i < NOT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  const uint32_t k_end = min(seq, (qt + 1) * QB);
  const int n_kt = (int)((k_end + KB - 1) / KB);
  load_tile(0, 0);
  cp_commit();
  // ldmatrix lane addressing: matrix mi = lane / 8, row = lane % 8
  const int mi = lane / 8, mr = lane % 8;
  for (int kt = 0; kt < n_kt; ++kt) {
    if (kt + 1 < n_kt) {
      load_tile((kt + 1) & 1, (uint32_t)(kt + 1) * KB);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const uint32_t k0 = (uint32_t)kt * KB;
    if (k0 <= wrow0 + 15) {  // some key of this tile is visible to this warp
      const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm + (kt & 1) * C::STAGE);
      const uint32_t sKh = sb, sVh = sb + C::TILE * 2;
      const uint32_t sKl = sb + 2 * C::TILE * 2, sVl = sb + 3 * C::TILE * 2;
      // ---- S = Q K^T (16 rows x 64 keys)
      float s[KB / 8][4];
#pragma unroll
      for (int nt = 0; nt < KB / 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
#pragma unroll
        for (int np = 0; np < KB / 16; ++np) {  // pairs of n-tiles
          // matrices: (keys np*16 + 0..7 | 8..15) x (dims ks*16 + 0..7 | 8..15)
          const uint32_t key = np * 16 + (mi >> 1) * 8 + mr;
          const uint32_t off = (uint32_t)(key * C::P + ks * 16 + (mi & 1) * 8) * 2;
          uint32_t b0, b1, b2, b3;
          ldsm_x4(sKh + off, b0, b1, b2, b3);
          mma16816(s[2 * np], qh[ks], b0, b1);
          mma16816(s[2 * np + 1], qh[ks], b2, b3);
          if (SPLIT) {
            uint32_t c0, c1, c2, c3;
            ldsm_x4(sKl + off, c0, c1, c2, c3);
            mma16816(s[2 * np], qh[ks], c0, c1);
            mma16816(s[2 * np + 1], qh[ks], c2, c3);
            mma16816(s[2 * np], ql[ks], b0, b1);
            mma16816(s[2 * np + 1], ql[ks], b2, b3);
          }
        }
      }
      // ---- scale, causal / length mask, online softmax
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < KB / 8; ++nt) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t key = k0 + nt * 8 + 2 * c + (j & 1);
          const uint32_t row = (j < 2) ? r0 : r1;
          float v = s[nt][j] * scale;
          if (key > row || key >= seq) v = -INFINITY;
          s[nt][j] = v;
        }
        mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
        mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
      }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
      const float b0 = n0 == -INFINITY ? 0.f : n0, b1 = n1 == -INFINITY ? 0.f : n1;
      const float cr0 = expf(m0 - b0), cr1 = expf(m1 - b1);
      m0 = n0;
      m1 = n1;
      float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
      for (int nt = 0; nt < KB / 8; ++nt) {
        s[nt][0] = expf(s[nt][0] - b0);
        s[nt][1] = expf(s[nt][1] - b0);
        s[nt][2] = expf(s[nt][2] - b1);
        s[nt][3] = expf(s[nt][3] - b1);
        ps0 += s[nt][0] + s[nt][1];
        ps1 += s[nt][2] + s[nt][3];
      }
      l0 = l0 * cr0 + ps0;
      l1 = l1 * cr1 + ps1;
#pragma unroll
      for (int i = 0; i < NOT; ++i) {
        o[i][0] *= cr0;
        o[i][1] *= cr0;
        o[i][2] *= cr1;
        o[i][3] *= cr1;
      }
      // ---- O += P V (P in registers as A; V^T fragments via ldmatrix.trans)
#pragma unroll
      for (int kk = 0; kk < KB / 16; ++kk) {
        uint32_t ph[4], pl[4];
        if (SPLIT) {
          split2(s[2 * kk][0], s[2 * kk][1], ph[0], pl[0]);
          split2(s[2 * kk][2], s[2 * kk][3], ph[1], pl[1]);
          split2(s[2 * kk + 1][0], s[2 * kk + 1][1], ph[2], pl[2]);
          split2(s[2 * kk + 1][2], s[2 * kk + 1][3], ph[3], pl[3]);
        } else {
          ph[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
          ph[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
          ph[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
          ph[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
        }
#pragma unroll
        for (int np = 0; np < NOT / 2; ++np) {  // pairs of dim n-tiles
          // matrices: (keys kk*16 + 0..7 | 8..15) x (dims np*16 + 0..7 | 8..15), transposed
          const uint32_t key = kk * 16 + (mi & 1) * 8 + mr;
          const uint32_t off = (uint32_t)(key * C::P + np * 16 + (mi >> 1) * 8) * 2;
          uint32_t v0, v1, v2, v3;
          ldsm_x4_t(sVh + off, v0, v1, v2, v3);
          mma16816(o[2 * np], ph, v0, v1);
          mma16816(o[2 * np + 1], ph, v2, v3);
          if (SPLIT) {
            uint32_t w0, w1, w2, w3;
            ldsm_x4_t(sVl + off, w0, w1, w2, w3);
            mma16816(o[2 * np], ph, w0, w1);
            mma16816(o[2 * np + 1], ph, w2, w3);
            mma16816(o[2 * np], pl, v0, v1);
            mma16816(o[2 * np + 1], pl, v2, v3);
          }
        }
      }
    }
    __syncthreads();  // everyone is done with this stage before it is refilled
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = 1.0f / l0, i1 = 1.0f / l1;
#pragma unroll
  for (int nt = 0; nt < NOT; ++nt) {
    const uint32_t col = h * HD + nt * 8 + 2 * c;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const uint32_t row = half ? r1 : r0;
      if (row >= seq) continue;
      const float inv = half ? i1 : i0;
      const uint64_t off = (tok0 + row) * dim + col;
      uint32_t hv, lv;
      split2(o[nt][2 * half] * inv, o[nt][2 * half + 1] * inv, hv, lv);
      *(uint32_t *)(out_hi + off) = hv;
      if (SPLIT) *(uint32_t *)(out_lo + off) = lv;
    }
  }
}

// Tiny head dims (toy models, hd not a multiple of 16): SIMT, one thread per
// (query, head), exact f32 softmax over the visible keys.
__global__ void k_attn_small(const __nv_bfloat16 *qkv_hi, const __nv_bfloat16 *qkv_lo,
                             uint32_t batch, uint32_t seq, uint32_t n_heads, uint32_t hd,
                             __nv_bfloat16 *out_hi, __nv_bfloat16 *out_lo) {
  const uint32_t dim = n_heads * hd, ld = 3 * dim;
  const uint64_t total = (uint64_t)batch * seq * n_heads;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t h = (uint32_t)(i % n_heads);
    const uint64_t t = i / n_heads;
    const uint32_t q = (uint32_t)(t % seq);
    const uint64_t tok0 = t - q;
    auto at = [&](uint64_t tok, uint32_t col) {
      float v = __bfloat162float(qkv_hi[tok * ld + col]);
      if (qkv_lo) v += __bfloat162float(qkv_lo[tok * ld + col]);
      return v;
    };
    const float scale = 1.0f / sqrtf((float)hd);
    float m = -INFINITY;
    for (uint32_t k = 0; k <= q; ++k) {
      float sdot = 0.f;
      for (uint32_t j = 0; j < hd; ++j) sdot += at(t, h * hd + j) * at(tok0 + k, dim + h * hd + j);
      m = fmaxf(m, sdot * scale);
    }
    float l = 0.f;
    float acc[32];
    for (uint32_t j = 0; j < hd && j < 32; ++j) acc[j] = 0.f;
    for (uint32_t k = 0; k <= q; ++k) {
      float sdot = 0.f;
      for (uint32_t j = 0; j < hd; ++j) sdot += at(t, h * hd + j) * at(tok0 + k, dim + h * hd + j);
      const float p = expf(sdot * scale - m);
      l += p;
      for (uint32_t j = 0; j < hd && j < 32; ++j) acc[j] += p * at(tok0 + k, 2 * dim + h * hd + j);
    }
    for (uint32_t j = 0; j < hd && j < 32; ++j) {
      const float y = acc[j] / l;
      const __nv_bfloat16 hv = __float2bfloat16_rn(y);
      out_hi[t * dim + h * hd + j] = hv;
      if (out_lo) out_lo[t * dim + h * hd + j] = __float2bfloat16_rn(y - __bfloat162float(hv));
    }
  }
}

template <int HD, bool SPLIT>
int launch(const void *qh, const void *ql, uint32_t batch, uint32_t seq, uint32_t nh, void *oh,
           void *ol, cudaStream_t s) {
  using C = AttnCfg<HD, SPLIT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_attn<HD, SPLIT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return zo2_set_cuda_error(e);
    attr = true;
  }
  dim3 grid((seq + QB - 1) / QB, nh, batch);
  k_attn<HD, SPLIT><<<grid, 32 * WARPS, C::SMEM, s>>>(
      (const __nv_bfloat16 *)qh, (const __nv_bfloat16 *)ql, seq, nh, (__nv_bfloat16 *)oh,
      (__nv_bfloat16 *)ol);
  return ZO2_OK;
}

}  // namespace

extern "C" int zo2_attention(const void *qkv_hi, const void *qkv_lo, uint32_t batch,
                             uint32_t seq, uint32_t n_heads, uint32_t head_dim, void *ctx_hi,
                             void *ctx_lo, void *cs) {
  if (batch == 0 || seq == 0) return ZO2_OK;
  if (!qkv_hi || !ctx_hi) return zo2_set_error(ZO2_E_ARG, "zo2_attention: null pointer");
  const bool split = qkv_lo != nullptr;
  if (split != (ctx_lo != nullptr))
    return zo2_set_error(ZO2_E_ARG, "zo2_attention: lo planes must be given for in and out");
  cudaStream_t s = (cudaStream_t)cs;
  int rc = ZO2_OK;
  if (g_attn_variant == 0) {
    // tcgen05 / TMEM kernel (zo2_gemm_sm100.cu) for seq % 128 == 0, hd 64 / 128
    rc = zo2_attention_tc(qkv_hi, qkv_lo, batch, seq, n_heads, head_dim, ctx_hi, ctx_lo, cs);
    if (rc == ZO2_OK) {
      zo2_count_launch();
      ZO2_CHECK_LAUNCH();
      return ZO2_OK;
    }
    if (rc != ZO2_E_UNSUPPORTED) return rc;
    rc = ZO2_OK;
  }
  switch (head_dim) {
    case 16: rc = split ? launch<16, true>(qkv_hi, qkv_lo, batch, seq, n_heads, ctx_hi, ctx_lo, s)
                        : launch<16, false>(qkv_hi, qkv_lo, batch, seq, n_heads, ctx_hi, ctx_lo, s); break;
    case 32: rc = split ? launch<32, true>(qkv_hi, qkv_lo, batch, seq, n_heads, ctx_hi, ctx_lo, s)
                        : launch<32, false>(qkv_hi, qkv_lo, batch, seq, n_heads, ctx_hi, ctx_lo, s); break;
    case 64: rc = split ? launch<64, true>(qkv_hi, qkv_lo, batch, seq, n_heads, ctx_hi, ctx_lo, s)
                        : launch<64, false>(qkv_hi, qkv_lo, batch, seq, n_heads, ctx_hi, ctx_lo, s); break;
    case 128: rc = split ? launch<128, true>(qkv_hi, qkv_lo, batch, seq, n_heads, ctx_hi, ctx_lo, s)
                         : launch<128, false>(qkv_hi, qkv_lo, batch, seq, n_heads, ctx_hi, ctx_lo, s); break;
    default:
      if (head_dim > 32)
        return zo2_set_error(ZO2_E_UNSUPPORTED, "zo2_attention: head_dim not in {<=32, 64, 128}");
      k_attn_small<<<zo2_grid_for((uint64_t)batch * seq * n_heads, 128, 148u * 8u), 128, 0, s>>>(
          (const __nv_bfloat16 *)qkv_hi, (const __nv_bfloat16 *)qkv_lo, batch, seq, n_heads,
          head_dim, (__nv_bfloat16 *)ctx_hi, (__nv_bfloat16 *)ctx_lo);
  }
  if (rc) return rc;
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}
