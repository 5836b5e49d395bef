// zo2_layers.cu -- memory-bound forward kernels of the dual forward
// (model.py:241-313): embedding gather with on-the-fly perturbation (K8),
// LayerNorm (K4), causal attention (K5), cross-entropy reduction (K7 tail).
#include "zo2_common.cuh"
#include "zo2_rng.h"

void zo2_count_launch(uint64_t n = 1);
static inline cudaStream_t S(void *s) { return (cudaStream_t)s; }

__device__ __forceinline__ float ax1(float w, double coef, double z) {
  return __double2float_rn(__dadd_rn((double)w, __dmul_rn(coef, z)));
}

// ------------------------------------------------------------------ K8
// One thread = 4 consecutive columns of one token.  tok and pos elements are
// regenerated through the module's op sequence: update(lrs) then +eps, -2eps.
__device__ __forceinline__ void embed_elem4(const float *table, uint64_t i, uint64_t base,
                                            int upd, double ucoef, uint64_t lrs, double eps,
                                            uint64_t rs, float wp[4], float wm[4]) {
  float4 v = *(const float4 *)(table + i);
  float w[4] = {v.x, v.y, v.z, v.w};
  uint64_t r[4];
  if (upd) {
    zo2_raw_block(lrs, ZO2_PERTURB_STREAM, (base + i) >> 2, r);
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = ax1(w[j], ucoef, zo2_ndtri(zo2_u53(r[j])));
  }
  zo2_raw_block(rs, ZO2_PERTURB_STREAM, (base + i) >> 2, r);
  const double m2 = -2.0 * eps;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double z = zo2_ndtri(zo2_u53(r[j]));
    wp[j] = ax1(w[j], eps, z);
    wm[j] = ax1(wp[j], m2, z);
  }
}

__global__ void k_embed_dual(const int64_t *ids, uint64_t n_tok, uint32_t seq, uint32_t dim,
                             uint32_t vocab, const float *table, uint64_t base, int upd,
                             const double *d_g, double lr, uint64_t lrs, double eps,
                             uint64_t rs, float *outp, float *outm) {
  double ucoef = 0.0;
  if (upd) {
    const double g = *d_g;
    if (g == 0.0) upd = 0;
    else ucoef = -(lr * g);
  }
  const uint32_t q_per_tok = dim / 4;
  const uint64_t total = n_tok * q_per_tok;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < total;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = q / q_per_tok;
    const uint32_t c = (uint32_t)(q % q_per_tok) * 4;
    const int64_t id = ids[t];
    const uint32_t s = (uint32_t)(t % seq);
    float tp[4], tm[4], pp[4], pm[4];
    embed_elem4(table, (uint64_t)id * dim + c, base, upd, ucoef, lrs, eps, rs, tp, tm);
    embed_elem4(table, (uint64_t)vocab * dim + (uint64_t)s * dim + c, base, upd, ucoef, lrs,
                eps, rs, pp, pm);
    *(float4 *)(outp + t * dim + c) =
        make_float4(tp[0] + pp[0], tp[1] + pp[1], tp[2] + pp[2], tp[3] + pp[3]);
    *(float4 *)(outm + t * dim + c) =
        make_float4(tm[0] + pm[0], tm[1] + pm[1], tm[2] + pm[2], tm[3] + pm[3]);
  }
}

extern "C" int zo2_embed_dual(const int64_t *ids, uint64_t n_tok, uint32_t seq, uint32_t dim,
                              uint32_t vocab, uint32_t max_seq, const float *table,
                              uint64_t base, int update, const double *d_g, double lr,
                              uint64_t lrs_seed, double eps, uint64_t rs_seed, float *outp,
                              float *outm, void *cs) {
  if (n_tok == 0) return ZO2_OK;
  if (dim % 4 != 0 || base % 4 != 0)
    return zo2_set_error(ZO2_E_UNSUPPORTED, "zo2_embed_dual: dim and base must be multiples of 4");
  if (seq > max_seq) return zo2_set_error(ZO2_E_ARG, "zo2_embed_dual: seq > max_seq");
  if (update && !d_g) return zo2_set_error(ZO2_E_ARG, "zo2_embed_dual: update needs d_g");
  const uint64_t total = n_tok * (dim / 4);
  k_embed_dual<<<zo2_grid_for(total, 256, 148u * 16u), 256, 0, S(cs)>>>(
      ids, n_tok, seq, dim, vocab, table, base, update, d_g, lr, lrs_seed, eps, rs_seed, outp,
      outm);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

// ------------------------------------------------------------------ K4
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int k = 0; k < NT / 32; ++k) t += sh[k];
  return t;
}

// One CTA per row; the row stays in registers (dim <= 256 * 64).
template <int NT, int MAXV>
__global__ void __launch_bounds__(NT) k_layernorm(const float *x, uint32_t dim,
                                                  const float *gamma, const float *beta,
                                                  __nv_bfloat16 *out_hi, __nv_bfloat16 *out_lo) {
  __shared__ double sh[NT / 32];
  const uint64_t row = blockIdx.x;
  const float *xr = x + row * dim;
  float v[MAXV];
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < MAXV; ++k) {
    const uint32_t c = threadIdx.x + k * NT;
    v[k] = c < dim ? xr[c] : 0.f;
    s += v[k];
  }
  const float mu = (float)(block_sum<NT>(s, sh) / dim);
  double q = 0.0;
#pragma unroll
  for (int k = 0; k < MAXV; ++k) {
    const uint32_t c = threadIdx.x + k * NT;
    if (c < dim) {
      const float d = v[k] - mu;
      q += (double)d * d;
    }
  }
  const float var = (float)(block_sum<NT>(q, sh) / dim);
  const float inv = 1.0f / sqrtf(var + 1e-5f);
#pragma unroll
  for (int k = 0; k < MAXV; ++k) {
    const uint32_t c = threadIdx.x + k * NT;
    if (c < dim) {
      const float y = (v[k] - mu) * inv * gamma[c] + beta[c];
      const __nv_bfloat16 h = __float2bfloat16_rn(y);
      out_hi[row * dim + c] = h;
      if (out_lo) out_lo[row * dim + c] = __float2bfloat16_rn(y - __bfloat162float(h));
    }
  }
}

extern "C" int zo2_layernorm(const float *x, uint64_t rows, uint32_t dim, const float *gamma,
                             const float *beta, void *out_hi, void *out_lo, void *cs) {
  if (rows == 0) return ZO2_OK;
  __nv_bfloat16 *hi = (__nv_bfloat16 *)out_hi, *lo = (__nv_bfloat16 *)out_lo;
  if (dim <= 256 * 8)
    k_layernorm<256, 8><<<(unsigned)rows, 256, 0, S(cs)>>>(x, dim, gamma, beta, hi, lo);
  else if (dim <= 256 * 24)
    k_layernorm<256, 24><<<(unsigned)rows, 256, 0, S(cs)>>>(x, dim, gamma, beta, hi, lo);
  else if (dim <= 512 * 32)
    k_layernorm<512, 32><<<(unsigned)rows, 512, 0, S(cs)>>>(x, dim, gamma, beta, hi, lo);
  else
    return zo2_set_error(ZO2_E_UNSUPPORTED, "zo2_layernorm: dim > 16384");
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

__global__ void k_to_operand(const float *x, uint64_t n, __nv_bfloat16 *hi,
                             __nv_bfloat16 *lo) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    hi[i] = h;
    if (lo) lo[i] = __float2bfloat16_rn(v - __bfloat162float(h));
  }
}

extern "C" int zo2_to_operand(const float *x, uint64_t n, void *hi, void *lo, void *cs) {
  if (n == 0) return ZO2_OK;
  k_to_operand<<<zo2_grid_for(n, 256, 148u * 16u), 256, 0, S(cs)>>>(
      x, n, (__nv_bfloat16 *)hi, (__nv_bfloat16 *)lo);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

// ------------------------------------------------------------------ K5
// SIMT flash attention (fp32): CTA = (query tile of 32, head, batch);
// 8 lanes per query, each owning HD/8 dims of q and of the accumulator.
template <int HD>
__global__ void __launch_bounds__(256) k_attention(const float *qkv, uint32_t seq,
                                                   uint32_t n_heads, __nv_bfloat16 *out_hi,
                                                   __nv_bfloat16 *out_lo) {
  constexpr int DPT = HD / 8;   // dims per thread
  constexpr int KT = 32;        // keys per smem tile
  __shared__ float ks[KT][HD + 4];
  __shared__ float vs[KT][HD + 4];
  const uint32_t dim = n_heads * HD;
  const uint32_t ld = 3 * dim;
  const uint32_t b = blockIdx.z, h = blockIdx.y;
  const uint32_t q0 = blockIdx.x * 32;
  const uint32_t qi = q0 + threadIdx.x / 8;
  const uint32_t sub = threadIdx.x % 8;
  const float scale = 1.0f / sqrtf((float)HD);
  const float *base = qkv + (uint64_t)b * seq * ld;
  float q[DPT], acc[DPT];
  const bool valid = qi < seq;
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    q[j] = valid ? base[(uint64_t)qi * ld + h * HD + sub * DPT + j] : 0.f;
    acc[j] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  const uint32_t kmax = min(seq, q0 + 32);  // causal: keys <= last query of tile
  for (uint32_t k0 = 0; k0 < kmax; k0 += KT) {
    __syncthreads();
    for (int e = threadIdx.x; e < KT * HD; e += 256) {
      const int kr = e / HD, c = e % HD;
      const uint32_t kk = k0 + kr;
      ks[kr][c] = kk < seq ? base[(uint64_t)kk * ld + dim + h * HD + c] : 0.f;
      vs[kr][c] = kk < seq ? base[(uint64_t)kk * ld + 2 * dim + h * HD + c] : 0.f;
    }
    __syncthreads();
    const int kend = (int)min((uint32_t)KT, kmax - k0);
    for (int kr = 0; kr < kend; ++kr) {
      float sdot = 0.f;
#pragma unroll
      for (int j = 0; j < DPT; ++j) sdot += q[j] * ks[kr][sub * DPT + j];
      sdot += __shfl_xor_sync(0xffffffffu, sdot, 1);
      sdot += __shfl_xor_sync(0xffffffffu, sdot, 2);
      sdot += __shfl_xor_sync(0xffffffffu, sdot, 4);
      const uint32_t kk = k0 + kr;
      if (valid && kk <= qi) {
        const float sc = sdot * scale;
        const float mn = fmaxf(m, sc);
        const float corr = __expf(m - mn);
        const float p = __expf(sc - mn);
        l = l * corr + p;
#pragma unroll
        for (int j = 0; j < DPT; ++j) acc[j] = acc[j] * corr + p * vs[kr][sub * DPT + j];
        m = mn;
      }
    }
  }
  if (valid) {
    const float inv = 1.0f / l;
    const uint64_t o = ((uint64_t)b * seq + qi) * dim + h * HD + sub * DPT;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const float y = acc[j] * inv;
      const __nv_bfloat16 hv = __float2bfloat16_rn(y);
      out_hi[o + j] = hv;
      if (out_lo) out_lo[o + j] = __float2bfloat16_rn(y - __bfloat162float(hv));
    }
  }
}

// Tensor-core flash attention (mma.sync m16n8k16 bf16 -> f32).  CTA = 64
// queries (4 warps x 16 rows) of one (batch, head); key tiles of 64 up to the
// causal diagonal; online softmax in f32 registers; P stays in registers as
// the A operand of P.V.  SPLIT (f32 arithmetic): Q, K, V and P carry bf16
// hi + lo parts and each product is hi.hi + hi.lo + lo.hi (~2^-16 relative).
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

template <int HD, bool SPLIT>
__global__ void __launch_bounds__(128) k_attn_mma(const float *qkv, uint32_t seq,
                                                  uint32_t n_heads, __nv_bfloat16 *out_hi,
                                                  __nv_bfloat16 *out_lo) {
  constexpr int KB = 64, QB = 64;
  constexpr int KP = HD + 8;  // padded row (bf16) for conflict-free 32-bit loads
  constexpr int VP = KB + 8;
  constexpr int NKS = HD / 16;     // k-steps of Q.K^T
  constexpr int NOT = HD / 8;      // n-tiles of O
  extern __shared__ __align__(16) uint8_t att_smem[];
  __nv_bfloat16 *Kh = (__nv_bfloat16 *)att_smem;
  __nv_bfloat16 *Kl = Kh + KB * KP;
  __nv_bfloat16 *Vh = Kl + (SPLIT ? KB * KP : 0);   // transposed [HD][VP]
  __nv_bfloat16 *Vl = Vh + HD * VP;

  const uint32_t dim = n_heads * HD, ld = 3 * dim;
  const uint32_t b = blockIdx.z, h = blockIdx.y;
  const uint32_t n_qt = (seq + QB - 1) / QB;
  const uint32_t qt = n_qt - 1 - blockIdx.x;  // heavy (late) tiles first
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = lane / 4, c = lane % 4;
  const float *base = qkv + (uint64_t)b * seq * ld;
  const uint32_t r0 = qt * QB + warp * 16 + g, r1 = r0 + 8;  // this thread's 2 rows
  const float scale = 1.0f / sqrtf((float)HD);

  // Q fragments (A operand, row-major 16 x 16 per k-step)
  uint32_t qh[NKS][4], ql[NKS][4];
#pragma unroll
  for (int ks = 0; ks < NKS; ++ks) {
#pragma unroll
    for (int part = 0; part < 4; ++part) {
      const uint32_t row = (part & 1) ? r1 : r0;
      const int col = ks * 16 + (part >> 1) * 8 + 2 * c;
      float x0 = 0.f, x1 = 0.f;
      if (row < seq) {
        const float2 v = *(const float2 *)(base + (uint64_t)row * ld + h * HD + col);
        x0 = v.x;
        x1 = v.y;
      }
      if (SPLIT) split2(x0, x1, qh[ks][part], ql[ks][part]);
      else qh[ks][part] = pack_bf16(x0, x1);
    }
  }
  float o[NOT][4];
#pragma unroll
  for (int i = 0; i < NOT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  const uint32_t k_end = min(seq, (qt + 1) * QB);
  for (uint32_t k0 = 0; k0 < k_end; k0 += KB) {
    __syncthreads();
    // K tile [KB][HD] row-major, V tile transposed [HD][KB]
    for (int e = threadIdx.x; e < KB * HD / 2; e += 128) {
      const int kr = e / (HD / 2), cc = 2 * (e % (HD / 2));
      const uint32_t key = k0 + kr;
      float2 kv = make_float2(0.f, 0.f), vv = make_float2(0.f, 0.f);
      if (key < seq) {
        kv = *(const float2 *)(base + (uint64_t)key * ld + dim + h * HD + cc);
        vv = *(const float2 *)(base + (uint64_t)key * ld + 2 * dim + h * HD + cc);
      }
      uint32_t kh, kl, vh2, vl2;
      if (SPLIT) {
        split2(kv.x, kv.y, kh, kl);
        split2(vv.x, vv.y, vh2, vl2);
        *(uint32_t *)(Kl + kr * KP + cc) = kl;
        Vl[cc * VP + kr] = ((__nv_bfloat16 *)&vl2)[0];
        Vl[(cc + 1) * VP + kr] = ((__nv_bfloat16 *)&vl2)[1];
      } else {
        kh = pack_bf16(kv.x, kv.y);
        vh2 = pack_bf16(vv.x, vv.y);
      }
      *(uint32_t *)(Kh + kr * KP + cc) = kh;
      Vh[cc * VP + kr] = ((__nv_bfloat16 *)&vh2)[0];
      Vh[(cc + 1) * VP + kr] = ((__nv_bfloat16 *)&vh2)[1];
    }
    __syncthreads();
    // S = Q K^T for this warp's 16 rows x 64 keys
    float s[KB / 8][4];
#pragma unroll
    for (int nt = 0; nt < KB / 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
      const int kr = nt * 8 + g;
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        const uint32_t bh0 = *(const uint32_t *)(Kh + kr * KP + ks * 16 + 2 * c);
        const uint32_t bh1 = *(const uint32_t *)(Kh + kr * KP + ks * 16 + 8 + 2 * c);
        mma16816(s[nt], qh[ks], bh0, bh1);
        if (SPLIT) {
          const uint32_t bl0 = *(const uint32_t *)(Kl + kr * KP + ks * 16 + 2 * c);
          const uint32_t bl1 = *(const uint32_t *)(Kl + kr * KP + ks * 16 + 8 + 2 * c);
          mma16816(s[nt], qh[ks], bl0, bl1);
          mma16816(s[nt], ql[ks], bh0, bh1);
        }
      }
    }
    // scale, causal / length mask, online softmax (rows r0 and r1)
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
    // rows with every key masked so far keep m = -inf; use 0 as the base
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
    // O += P V : P (registers) as A, V^T rows as B
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
      for (int nt = 0; nt < NOT; ++nt) {
        const int vr = nt * 8 + g;
        const uint32_t bh0 = *(const uint32_t *)(Vh + vr * VP + kk * 16 + 2 * c);
        const uint32_t bh1 = *(const uint32_t *)(Vh + vr * VP + kk * 16 + 8 + 2 * c);
        mma16816(o[nt], ph, bh0, bh1);
        if (SPLIT) {
          const uint32_t bl0 = *(const uint32_t *)(Vl + vr * VP + kk * 16 + 2 * c);
          const uint32_t bl1 = *(const uint32_t *)(Vl + vr * VP + kk * 16 + 8 + 2 * c);
          mma16816(o[nt], ph, bl0, bl1);
          mma16816(o[nt], pl, bh0, bh1);
        }
      }
    }
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = 1.0f / l0, i1 = 1.0f / l1;
#pragma unroll
  for (int nt = 0; nt < NOT; ++nt) {
    const int col = h * HD + nt * 8 + 2 * c;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const uint32_t row = half ? r1 : r0;
      if (row >= seq) continue;
      const float a = o[nt][2 * half] * (half ? i1 : i0);
      const float bb = o[nt][2 * half + 1] * (half ? i1 : i0);
      const uint64_t off = ((uint64_t)b * seq + row) * dim + col;
      uint32_t hv, lv;
      split2(a, bb, hv, lv);
      *(uint32_t *)(out_hi + off) = hv;
      if (SPLIT) *(uint32_t *)(out_lo + off) = lv;
    }
  }
}

template <int HD, bool SPLIT>
static int launch_attn(const float *qkv, uint32_t batch, uint32_t seq, uint32_t nh,
                       __nv_bfloat16 *hi, __nv_bfloat16 *lo, cudaStream_t s) {
  constexpr int KB = 64, KP = HD + 8, VP = KB + 8;
  const int smem = (SPLIT ? 2 : 1) * (KB * KP + HD * VP) * 2;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_attn_mma<HD, SPLIT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return zo2_set_cuda_error(e);
    attr = true;
  }
  dim3 grid((seq + 63) / 64, nh, batch);
  k_attn_mma<HD, SPLIT><<<grid, 128, smem, s>>>(qkv, seq, nh, hi, lo);
  return ZO2_OK;
}

extern "C" int zo2_attention(const float *qkv, uint32_t batch, uint32_t seq, uint32_t n_heads,
                             uint32_t head_dim, void *ctx_hi, void *ctx_lo, void *cs) {
  if (batch == 0 || seq == 0) return ZO2_OK;
  __nv_bfloat16 *hi = (__nv_bfloat16 *)ctx_hi, *lo = (__nv_bfloat16 *)ctx_lo;
  const bool split = lo != nullptr;
  cudaStream_t s = S(cs);
  int rc = ZO2_OK;
  switch (head_dim) {
    case 16: rc = split ? launch_attn<16, true>(qkv, batch, seq, n_heads, hi, lo, s)
                        : launch_attn<16, false>(qkv, batch, seq, n_heads, hi, lo, s); break;
    case 32: rc = split ? launch_attn<32, true>(qkv, batch, seq, n_heads, hi, lo, s)
                        : launch_attn<32, false>(qkv, batch, seq, n_heads, hi, lo, s); break;
    case 64: rc = split ? launch_attn<64, true>(qkv, batch, seq, n_heads, hi, lo, s)
                        : launch_attn<64, false>(qkv, batch, seq, n_heads, hi, lo, s); break;
    case 128: rc = split ? launch_attn<128, true>(qkv, batch, seq, n_heads, hi, lo, s)
                         : launch_attn<128, false>(qkv, batch, seq, n_heads, hi, lo, s); break;
    case 8: {  // tiny heads (toy configs): SIMT path
      dim3 grid((seq + 31) / 32, n_heads, batch);
      k_attention<8><<<grid, 256, 0, s>>>(qkv, seq, n_heads, hi, lo);
      break;
    }
    default:
      return zo2_set_error(ZO2_E_UNSUPPORTED, "zo2_attention: head_dim not in {8,16,32,64,128}");
  }
  if (rc) return rc;
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

// ------------------------------------------------------------------ K7 tail
// Combine per-(row, n-tile) partials {max, sum exp(x - max), target logit}
// into sum over rows of (logsumexp - logit[target]) in f64.
__global__ void k_ce_reduce(const float *part, uint32_t M, uint32_t n_tiles,
                            uint64_t stride, double *work) {
  const int b = blockIdx.y;
  const float *P = part + b * stride;
  double acc = 0.0;
  // contiguous row range per CTA, fixed-order reductions: the sum (and so g)
  // is bitwise reproducible run to run (no floating-point atomics)
  const uint32_t per = (M + gridDim.x - 1) / gridDim.x;
  const uint32_t r0 = blockIdx.x * per, r1 = min(M, r0 + per);
  for (uint32_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const float *pr = P + (uint64_t)r * n_tiles * 3;
    double mx = -INFINITY, tgt = 0.0;
    for (uint32_t t = 0; t < n_tiles; ++t) mx = fmax(mx, (double)pr[3 * t]);
    double s = 0.0;
    for (uint32_t t = 0; t < n_tiles; ++t) {
      s += (double)pr[3 * t + 1] * exp((double)pr[3 * t] - mx);
      const float tl = pr[3 * t + 2];
      if (tl != -INFINITY) tgt = (double)tl;
    }
    acc += mx + log(s) - tgt;
  }
  __shared__ double sh[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) t += sh[w];
    work[b * gridDim.x + blockIdx.x] = t;
  }
}

__global__ void k_ce_finish(const double *work, int nparts, int batch, double *sums) {
  const int b = threadIdx.x;
  if (b < batch) {
    double t = 0.0;
    for (int i = 0; i < nparts; ++i) t += work[b * nparts + i];
    sums[b] = t;
  }
}

extern "C" int zo2_ce_reduce(const float *part, uint32_t M, uint32_t n_tiles, int batch,
                             uint64_t part_stride, double *d_work, double *d_sums, void *cs) {
  if (M == 0 || batch < 1) return ZO2_OK;
  if (!d_work || !d_sums) return zo2_set_error(ZO2_E_ARG, "zo2_ce_reduce: null workspace");
  dim3 grid(ZO2_CE_PARTS, batch);
  k_ce_reduce<<<grid, 256, 0, S(cs)>>>(part, M, n_tiles, part_stride, d_work);
  k_ce_finish<<<1, 32, 0, S(cs)>>>(d_work, ZO2_CE_PARTS, batch, d_sums);
  zo2_count_launch(2);
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}
