// zo2_f64.cu -- the arith=f64 forward (the reference's default arithmetic,
// harness/config.py:53; model.py:241-313 in float64).
//
// The f64 path keeps the reference's own per-module sequence: the bucket is
// perturbed in place (+eps, -2eps, +eps with zo2_axpy_z, the update before it
// with K2) and these kernels run the forward of one sign straight from the
// perturbed bucket.  Every operation is an IEEE binary64 operation on B200's
// FP64 pipe (DFMA); summation orders differ from numpy's pairwise/BLAS orders,
// so losses agree to ~1e-13 relative, not bit for bit (the parity tests
// state the tolerance).  Sizes: the reference runs f64 only at toy and
// OPT-125M scale; the GEMM is a 64x64x16 shared-memory-tiled SIMT kernel
// (4x4 DFMA register tile per thread), ample for those shapes.
#include <math.h>

#include "zo2_common.cuh"

void zo2_count_launch(uint64_t n = 1);

namespace {
inline cudaStream_t S(void *s) { return (cudaStream_t)s; }

constexpr int TM = 64, TN = 64, TK = 16;

// C[M,N] (=|+=) A[M,K] @ B + bias; B is [K,N] row-major, or [N,K] (BT: C = A B^T).
template <bool BT>
__global__ void __launch_bounds__(256) k_f64_gemm(const double *__restrict__ A,
                                                  const double *__restrict__ B,
                                                  const double *__restrict__ bias, double *C,
                                                  int M, int N, int K, int epi) {
  __shared__ double As[TK][TM + 1];
  __shared__ double Bs[TK][TN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int e = threadIdx.x; e < TM * TK; e += 256) {
      const int r = e / TK, c = e % TK;
      const int gm = m0 + r, gk = k0 + c;
      As[c][r] = (gm < M && gk < K) ? A[(size_t)gm * K + gk] : 0.0;
    }
    for (int e = threadIdx.x; e < TN * TK; e += 256) {
      if (BT) {
        const int n = e / TK, c = e % TK;
        const int gn = n0 + n, gk = k0 + c;
        Bs[c][n] = (gn < N && gk < K) ? B[(size_t)gn * K + gk] : 0.0;
      } else {
        const int c = e / TN, n = e % TN;
        const int gn = n0 + n, gk = k0 + c;
        Bs[c][n] = (gn < N && gk < K) ? B[(size_t)gk * N + gn] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx + 16 * j;
      if (gn >= N) continue;
      double v = acc[i][j];
      if (bias) v = v + bias[gn];
      double *c = C + (size_t)gm * N + gn;
      if (epi == ZO2_F64_EPI_GELU) {
        v = 0.5 * v * (1.0 + erf(v / 1.4142135623730951));  // model.py _gelu
        *c = v;
      } else if (epi == ZO2_F64_EPI_RESIDUAL) {
        *c = *c + v;  // h + (x @ W + b)
      } else {
        *c = v;
      }
    }
  }
}

template <int NT>
__device__ double block_sum(double v, double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < NT / 32; ++w) t += sh[w];
    sh[32] = t;
  }
  __syncthreads();
  t = sh[32];
  __syncthreads();
  return t;
}

// model.py _ln: (x - mu) / sqrt(var + 1e-5) * g + b, var the biased mean square.
__global__ void __launch_bounds__(256) k_f64_layernorm(const double *x, uint32_t dim,
                                                       const double *g, const double *b,
                                                       double *out) {
  __shared__ double sh[33];
  const double *xr = x + (size_t)blockIdx.x * dim;
  double s = 0.0;
  for (uint32_t c = threadIdx.x; c < dim; c += 256) s += xr[c];
  const double mu = block_sum<256>(s, sh) / (double)dim;
  double q = 0.0;
  for (uint32_t c = threadIdx.x; c < dim; c += 256) {
    const double t = xr[c] - mu;
    q += t * t;
  }
  const double var = block_sum<256>(q, sh) / (double)dim;
  const double den = sqrt(var + 1e-5);
  double *o = out + (size_t)blockIdx.x * dim;
  for (uint32_t c = threadIdx.x; c < dim; c += 256) o[c] = (xr[c] - mu) / den * g[c] + b[c];
}

__global__ void k_f64_embed(const int64_t *ids, uint64_t n_tok, uint32_t seq, uint32_t dim,
                            const double *tok, const double *pos, double *out) {
  const uint64_t n = n_tok * dim;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = i / dim, c = i % dim;
    out[i] = tok[(uint64_t)ids[t] * dim + c] + pos[(t % seq) * dim + c];
  }
}

// Causal softmax attention, one warp per query row (model.py:273-283):
// s_j = (q . k_j) / sqrt(hd), w = exp(s - max) / sum, ctx = sum_j w_j v_j.
constexpr int ATT_WARPS = 4;
__global__ void __launch_bounds__(ATT_WARPS * 32) k_f64_attention(const double *qkv, uint32_t seq,
                                                                  uint32_t n_heads,
                                                                  uint32_t hd, double *ctx) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t i = blockIdx.x * ATT_WARPS + warp;
  if (i >= seq) return;
  const uint32_t h = blockIdx.y, b = blockIdx.z, d = n_heads * hd;
  double *sc = sm + (size_t)warp * (seq + hd);
  double *qs = sc + seq;
  const double *base = qkv + (size_t)b * seq * 3 * d;
  const double *q = base + (size_t)i * 3 * d + h * hd;
  for (uint32_t c = lane; c < hd; c += 32) qs[c] = q[c];
  __syncwarp();
  const double scale = sqrt((double)hd);
  double mx = -INFINITY;
  for (uint32_t j = lane; j <= i; j += 32) {
    const double *k = base + (size_t)j * 3 * d + d + h * hd;
    double dot = 0.0;
    for (uint32_t c = 0; c < hd; ++c) dot = fma(qs[c], k[c], dot);
    const double s = dot / scale;
    sc[j] = s;
    mx = fmax(mx, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double sum = 0.0;
  for (uint32_t j = lane; j <= i; j += 32) {
    const double p = exp(sc[j] - mx);
    sc[j] = p;
    sum += p;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  __syncwarp();
  double *out = ctx + ((size_t)b * seq + i) * d + h * hd;
  for (uint32_t c = lane; c < hd; c += 32) {
    double acc = 0.0;
    for (uint32_t j = 0; j <= i; ++j) {
      const double *v = base + (size_t)j * 3 * d + 2 * d + h * hd;
      acc = fma(sc[j] / sum, v[c], acc);
    }
    out[c] = acc;
  }
}

// Per row: logsumexp(logits) - logits[target] (model.py:308-313 in f64);
// an out-of-range target yields NaN (the engine checks targets beforehand).
__global__ void __launch_bounds__(256) k_f64_ce_rows(const double *logits,
                                                     const int64_t *targets, uint32_t vocab,
                                                     double *row) {
  __shared__ double sh[33];
  const double *l = logits + (size_t)blockIdx.x * vocab;
  double mx = -INFINITY;
  for (uint32_t c = threadIdx.x; c < vocab; c += 256) mx = fmax(mx, l[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = sh[0];
    for (int w = 1; w < 8; ++w) m = fmax(m, sh[w]);
    sh[32] = m;
  }
  __syncthreads();
  mx = sh[32];
  __syncthreads();
  double s = 0.0;
  for (uint32_t c = threadIdx.x; c < vocab; c += 256) s += exp(l[c] - mx);
  s = block_sum<256>(s, sh);
  if (threadIdx.x == 0) {
    const int64_t t = targets[blockIdx.x];
    row[blockIdx.x] = (t >= 0 && t < (int64_t)vocab) ? mx + log(s) - l[t] : NAN;
  }
}

// Fixed-order (deterministic) sum of the row losses into *sum.
__global__ void __launch_bounds__(1024) k_f64_sum(const double *row, uint64_t n, double *sum) {
  __shared__ double sh[33];
  double s = 0.0;
  for (uint64_t i = threadIdx.x; i < n; i += 1024) s += row[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += sh[w];
    *sum = t;
  }
}
}  // namespace

extern "C" int zo2_f64_gemm(const double *A, const double *B, int b_trans, const double *bias,
                            double *C, uint64_t M, uint64_t N, uint64_t K, int epi, void *cs) {
  if (M == 0 || N == 0) return ZO2_OK;
  if (!A || !B || !C) return zo2_set_error(ZO2_E_ARG, "zo2_f64_gemm: null operand");
  if (M > 0x7fffffffull || N > 0x7fffffffull || K > 0x7fffffffull || M / TM >= 65535)
    return zo2_set_error(ZO2_E_UNSUPPORTED, "zo2_f64_gemm: shape too large");
  if (epi < ZO2_F64_EPI_STORE || epi > ZO2_F64_EPI_RESIDUAL)
    return zo2_set_error(ZO2_E_ARG, "zo2_f64_gemm: unknown epilogue");
  dim3 grid((unsigned)((N + TN - 1) / TN), (unsigned)((M + TM - 1) / TM));
  if (b_trans)
    k_f64_gemm<true><<<grid, 256, 0, S(cs)>>>(A, B, bias, C, (int)M, (int)N, (int)K, epi);
  else
    k_f64_gemm<false><<<grid, 256, 0, S(cs)>>>(A, B, bias, C, (int)M, (int)N, (int)K, epi);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

extern "C" int zo2_f64_layernorm(const double *x, uint64_t rows, uint32_t dim, const double *g,
                                 const double *b, double *out, void *cs) {
  if (rows == 0) return ZO2_OK;
  if (rows > 0x7fffffffull) return zo2_set_error(ZO2_E_UNSUPPORTED, "zo2_f64_layernorm: rows");
  k_f64_layernorm<<<(unsigned)rows, 256, 0, S(cs)>>>(x, dim, g, b, out);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

extern "C" int zo2_f64_embed(const int64_t *ids, uint64_t n_tok, uint32_t seq, uint32_t dim,
                             const double *tok_emb, const double *pos_emb, double *out,
                             void *cs) {
  if (n_tok == 0) return ZO2_OK;
  if (seq == 0) return zo2_set_error(ZO2_E_ARG, "zo2_f64_embed: seq == 0");
  k_f64_embed<<<zo2_grid_for(n_tok * dim, 256), 256, 0, S(cs)>>>(ids, n_tok, seq, dim, tok_emb,
                                                                  pos_emb, out);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

extern "C" int zo2_f64_attention(const double *qkv, uint32_t batch, uint32_t seq,
                                 uint32_t n_heads, uint32_t head_dim, double *ctx, void *cs) {
  if (batch == 0 || seq == 0) return ZO2_OK;
  const size_t smem = (size_t)ATT_WARPS * (seq + head_dim) * sizeof(double);
  if (smem > 200 * 1024) return zo2_set_error(ZO2_E_UNSUPPORTED, "zo2_f64_attention: seq");
  static size_t opted = 0;
  if (smem > 48 * 1024 && smem > opted) {
    ZO2_CUDA_TRY(cudaFuncSetAttribute(k_f64_attention,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    opted = smem;
  }
  dim3 grid((seq + ATT_WARPS - 1) / ATT_WARPS, n_heads, batch);
  k_f64_attention<<<grid, ATT_WARPS * 32, smem, S(cs)>>>(qkv, seq, n_heads, head_dim, ctx);
  zo2_count_launch();
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}

extern "C" int zo2_f64_ce(const double *logits, const int64_t *targets, uint64_t rows,
                          uint32_t vocab, double *row_loss, double *d_sum, void *cs) {
  if (rows == 0) return ZO2_OK;
  if (rows > 0x7fffffffull) return zo2_set_error(ZO2_E_UNSUPPORTED, "zo2_f64_ce: rows");
  k_f64_ce_rows<<<(unsigned)rows, 256, 0, S(cs)>>>(logits, targets, vocab, row_loss);
  k_f64_sum<<<1, 1024, 0, S(cs)>>>(row_loss, rows, d_sum);
  zo2_count_launch(2);
  ZO2_CHECK_LAUNCH();
  return ZO2_OK;
}
