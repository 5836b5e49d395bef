/*
 * zo2b200.h -- C ABI of the B200 (sm_100a) ZO2 step library
 * (paper_2503_12668_b200/_lib/libzo2b200.so).
 *
 * The reference (zo2lab, /root/reference/pkg/src/zo2lab) is pure NumPy and
 * has no FFI; each entry point below replaces one computation of its
 * Python hot path, cited as file:line.  Conventions:
 *   - every function returns 0 (ZO2_OK) or a ZO2_E_* status; the Python host
 *     maps statuses onto the reference's exception taxonomy (errors.py:4-21);
 *     zo2_last_error() returns a message for the last failure.
 *   - device pointers are plain pointers allocated by the caller (torch);
 *     `stream` is a cudaStream_t passed as void*; nothing here allocates on
 *     the hot path and nothing synchronises unless its name ends in _sync.
 *   - host-side functions (zo2_host_*) touch host memory only.
 *   - element formats: ZO2_F64, ZO2_F32, ZO2_F16, ZO2_BF16, ZO2_F8E4M3 follow
 *     numerics.py:48-84 (ElemFormat); low-bit formats are storage only.
 */
#ifndef ZO2B200_H
#define ZO2B200_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:4-21) ---- */
#define ZO2_OK 0
#define ZO2_E_ARG 1          /* UsageError / ValueError               */
#define ZO2_E_CUDA 2         /* CUDA runtime failure (RuntimeError)   */
#define ZO2_E_CAPACITY 3     /* CapacityError                         */
#define ZO2_E_SCHED 4        /* SchedulingContractError               */
#define ZO2_E_STATE 5        /* StateCorruptionError                  */
#define ZO2_E_NONFINITE 6    /* NonFiniteLossError                    */
#define ZO2_E_UNSUPPORTED 7  /* shape/format outside the kernels' set */

/* ---- element formats (numerics.py:48-84) ---- */
#define ZO2_F64 0
#define ZO2_F32 1
#define ZO2_F16 2
#define ZO2_BF16 3
#define ZO2_F8E4M3 4

/* ---- RNG stream ids (numerics.py:42-45) ---- */
#define ZO2_PERTURB_STREAM 0
#define ZO2_BATCH_STREAM 1
#define ZO2_INIT_STREAM 2
#define ZO2_DATA_STREAM 3

const char *zo2_last_error(void);
int zo2_version(void);
/* number of kernel launches issued by this library since load (evidence for
 * bench.py's gpu_launches) */
uint64_t zo2_launch_count(void);

/* ======================= K1: counter-based Gaussian direction =========== */
/* numerics.py:171-182 gaussian_fill(RngState(seed, stream, counter), n):
 * out[i] = ndtri(((raw(counter+i) >> 11) + 0.5) * 2^-53), bit-exact. */
int zo2_z_fill(double *out, uint64_t n, uint64_t seed, uint64_t stream,
               uint64_t counter, void *cuda_stream);
/* numerics.py:161-168 raw_uint64. */
int zo2_raw_fill(uint64_t *out, uint64_t n, uint64_t seed, uint64_t stream,
                 uint64_t counter, void *cuda_stream);
/* Host restatements of the same generator (same source as the device code;
 * used by the host runtime for batch sampling, model.py:198-224 init is on
 * device). */
int zo2_host_raw_u64(uint64_t *out, uint64_t n, uint64_t seed,
                     uint64_t stream, uint64_t counter);
int zo2_host_gaussian_fill(double *out, uint64_t n, uint64_t seed,
                           uint64_t stream, uint64_t counter);
uint64_t zo2_host_derive_step_seed(uint64_t base_seed, uint64_t step_index);

/* z generator used by K2 (update / perturb / restore) and K8 (embedding):
 *   0 = reference-exact (default): the gaussian_fill stream above;
 *   1 = fast: Philox4x32-10 + binary32 erfinv (zo2_rng_fast.h) keyed on the
 *       same (seed, stream, absolute parameter position) -- self-consistent
 *       across every kernel, statistically equivalent, not the reference's
 *       values.  No reference counterpart (the reference has one generator).
 * Process-wide; read at kernel launch. */
int zo2_set_rng_mode(int mode);
int zo2_rng_mode(void);
/* The fast direction itself (binary32), device and host restatement. */
int zo2_z_fill_fast(float *out, uint64_t n, uint64_t seed, uint64_t stream,
                    uint64_t counter, void *cuda_stream);
int zo2_host_z_fill_fast(float *out, uint64_t n, uint64_t seed, uint64_t stream,
                         uint64_t counter);

/* model.py:198-224 init_params, one segment: out = fmt(std * z) with z drawn
 * at (seed, INIT_STREAM, counter); fmt is ZO2_F32 or ZO2_F64. */
int zo2_init_normal(void *out, int fmt, uint64_t n, double std, uint64_t seed,
                    uint64_t counter, void *cuda_stream);
int zo2_fill_const(void *out, int fmt, uint64_t n, double value,
                   void *cuda_stream);

/* ======================= K2: perturb / update ============================ */
/* model.py:227-233 axpy with regenerated z (zo_ref.py:59-74 perturb_all for
 * one bucket; zo2_engine.py:161-174 _perturb / _update_flat):
 *   w[i] = store(f64(w[i]) + coef * z(seed, stream, counter + i)).
 * fmt is ZO2_F32 or ZO2_F64. */
int zo2_axpy_z(void *w, int fmt, uint64_t n, double coef, uint64_t seed,
               uint64_t stream, uint64_t counter, void *cuda_stream);

/* Operand emission for one bucket segment during the fused update+perturb
 * (the dual forward's W+eps*z and W-eps*z). */
#define ZO2_OUT_NONE 0
#define ZO2_OUT_F32 1        /* f32 copy, same layout (vectors: LN g/b, biases) */
#define ZO2_OUT_BF16_T 2     /* bf16, transposed to [cols, rows] (K-major B)   */
#define ZO2_OUT_SPLIT_T 3    /* bf16 hi + bf16 lo planes, transposed           */
#define ZO2_OUT_BF16 4       /* bf16, same layout ([rows, cols] already K-major) */
#define ZO2_OUT_SPLIT 5      /* bf16 hi + lo planes, same layout               */
typedef struct zo2_segment_desc {
  uint64_t offset;       /* element offset in the bucket (= RNG offset)   */
  uint32_t rows, cols;   /* row-major segment shape; vectors rows = 1     */
  int32_t out_kind;      /* ZO2_OUT_*                                     */
  int32_t pad_;
  void *out_plus;        /* W + eps z   (hi plane for split kinds)        */
  void *out_minus;       /* W - eps z                                     */
  void *out_plus_lo;     /* lo planes (split kinds only)                  */
  void *out_minus_lo;
} zo2_segment_desc;

/* K2, fused per-module step arithmetic of zo2_engine.py:183-204 dual_forward:
 *   if (update && *d_g != 0):  w = st(w + (-(lr * *d_g)) * z(lrs_seed, 0, base+i))
 *   w+ = st(w + eps z(rs)); w- = st(w+ + (-2 eps) z(rs)); w = st(w- + eps z(rs))
 * (each st() is one axpy rounding, model.py:233).  update = 2 applies the
 * update without the g != 0 gate (naive update-after-forward,
 * zo2_engine.py:251-260).  `arena` holds the module
 * in `wire_fmt` (F64/F32, or a codec format decoded to F32 on read and
 * encoded on write, runtime.py:172-184); arithmetic is f64 when wire_fmt is
 * ZO2_F64 and f32 otherwise.  perturb=0 skips the +eps/-2eps/+eps sequence
 * (naive-mode update pass, finalize drain).  codec conversions tally into
 * d_conv_counts[0] (NaN) and [1] (saturated) if non-null (ConversionSummary,
 * numerics.py:210-217). */
/* Grid sizing of K2: 0 (default) = 148 x occupancy CTAs; n = at most n CTAs
 * per SM (the engine sets 1 when K2 runs on the prepare stream concurrently
 * with the GEMMs, operand_sets = 2). */
int zo2_set_k2_ctas_per_sm(int n);
/* K2 variant (process-wide).  0 (default): codec arenas (bf16 / f16 / e4m3
 * wire) with bf16 or no operands take the certified path -- binary32 chain on
 * an approximate z with a verified error bound, each output kept only when
 * its rounding is provably the exact chain's, else recomputed with the exact
 * z; bit-identical results.  1: always the queued exact kernel (A/B). */
int zo2_set_k2_variant(int variant);
/* Exhaustive check of the approximate z's bound (zo2_zapprox.cuh) over every
 * binary32 y in [2^-24, 1/2]; writes 32 floats to d_out (device): [0] max
 * |z~ - z| / tau, [1] max |z~ - z|, [2] mapping mismatches, [3 + b] max
 * |z~ - z| / (1 + |z~|) per binade of y.  Test support. */
int zo2_zapprox_bound_probe(float *d_out, void *cuda_stream);
/* Elements the certified K2 path recomputed with the exact z since the last
 * reset (synchronous read of a device counter; diagnostics and tests). */
int zo2_k2c_fallbacks(uint64_t *out, int reset);
int zo2_update_perturb(void *arena, int wire_fmt, uint64_t n, uint64_t base,
                       int update, const double *d_g, double lr,
                       uint64_t lrs_seed, int perturb, double eps,
                       uint64_t rs_seed, const zo2_segment_desc *segs,
                       int n_segs, uint64_t *d_conv_counts, void *cuda_stream);

/* ======================= host tier ===================================== */
/* cudaHostRegister(ptr, bytes, portable) / cudaHostUnregister: pins the
 * node-wide shared block masters of a data-parallel job (runtime.py
 * HostBlockStore, one copy per node instead of one per rank). */
int zo2_host_register(void *ptr, uint64_t bytes);
int zo2_host_unregister(void *ptr);

/* ======================= K9: wire codecs ================================= */
/* numerics.py:281-311 encode/decode; fmt in {ZO2_F16, ZO2_BF16, ZO2_F8E4M3}. */
int zo2_encode(const float *src, void *dst, int fmt, uint64_t n,
               uint64_t *d_conv_counts, void *cuda_stream);
int zo2_decode(const void *src, float *dst, int fmt, uint64_t n,
               void *cuda_stream);

/* ======================= K10: projected gradient ========================= */
/* zo2_engine.py:239-246: l+- = sums[0|1] / count ; g = (l+ - l-) / (2 eps).
 * Writes out[0]=l+, out[1]=l-, out[2]=g; out[2] is left at 0 and *d_flag=1
 * when either loss is non-finite (NonFiniteLossError is raised by the host). */
int zo2_form_g(const double *d_sums, double count, double eps, double *d_out,
               int *d_flag, void *cuda_stream);

/* ======================= forward kernels ================================= */
/* model.py:251-261 forward_embedding for both signs, with the module's
 * deferred update and perturbation recomputed for the gathered rows:
 *   out+-[t, c] = f32(tok+-[ids[t], c] + pos+-[t % S, c]).
 * `table` is the f32 embedding bucket ([V*d] tok then [S*d] pos) BEFORE this
 * step's update; base is the bucket's RNG offset (0 in canonical order). */
int zo2_embed_dual(const int64_t *ids, uint64_t n_tok, uint32_t seq,
                   uint32_t dim, uint32_t vocab, uint32_t max_seq,
                   const float *table, uint64_t base, int update,
                   const double *d_g, double lr, uint64_t lrs_seed,
                   double eps, uint64_t rs_seed, float *out_plus,
                   float *out_minus, void *cuda_stream);

/* model.py:241-244 _layer_norm (population variance, eps 1e-5) on f32 rows,
 * writing a GEMM A operand: bf16 (lo == NULL) or bf16 hi+lo planes. */
int zo2_layernorm(const float *x, uint64_t rows, uint32_t dim,
                  const float *gamma, const float *beta, void *out_hi,
                  void *out_lo, void *cuda_stream);

/* f32 activations -> GEMM A operand (bf16, or bf16 hi+lo planes when lo != NULL). */
int zo2_to_operand(const float *x, uint64_t n, void *out_hi, void *out_lo,
                   void *cuda_stream);

/* Generic sm_100a tcgen05 GEMM  C[M,N] = A[M,K] . B[N,K]^T  (both K-major
 * bf16, fp32 accumulation in TMEM), batched over `batch` independent
 * problems (the +eps and -eps forwards).  With split (A_lo, B_lo non-null)
 * it computes A_hi.B_hi + A_hi.B_lo + A_lo.B_hi (f32-faithful 3-pass bf16).
 * Epilogues (model.py:272-301):
 *   ZO2_EPI_STORE      C = acc + bias                (f32 out)
 *   ZO2_EPI_RESIDUAL   C += acc + bias               (f32 in/out, h + (x@W+b))
 *   ZO2_EPI_GELU       C = gelu_erf(acc + bias) as an operand (bf16 / split)
 *   ZO2_EPI_CE         cross-entropy partials of the head logits per
 *                      (row, n-tile): max, sum exp, target logit  (model.py:304)
 *   ZO2_EPI_OPERAND    C = acc + bias as bf16 (hi + lo) planes (qkv for attention)
 */
#define ZO2_EPI_STORE 0
#define ZO2_EPI_RESIDUAL 1
#define ZO2_EPI_GELU 2
#define ZO2_EPI_CE 3
#define ZO2_EPI_OPERAND 4
typedef struct zo2_gemm_problem {
  const void *a_hi, *a_lo;   /* [M, K] bf16                               */
  const void *b_hi, *b_lo;   /* [N, K] bf16                               */
  const float *bias;         /* [N] f32 or NULL                           */
  void *c;                   /* f32 [M, N] (STORE/RESIDUAL) / bf16 hi (GELU) */
  void *c_lo;                /* GELU split lo plane                       */
  const int64_t *targets;    /* CE: [M] target ids                        */
  float *ce_part;            /* CE: [M, n_tiles_n, 3] partials            */
} zo2_gemm_problem;
int zo2_gemm(const zo2_gemm_problem *probs, int batch, uint32_t M, uint32_t N,
             uint32_t K, int epilogue, void *cuda_stream);
/* Column width of the CE partials (CE partial count = ceil(N / width)). */
int zo2_gemm_tile_n(int split);
/* Kernel choice: 0 auto (CTA-pair cta_group::2 256x256 tiles when M >= 256,
 * N >= 256 and K > 1024, else single-CTA 128-row tiles), 1 single-CTA only,
 * 2 pair whenever legal.  For A/B measurements and tests. */
int zo2_set_gemm_variant(int variant);
/* Tile raster: groups of `group_m` M tiles visited n-major (1 = row-major).
 * 0 (default) = automatic: row-major when the whole B operand fits in 80 MB
 * of L2, else 12 (single-CTA kernel) / 8 (CTA-pair kernel).  For A/B
 * measurements; results do not depend on it. */
int zo2_set_gemm_raster(int group_m_cta, int group_m_pair);

/* Combine CE partials into per-problem token sums (f64): sums[b] =
 * sum_t (logsumexp_t - logit_t[target_t])  (model.py:304-313 numerator).
 * Fixed-order two-phase reduction (bitwise reproducible); d_work holds
 * batch * ZO2_CE_PARTS doubles. */
#define ZO2_CE_PARTS 148
int zo2_ce_reduce(const float *ce_part, uint32_t M, uint32_t n_tiles,
                  int batch, uint64_t part_stride, double *d_work,
                  double *d_sums, void *cuda_stream);

/* model.py:273-283 causal softmax attention on packed qkv given as bf16
 * planes [B*S, 3d] (hi, and lo when split; heads split as reshape(B,S,H,hd)),
 * writing ctx as an A operand (bf16 hi, + lo when split). */
/* 0 (default): the tcgen05/TMEM attention kernel where it applies (seq a
 * multiple of 128, head_dim 64, or 128 without split planes), else the
 * mma.sync kernel; 1: mma.sync kernel only (A/B). */
int zo2_set_attention_variant(int variant);
int zo2_attention(const void *qkv_hi, const void *qkv_lo, uint32_t batch,
                  uint32_t seq, uint32_t n_heads, uint32_t head_dim,
                  void *ctx_hi, void *ctx_lo, void *cuda_stream);

/* ======================= f64 forward (arith=f64) ========================
 * The reference's default arithmetic (harness/config.py:53): the forward of
 * model.py:241-313 in IEEE binary64, run by the engine between in-place
 * perturbation passes (zo2_axpy_z), exactly the reference's per-module
 * sequence (zo2_engine.py:183-204).  Row-major f64 tensors throughout. */
#define ZO2_F64_EPI_STORE 0     /* C = A@B + bias                          */
#define ZO2_F64_EPI_GELU 1      /* C = gelu_erf(A@B + bias)   (model.py _gelu) */
#define ZO2_F64_EPI_RESIDUAL 2  /* C = C + (A@B + bias)       (h + (x@W + b)) */
/* C[M,N] from A[M,K] and B [K,N] (b_trans 0) or [N,K] (b_trans 1: A@B^T,
 * the head's h @ W^T, model.py:301); bias [N] or NULL. */
int zo2_f64_gemm(const double *A, const double *B, int b_trans, const double *bias,
                 double *C, uint64_t M, uint64_t N, uint64_t K, int epi, void *cuda_stream);
/* model.py:259-262 _ln: (x - mean) / sqrt(var + 1e-5) * g + b per row. */
int zo2_f64_layernorm(const double *x, uint64_t rows, uint32_t dim, const double *gamma,
                      const double *beta, double *out, void *cuda_stream);
/* model.py:251-261: out[t] = tok_emb[ids[t]] + pos_emb[t % seq]. */
int zo2_f64_embed(const int64_t *ids, uint64_t n_tok, uint32_t seq, uint32_t dim,
                  const double *tok_emb, const double *pos_emb, double *out,
                  void *cuda_stream);
/* model.py:273-283 causal softmax attention on packed qkv [B*S, 3d] -> ctx [B*S, d]. */
int zo2_f64_attention(const double *qkv, uint32_t batch, uint32_t seq, uint32_t n_heads,
                      uint32_t head_dim, double *ctx, void *cuda_stream);
/* model.py:308-313: row_loss[r] = logsumexp(logits[r]) - logits[r, target[r]],
 * *d_sum = sum over rows in a fixed order (NaN rows for out-of-range targets). */
int zo2_f64_ce(const double *logits, const int64_t *targets, uint64_t rows, uint32_t vocab,
               double *row_loss, double *d_sum, void *cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* ZO2B200_H */
