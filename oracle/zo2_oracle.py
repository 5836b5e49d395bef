"""TEST INFRASTRUCTURE ONLY -- CPU parity oracle for the ZO2 step.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this module; the product package
(paper_2503_12668_b200) never does and has no CPU fallback.

A restatement of the reference's hot-path arithmetic (zo2lab, reference at
/root/reference/pkg/src/zo2lab), written for checking, not speed:
  RNG / axpy / codecs   C restatement in oracle/zo2_oracle.c (built by
                        `make -C oracle`): numerics.py:161-311, model.py:227-233
  forward               numpy, following model.py:241-313 (f32 or f64 like the
                        reference, logits -> f64 for the loss)
  init / data / batch   model.py:198-224, harness/data.py:35-62, zo_ref.py:49-56
  steps                 MeZO (zo_ref.py:97-112) and the deferred ZO2 step
                        (zo2_engine.py:183-204, :264-336) run sequentially --
                        lanes do not change the arithmetic.
Pinned by tests/golden/* generated from the reference itself
(tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np
from scipy.special import erf

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libzo2oracle.so")
_lib = None
U64 = ctypes.c_uint64


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        vp = ctypes.c_void_p
        L.oracle_raw_u64.argtypes = [U64, U64, U64, U64, vp]
        L.oracle_gaussian_fill.argtypes = [U64, U64, U64, U64, vp]
        L.oracle_gauss_at.argtypes = [U64, U64, U64, vp, U64, vp]
        L.oracle_derive_step_seed.argtypes = [U64, U64]
        L.oracle_derive_step_seed.restype = U64
        L.oracle_axpy_z_f32.argtypes = [vp, U64, ctypes.c_double, U64, U64, U64]
        L.oracle_axpy_z_f64.argtypes = [vp, U64, ctypes.c_double, U64, U64, U64]
        L.oracle_ndtri.argtypes = [ctypes.c_double]
        L.oracle_ndtri.restype = ctypes.c_double
        for name in ("oracle_encode_bf16", "oracle_encode_f16", "oracle_encode_e4m3"):
            getattr(L, name).argtypes = [vp, U64, vp, vp, vp]
        for name in ("oracle_decode_bf16", "oracle_decode_f16", "oracle_decode_e4m3"):
            getattr(L, name).argtypes = [vp, U64, vp]
        _lib = L
    return _lib


M64 = (1 << 64) - 1
PERTURB, BATCH, INIT, DATA = 0, 1, 2, 3


# ------------------------------------------------------------ numerics.py
def raw_u64(seed: int, stream: int, counter: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().oracle_raw_u64(seed & M64, stream & M64, counter & M64, n, out.ctypes.data)
    return out


def gauss(seed: int, stream: int, counter: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().oracle_gaussian_fill(seed & M64, stream & M64, counter & M64, n, out.ctypes.data)
    return out


# ------------------------------------------------------------ rng = "fast"
# Restatement of paper_2503_12668_b200/csrc/zo2_rng_fast.h (Philox4x32-10 +
# Giles' single-precision erfinv, every step one IEEE binary32 operation):
# the B200 fast direction must match it bit for bit.  Not a reference
# stream -- the reference's z is gauss() above.
_M32 = 0xFFFFFFFF


def fast_raw(seed: int, stream: int, counter: int, n: int) -> np.ndarray:
    pos = np.uint64(counter & M64) + np.arange(n, dtype=np.uint64)
    b = pos >> np.uint64(2)
    c0 = (b & np.uint64(_M32)).astype(np.uint32)
    c1 = (b >> np.uint64(32)).astype(np.uint32)
    c2 = np.full(n, stream & _M32, np.uint32)
    c3 = np.full(n, (stream >> 32) & _M32, np.uint32)
    k0, k1 = seed & _M32, (seed >> 32) & _M32
    for _ in range(10):
        p0 = np.uint64(0xD2511F53) * c0.astype(np.uint64)
        p1 = np.uint64(0xCD9E8D57) * c2.astype(np.uint64)
        hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & np.uint64(_M32)).astype(np.uint32)
        hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & np.uint64(_M32)).astype(np.uint32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint32(k0), lo1, hi0 ^ c3 ^ np.uint32(k1), lo0
        k0, k1 = (k0 + 0x9E3779B9) & _M32, (k1 + 0xBB67AE85) & _M32
    lanes = (pos & np.uint64(3)).astype(np.int64)
    return np.stack([c0, c1, c2, c3], 1)[np.arange(n), lanes]


def _f32(x):
    return np.asarray(x, dtype=np.float32)


def _fast_log(a: np.ndarray) -> np.ndarray:
    ia = a.view(np.uint32)
    e = ((ia >> np.uint32(23)) & np.uint32(0xFF)).astype(np.int32) - 127
    im = (ia & np.uint32(0x007FFFFF)) | np.uint32(0x3F800000)
    big = im > np.uint32(0x3FB504F3)
    im = np.where(big, im - np.uint32(0x00800000), im).astype(np.uint32)
    e = e + big.astype(np.int32)
    m = im.view(np.float32)
    one = np.float32(1.0)
    s = (m - one) / (m + one)
    s2 = s * s
    p = np.full(a.shape, np.float32(0.11111111), np.float32)
    for c in (0.14285715, 0.2, 0.33333334, 1.0):
        p = p * s2 + np.float32(c)
    lm = (np.float32(2.0) * s) * p
    return e.astype(np.float32) * np.float32(0.6931472) + lm


_GILES_A = (2.81022636e-08, 3.43273939e-07, -3.5233877e-06, -4.39150654e-06, 0.00021858087,
            -0.00125372503, -0.00417768164, 0.246640727, 1.50140941)
_GILES_B = (-0.000200214257, 0.000100950558, 0.00134934322, -0.00367342844, 0.00573950773,
            -0.0076224613, 0.00943887047, 1.00167406, 2.83297682)


def fast_gauss_from_raw(r: np.ndarray) -> np.ndarray:
    r = np.asarray(r, np.uint32)
    u = ((r >> np.uint32(9)).astype(np.float32) + np.float32(0.5)) * np.float32(1.1920929e-07)
    x = np.float32(2.0) * u - np.float32(1.0)
    a = (np.float32(4.0) * u) * (np.float32(1.0) - u)
    w = np.float32(0.0) - _fast_log(a)
    lo = w < np.float32(5.0)
    wa = w - np.float32(2.5)
    pa = np.full(r.shape, np.float32(_GILES_A[0]), np.float32)
    for c in _GILES_A[1:]:
        pa = np.float32(c) + pa * wa
    wb = np.sqrt(np.where(lo, np.float32(25.0), w)) - np.float32(3.0)
    pb = np.full(r.shape, np.float32(_GILES_B[0]), np.float32)
    for c in _GILES_B[1:]:
        pb = np.float32(c) + pb * wb
    p = np.where(lo, pa, pb)
    return np.float32(1.4142135) * (p * x)


def fast_gauss(seed: int, stream: int, counter: int, n: int) -> np.ndarray:
    return fast_gauss_from_raw(fast_raw(seed, stream, counter, n))


def axpy_z_fast(flat: np.ndarray, coef: float, seed: int, counter: int) -> None:
    """flat += coef * z_fast, f64 product and sum, one rounding (model.py:233
    arithmetic with the fast direction)."""
    if flat.size == 0:
        return
    z = fast_gauss(seed, PERTURB, counter, flat.size).astype(np.float64)
    flat[:] = (flat.astype(np.float64) + np.float64(coef) * z).astype(flat.dtype)


def gauss_at(seed: int, stream: int, counter: int, idx: np.ndarray) -> np.ndarray:
    """z(seed, stream, counter + idx[i]) for arbitrary positions (numerics.py:161-168)."""
    idx = np.ascontiguousarray(idx, np.uint64)
    out = np.empty(idx.size, np.float64)
    lib().oracle_gauss_at(seed & M64, stream & M64, counter & M64, idx.ctypes.data, idx.size,
                          out.ctypes.data)
    return out


def axpy_z_at(vals: np.ndarray, idx: np.ndarray, coef: float, seed: int,
              counter: int) -> np.ndarray:
    """vals[i] + coef * z(seed, PERTURB, counter + idx[i]) with axpy_z's single
    rounding (f64 product and sum, store in vals' dtype; model.py:227-233)."""
    z = gauss_at(seed, PERTURB, counter, idx)
    return (vals.astype(np.float64) + np.float64(coef) * z).astype(vals.dtype)


def derive_step_seed(base: int, j: int) -> int:
    return int(lib().oracle_derive_step_seed(base & M64, j & M64))


def axpy_z(flat: np.ndarray, coef: float, seed: int, counter: int) -> None:
    """flat += coef * z(seed, PERTURB, counter + i), one rounding (model.py:233)."""
    if flat.size == 0:
        return
    assert flat.flags.c_contiguous
    f = lib().oracle_axpy_z_f32 if flat.dtype == np.float32 else lib().oracle_axpy_z_f64
    f(flat.ctypes.data, flat.size, float(coef), seed & M64, PERTURB, counter & M64)


def encode(x: np.ndarray, fmt: str):
    x = np.ascontiguousarray(x, np.float32)
    counts = np.zeros(2, np.uint64)
    out = np.empty(x.size, np.uint8 if fmt == "f8" else np.uint16)
    fn = {"bf16": "oracle_encode_bf16", "f16": "oracle_encode_f16", "f8": "oracle_encode_e4m3"}[fmt]
    getattr(lib(), fn)(x.ctypes.data, x.size, out.ctypes.data, counts[0:].ctypes.data,
                       counts[1:].ctypes.data)
    return out, int(counts[0]), int(counts[1])


def decode(bits: np.ndarray, fmt: str) -> np.ndarray:
    bits = np.ascontiguousarray(bits)
    out = np.empty(bits.size, np.float32)
    fn = {"bf16": "oracle_decode_bf16", "f16": "oracle_decode_f16", "f8": "oracle_decode_e4m3"}[fmt]
    getattr(lib(), fn)(bits.ctypes.data, bits.size, out.ctypes.data)
    return out


# ------------------------------------------------------------ model.py
@dataclass(frozen=True)
class Spec:
    n_blocks: int
    dim: int
    n_heads: int
    vocab: int
    seq_len: int
    tie_lm_head: bool = False


def layouts(spec: Spec) -> dict[str, list[tuple[str, tuple]]]:
    d = spec.dim
    blk = [("ln1_g", (d,)), ("ln1_b", (d,)), ("qkv_w", (d, 3 * d)), ("qkv_b", (3 * d,)),
           ("attn_out_w", (d, d)), ("attn_out_b", (d,)), ("ln2_g", (d,)), ("ln2_b", (d,)),
           ("mlp_in_w", (d, 4 * d)), ("mlp_in_b", (4 * d,)), ("mlp_out_w", (4 * d, d)),
           ("mlp_out_b", (d,))]
    out = {"embed": [("tok_emb", (spec.vocab, d)), ("pos_emb", (spec.seq_len, d))]}
    for i in range(spec.n_blocks):
        out[f"block.{i}"] = blk
    out["head"] = [] if spec.tie_lm_head else [("head_w", (spec.vocab, d))]
    return out


def views(flat: np.ndarray, layout) -> dict[str, np.ndarray]:
    v, off = {}, 0
    for name, shape in layout:
        n = math.prod(shape)
        v[name] = flat[off:off + n].reshape(shape)
        off += n
    return v


def init_params(spec: Spec, seed: int, dtype=np.float32) -> dict[str, np.ndarray]:
    """model.py:198-224."""
    params, ctr = {}, 0
    for m, lay in layouts(spec).items():
        n = sum(math.prod(s) for _, s in lay)
        flat = np.zeros(n, dtype)
        vv = views(flat, lay)
        for name, shape in lay:
            if name.endswith("_g"):
                vv[name][...] = 1.0
            elif name.endswith("_b"):
                vv[name][...] = 0.0
            else:
                if name == "head_w":
                    std = 0.2 / math.sqrt(spec.dim)
                elif name in ("tok_emb", "pos_emb"):
                    std = 1.0 / math.sqrt(spec.dim)
                else:
                    std = 1.0 / math.sqrt(shape[0])
                z = gauss(seed, INIT, ctr, math.prod(shape))
                ctr += z.size
                vv[name][...] = (std * z).reshape(shape).astype(dtype)
        params[m] = flat
    return params


def _ln(x, g, b):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + x.dtype.type(1e-5)) * g + b


def _gelu(x):
    return 0.5 * x * (1.0 + erf(x / np.sqrt(x.dtype.type(2.0))))


def fwd_embed(spec, flat, tokens):
    v = views(flat, layouts(spec)["embed"])
    return v["tok_emb"][tokens] + v["pos_emb"][: tokens.shape[1]]


def fwd_block(spec, flat, h):
    v = views(flat, layouts(spec)["block.0"])
    B, S, d = h.shape
    H = spec.n_heads
    hd = d // H
    x = _ln(h, v["ln1_g"], v["ln1_b"])
    qkv = x @ v["qkv_w"] + v["qkv_b"]
    q, k, vv = (t.reshape(B, S, H, hd).transpose(0, 2, 1, 3) for t in np.split(qkv, 3, -1))
    sc = q @ k.transpose(0, 1, 3, 2) / np.sqrt(h.dtype.type(hd))
    sc = np.where(np.tril(np.ones((S, S), bool)), sc, h.dtype.type(-np.inf))
    sc = sc - sc.max(-1, keepdims=True)
    w = np.exp(sc)
    w = w / w.sum(-1, keepdims=True)
    ctx = (w @ vv).transpose(0, 2, 1, 3).reshape(B, S, d)
    h = h + (ctx @ v["attn_out_w"] + v["attn_out_b"])
    x = _ln(h, v["ln2_g"], v["ln2_b"])
    return h + (_gelu(x @ v["mlp_in_w"] + v["mlp_in_b"]) @ v["mlp_out_w"] + v["mlp_out_b"])


def ce_loss(logits, targets) -> float:
    lg = logits.astype(np.float64, copy=False)
    m = lg.max(-1, keepdims=True)
    lse = m[..., 0] + np.log(np.exp(lg - m).sum(-1))
    picked = np.take_along_axis(lg, targets[..., None], -1)[..., 0]
    return float((lse - picked).mean())


def full_loss(spec, params, tokens, targets, head_w=None) -> float:
    h = fwd_embed(spec, params["embed"], tokens)
    for i in range(spec.n_blocks):
        h = fwd_block(spec, params[f"block.{i}"], h)
    if head_w is None:
        head_w = (views(params["embed"], layouts(spec)["embed"])["tok_emb"] if spec.tie_lm_head
                  else params["head"].reshape(spec.vocab, spec.dim))
    return ce_loss(h @ head_w.T, targets)


def offsets(spec) -> dict[str, int]:
    out, c = {}, 0
    for m, lay in layouts(spec).items():
        out[m] = c
        c += sum(math.prod(s) for _, s in lay)
    return out


# ------------------------------------------------------------ data / batches
def gen_synthetic(vocab, seq_len, n_samples, seed, pattern="affine"):
    """harness/data.py:35-62."""
    if pattern == "copy":
        raw = raw_u64(seed, DATA, 0, n_samples * seq_len)
        tok = (raw % np.uint64(vocab)).astype(np.int64).reshape(n_samples, seq_len)
        return tok, tok.copy()
    start = (raw_u64(seed, DATA, 0, n_samples) % np.uint64(vocab)).astype(np.int64)
    seq = np.empty((n_samples, seq_len + 1), np.int64)
    seq[:, 0] = start
    for t in range(seq_len):
        seq[:, t + 1] = (5 * seq[:, t] + 3) % vocab
    return seq[:, :-1].copy(), seq[:, 1:].copy()


def batch_for_step(seed, j, n_samples, batch_size):
    """zo_ref.py:49-56."""
    raw = raw_u64(derive_step_seed(seed, j), BATCH, 0, batch_size)
    return (raw % np.uint64(n_samples)).astype(np.int64)


# ------------------------------------------------------------ engines
class MeZO:
    """zo_ref.py:97-112, sequential restatement."""

    def __init__(self, spec, params, eps, lr, seed, rng="exact"):
        self.spec, self.p, self.eps, self.lr, self.seed = spec, params, eps, lr, seed
        self.losses, self.gs, self.losses_minus = [], [], []
        self.off = offsets(spec)
        self.axpy = axpy_z_fast if rng == "fast" else axpy_z

    def _all(self, coef, s):
        for m, flat in self.p.items():
            self.axpy(flat, coef, s, self.off[m])

    def step(self, tokens, targets, j, g_override=None) -> float:
        s = derive_step_seed(self.seed, j)
        self._all(self.eps, s)
        lp = full_loss(self.spec, self.p, tokens, targets)
        self._all(-2.0 * self.eps, s)
        lm = full_loss(self.spec, self.p, tokens, targets)
        self._all(self.eps, s)
        if not (math.isfinite(lp) and math.isfinite(lm)):
            raise FloatingPointError(f"non-finite loss at step {j}")
        g = (lp - lm) / (2.0 * self.eps)
        self.losses.append(lp)
        self.losses_minus.append(lm)
        self.gs.append(g)
        if g_override is not None:
            g = g_override
        self._all(-(self.lr * g), s)
        return g


def axpy_z_threaded(flat: np.ndarray, coef: float, seed: int, counter: int, pool) -> None:
    """axpy_z over disjoint chunks in a thread pool (ctypes releases the GIL):
    z positions are absolute (numerics.py:161-168), so the bytes equal one call."""
    n, step = flat.size, 1 << 22
    list(pool.map(lambda o: axpy_z(flat[o:o + step], coef, seed, counter + o),
                  range(0, n, step)))


def codec_roundtrip_threaded(flat: np.ndarray, fmt: str, pool) -> None:
    """The reference's offload encode + upload decode of one block master
    (runtime.py:145-199), chunk-parallel: flat <- decode(encode(flat))."""
    step = 1 << 22

    def job(o):
        flat[o:o + step] = decode(encode(flat[o:o + step], fmt)[0], fmt)
    list(pool.map(job, range(0, flat.size, step)))


class Zo2Sequential:
    """The deferred per-module ZO2 step (zo2_engine.py:183-204, :264-336),
    executed module by module on the CPU; used as the timed CPU baseline.

    pool: optional thread pool for the RNG passes and the wire codec; codec:
    the AMP wire format of transferable blocks (upload decode + offload encode
    per block per step); self.t accumulates seconds per (module kind, phase)
    for the bench's explicit full-depth extrapolation."""

    def __init__(self, spec, params, eps, lr, seed, pool=None, codec=None):
        self.spec, self.p, self.eps, self.lr, self.seed = spec, params, eps, lr, seed
        self.off = offsets(spec)
        self.pending_g, self.lrs_seed = 0.0, None
        self.losses, self.gs = [], []
        self.pool, self.codec = pool, codec
        self.t: dict = {}

    def _axpy(self, flat, coef, seed, ctr):
        if self.pool is None:
            axpy_z(flat, coef, seed, ctr)
        else:
            axpy_z_threaded(flat, coef, seed, ctr, self.pool)

    def _tick(self, m, phase, t0):
        import time
        kind = "block" if m.startswith("block.") else m
        now = time.perf_counter()
        self.t[(kind, phase)] = self.t.get((kind, phase), 0.0) + now - t0
        return now

    def _module(self, m, x_plus, x_minus, s):
        import time
        flat = self.p[m]
        t0 = time.perf_counter()
        block = m.startswith("block.")
        if block and self.codec:
            codec_roundtrip_threaded(flat, self.codec, self.pool)  # upload + last offload
            t0 = self._tick(m, "codec", t0)
        if self.pending_g != 0.0 and flat.size:
            self._axpy(flat, -(self.lr * self.pending_g), self.lrs_seed, self.off[m])
        self._axpy(flat, self.eps, s, self.off[m])
        t0 = self._tick(m, "rng", t0)
        op = self._fwd(m, x_plus)
        t0 = self._tick(m, "fwd", t0)
        self._axpy(flat, -2.0 * self.eps, s, self.off[m])
        t0 = self._tick(m, "rng", t0)
        om = self._fwd(m, x_minus)
        t0 = self._tick(m, "fwd", t0)
        self._axpy(flat, self.eps, s, self.off[m])
        self._tick(m, "rng", t0)
        return op, om

    def _fwd(self, m, x):
        if m == "embed":
            return fwd_embed(self.spec, self.p["embed"], x)
        if m == "head":
            return x @ self.p["head"].reshape(self.spec.vocab, self.spec.dim).T
        return fwd_block(self.spec, self.p[m], x)

    def step(self, tokens, targets, j) -> float:
        s = derive_step_seed(self.seed, j)
        xp, xm = tokens, tokens
        for m in self.p:
            xp, xm = self._module(m, xp, xm, s)
        import time
        t0 = time.perf_counter()
        lp, lm = ce_loss(xp, targets), ce_loss(xm, targets)
        self._tick("head", "fwd", t0)
        g = (lp - lm) / (2.0 * self.eps)
        self.pending_g, self.lrs_seed = g, s
        self.losses.append(lp)
        self.gs.append(g)
        return g

    def finalize(self):
        if self.pending_g != 0.0:
            for m, flat in self.p.items():
                axpy_z(flat, -(self.lr * self.pending_g), self.lrs_seed, self.off[m])
        self.pending_g = 0.0
        return self.p
