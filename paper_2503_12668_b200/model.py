"""Model geometry and the device-side dual forward.

Geometry (ModelSpec, bucket layouts, canonical module order, init plan) keeps
the reference's names and frozen segment order (zo2lab model.py:30-224): the
segment order IS the RNG offset contract, so a parameter's z
lives at (module RNG base + flat index) in both implementations.

DualForward owns the HBM working set of one engine and drives the sm_100a
kernels for one module's dual forward (both perturbation signs at once):
  embed  model.py:251-261   zo2_embed_dual (gather + on-the-fly W+-eps z)
  block  model.py:264-288   LN -> QKV GEMM -> attention -> out GEMM(+res)
                            -> LN -> MLP-in GEMM(+GELU) -> MLP-out GEMM(+res)
  head   model.py:291-313   head GEMM with fused cross-entropy partials
HBM layout: residual streams h+- are f32 [T, d]; GEMM A operands are bf16
(arith=bf16) or bf16 hi+lo planes (arith=f32) [T, K]; weight operands W+-eps z
are emitted by K2 already transposed to [N, K] (K-major) so both tcgen05
operands load with the same TMA/UMMA 128B-swizzle layout.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _lib

LN_EPS = 1e-5            # model.py:20
EMBED_ID = "embed"       # model.py:22
HEAD_ID = "head"         # model.py:23
HEAD_INIT_SCALE = 0.2    # model.py:184


def block_id(i: int) -> str:
    return f"block.{i}"


@dataclass(frozen=True)
class ModelSpec:
    """model.py:30-50."""

    n_blocks: int
    dim: int
    n_heads: int
    vocab: int
    seq_len: int
    tie_lm_head: bool = False

    def __post_init__(self):
        for name in ("n_blocks", "dim", "n_heads", "vocab", "seq_len"):
            if getattr(self, name) < 1:
                raise ValueError(f"ModelSpec.{name} must be >= 1")
        if self.dim % self.n_heads != 0:
            raise ValueError(f"dim {self.dim} not divisible by n_heads {self.n_heads}")

    @property
    def head_dim(self) -> int:
        return self.dim // self.n_heads


@dataclass(frozen=True)
class Segment:
    name: str
    offset: int
    shape: tuple[int, ...]

    @property
    def size(self) -> int:
        return math.prod(self.shape)


def embed_layout(spec: ModelSpec):
    return [("tok_emb", (spec.vocab, spec.dim)), ("pos_emb", (spec.seq_len, spec.dim))]


def block_layout(spec: ModelSpec):
    d = spec.dim
    return [("ln1_g", (d,)), ("ln1_b", (d,)), ("qkv_w", (d, 3 * d)), ("qkv_b", (3 * d,)),
            ("attn_out_w", (d, d)), ("attn_out_b", (d,)), ("ln2_g", (d,)), ("ln2_b", (d,)),
            ("mlp_in_w", (d, 4 * d)), ("mlp_in_b", (4 * d,)), ("mlp_out_w", (4 * d, d)),
            ("mlp_out_b", (d,))]


def head_layout(spec: ModelSpec):
    return [] if spec.tie_lm_head else [("head_w", (spec.vocab, spec.dim))]


def segments(layout) -> list[Segment]:
    out, off = [], 0
    for name, shape in layout:
        out.append(Segment(name, off, tuple(shape)))
        off += math.prod(shape)
    return out


def module_order(spec: ModelSpec) -> list[str]:
    """Canonical whole-model order (model.py:166-171)."""
    return [EMBED_ID] + [block_id(i) for i in range(spec.n_blocks)] + [HEAD_ID]


def module_layout(spec: ModelSpec, module: str):
    if module == EMBED_ID:
        return embed_layout(spec)
    if module == HEAD_ID:
        return head_layout(spec)
    return block_layout(spec)


def module_size(spec: ModelSpec, module: str) -> int:
    return sum(math.prod(s) for _, s in module_layout(spec, module))


def param_count(spec: ModelSpec) -> int:
    return sum(module_size(spec, m) for m in module_order(spec))


def rng_offsets(spec: ModelSpec) -> dict[str, int]:
    """Counter base of each module's z: perturb_all / dual_forward advance the
    PERTURB_STREAM state by each bucket's size in canonical order
    (zo_ref.py:59-74, zo2_engine.py:203)."""
    out, c = {}, 0
    for m in module_order(spec):
        out[m] = c
        c += module_size(spec, m)
    return out


def _init_std(name: str, shape, dim: int) -> float:
    """model.py:187-195."""
    if name == "head_w":
        return HEAD_INIT_SCALE / math.sqrt(dim)
    if name in ("tok_emb", "pos_emb"):
        return 1.0 / math.sqrt(dim)
    return 1.0 / math.sqrt(shape[0])


def init_plan(spec: ModelSpec) -> dict[str, list[tuple[Segment, str, float, int]]]:
    """Per module: (segment, kind, std, INIT_STREAM counter) in the order
    init_params consumes draws (model.py:198-224): gains = 1, biases = 0,
    weights = std * z with the counter advancing only over weights."""
    plan, counter = {}, 0
    for m in module_order(spec):
        rows = []
        for seg in segments(module_layout(spec, m)):
            if seg.name.endswith("_g"):
                rows.append((seg, "one", 0.0, 0))
            elif seg.name.endswith("_b"):
                rows.append((seg, "zero", 0.0, 0))
            else:
                rows.append((seg, "normal", _init_std(seg.name, seg.shape, spec.dim), counter))
                counter += seg.size
        plan[m] = rows
    return plan


def init_module_(spec: ModelSpec, module: str, seed: int, out: torch.Tensor,
                 stream: torch.cuda.Stream | None = None) -> None:
    """Deterministic init of one module bucket on device (f32 or f64),
    bit-identical to init_params(spec, RngState(seed), fmt) (model.py:198-224)."""
    fmt = {torch.float32: _lib.F32, torch.float64: _lib.F64}[out.dtype]
    s = (stream or torch.cuda.current_stream()).cuda_stream
    esz = out.element_size()
    base = out.data_ptr()
    for seg, kind, std, ctr in init_plan(spec)[module]:
        ptr = base + seg.offset * esz
        if kind == "one":
            _lib.call("zo2_fill_const", ptr, fmt, seg.size, 1.0, s)
        elif kind == "zero":
            _lib.call("zo2_fill_const", ptr, fmt, seg.size, 0.0, s)
        else:
            _lib.call("zo2_init_normal", ptr, fmt, seg.size, std, int(seed), ctr, s)


# ----------------------------------------------------------------------------
# Device dual forward
# ----------------------------------------------------------------------------

def _bf16(n: int, dev) -> torch.Tensor:
    return torch.empty(n, dtype=torch.bfloat16, device=dev)


class _Operand:
    """A GEMM operand: one bf16 plane, or bf16 hi + lo planes (split)."""

    def __init__(self, n: int, split: bool, dev):
        self.hi = _bf16(n, dev)
        self.lo = _bf16(n, dev) if split else None

    @property
    def nbytes(self) -> int:
        return self.hi.numel() * 2 * (2 if self.lo is not None else 1)

    def ptrs(self):
        return self.hi.data_ptr(), (self.lo.data_ptr() if self.lo is not None else None)


class DualForward:
    """HBM working set + kernel sequence for the dual forward of one engine."""

    def __init__(self, spec: ModelSpec, batch_size: int, arith: str, device,
                 operand_sets: int = 1):
        if arith not in ("f32", "bf16"):
            raise ValueError(f"device forward supports arith f32 (3-pass bf16 split) or bf16, "
                             f"got {arith!r}")
        if spec.dim % 8 != 0:
            raise ValueError("device forward needs dim % 8 == 0 (TMA row alignment)")
        self.spec, self.B, self.arith = spec, int(batch_size), arith
        self.split = arith == "f32"
        self.dev = torch.device(device)
        d, V = spec.dim, spec.vocab
        T = self.T = self.B * spec.seq_len
        dev = self.dev
        split = self.split
        # residual streams and activations, one per sign
        self.h = [torch.empty(T * d, dtype=torch.float32, device=dev) for _ in range(2)]
        self.xop = [_Operand(T * d, split, dev) for _ in range(2)]
        self.qkv = [_Operand(T * 3 * d, split, dev) for _ in range(2)]
        self.ctx = [_Operand(T * d, split, dev) for _ in range(2)]
        self.mid = [_Operand(T * 4 * d, split, dev) for _ in range(2)]
        # block operands W +- eps z (vectors f32, matrices [N, K] bf16 planes),
        # `operand_sets` copies so K2 of block i+1 overlaps the forward of block i
        self.block_segs = segments(block_layout(spec))
        self.sets = []
        for _ in range(operand_sets):
            vec, mat = {}, {}
            for seg in self.block_segs:
                if len(seg.shape) == 1:
                    vec[seg.name] = [torch.empty(seg.size, dtype=torch.float32, device=dev)
                                     for _ in range(2)]
                else:
                    mat[seg.name] = [_Operand(seg.size, split, dev) for _ in range(2)]
            self.sets.append((vec, mat))
        # head operands [V, d] (head_w, or the tied tok_emb)
        self.head_op = [_Operand(V * d, split, dev) for _ in range(2)]
        self.tile_n = _lib.load().zo2_gemm_tile_n(1 if split else 0)
        self.n_tiles_v = (V + self.tile_n - 1) // self.tile_n
        self.ce_all = torch.empty(2, T * self.n_tiles_v * 3, dtype=torch.float32, device=dev)
        self.ce_part = [self.ce_all[0], self.ce_all[1]]
        self.d_sums = torch.zeros(2, dtype=torch.float64, device=dev)
        self.d_ce_work = torch.zeros(2 * _lib.CE_PARTS, dtype=torch.float64, device=dev)
        # optional live kernel timing: list of (kind, work, start_evt, end_evt)
        self.prof: list | None = None
        self.ids = torch.empty(T, dtype=torch.int64, device=dev)
        self.targets = torch.empty(T, dtype=torch.int64, device=dev)
        self._seg_cache: dict = {}

    # ---------------------------------------------------------------- sizes
    @staticmethod
    def estimate_nbytes(spec: ModelSpec, batch_size: int, arith: str,
                        operand_sets: int = 1) -> int:
        """Bytes the constructor allocates (same accounting as nbytes())."""
        d, V, T = spec.dim, spec.vocab, int(batch_size) * spec.seq_len
        ob = 4 if arith == "f32" else 2  # operand bytes per element (split: hi + lo)
        act = 2 * T * d * 4 + 2 * ob * T * (d + 3 * d + d + 4 * d)
        segs = segments(block_layout(spec))
        per_set = sum(2 * sg.size * (4 if len(sg.shape) == 1 else ob) for sg in segs)
        act += 2 * T * ((V + 127) // 128) * 3 * 4  # CE partials (N tile >= 128)
        return act + operand_sets * per_set + 2 * V * d * ob + 2 * T * 8

    def nbytes(self) -> dict[str, int]:
        act = sum(t.numel() * t.element_size() for t in self.h)
        act += sum(o.nbytes for o in self.xop + self.ctx + self.mid + self.qkv)
        act += self.ce_all.numel() * 4
        ops = sum(o.nbytes for _, mat in self.sets for pair in mat.values() for o in pair)
        ops += sum(t.numel() * 4 for vec, _ in self.sets for pair in vec.values() for t in pair)
        ops += sum(o.nbytes for o in self.head_op)
        return {"activations": act, "operands": ops, "io": 2 * self.T * 8}

    # ---------------------------------------------------------------- K2 descriptors
    def block_descs(self, set_idx: int = 0):
        key = ("block", set_idx)
        vec, mat = self.sets[set_idx]
        if key not in self._seg_cache:
            arr = (_lib.SegmentDesc * len(self.block_segs))()
            for k, seg in enumerate(self.block_segs):
                dsc = arr[k]
                dsc.offset = seg.offset
                if len(seg.shape) == 1:
                    dsc.rows, dsc.cols = 1, seg.shape[0]
                    dsc.out_kind = _lib.OUT_F32
                    dsc.out_plus = vec[seg.name][0].data_ptr()
                    dsc.out_minus = vec[seg.name][1].data_ptr()
                else:
                    dsc.rows, dsc.cols = seg.shape
                    dsc.out_kind = _lib.OUT_SPLIT_T if self.split else _lib.OUT_BF16_T
                    p_hi, p_lo = mat[seg.name][0].ptrs()
                    m_hi, m_lo = mat[seg.name][1].ptrs()
                    dsc.out_plus, dsc.out_minus = p_hi, m_hi
                    dsc.out_plus_lo, dsc.out_minus_lo = p_lo, m_lo
            self._seg_cache[key] = arr
        return self._seg_cache[key]

    def head_descs(self):
        """head_w [V, d] is already K-major for h @ W^T (model.py:301)."""
        key = "head"
        if key not in self._seg_cache:
            arr = (_lib.SegmentDesc * 1)()
            dsc = arr[0]
            dsc.offset, dsc.rows, dsc.cols = 0, self.spec.vocab, self.spec.dim
            dsc.out_kind = _lib.OUT_SPLIT if self.split else _lib.OUT_BF16
            p_hi, p_lo = self.head_op[0].ptrs()
            m_hi, m_lo = self.head_op[1].ptrs()
            dsc.out_plus, dsc.out_minus, dsc.out_plus_lo, dsc.out_minus_lo = p_hi, m_hi, p_lo, m_lo
            self._seg_cache[key] = arr
        return self._seg_cache[key]

    def embed_descs(self):
        """Embedding bucket: in-place update/perturb/restore; with a tied head the
        tok_emb W+- become the head operands (model.py:367-369 stash)."""
        key = "embed"
        if key not in self._seg_cache:
            segs = segments(embed_layout(self.spec))
            arr = (_lib.SegmentDesc * len(segs))()
            for k, seg in enumerate(segs):
                dsc = arr[k]
                dsc.offset = seg.offset
                dsc.rows, dsc.cols = seg.shape
                dsc.out_kind = _lib.OUT_NONE
                if self.spec.tie_lm_head and seg.name == "tok_emb":
                    dsc.out_kind = _lib.OUT_SPLIT if self.split else _lib.OUT_BF16
                    p_hi, p_lo = self.head_op[0].ptrs()
                    m_hi, m_lo = self.head_op[1].ptrs()
                    dsc.out_plus, dsc.out_minus = p_hi, m_hi
                    dsc.out_plus_lo, dsc.out_minus_lo = p_lo, m_lo
            self._seg_cache[key] = arr
        return self._seg_cache[key]

    # ---------------------------------------------------------------- kernels
    def _gemm(self, a_ops, b_ops, bias, c, c_lo, M, N, K, epi, stream, targets=None,
              ce=None):
        probs = (_lib.GemmProblem * 2)()
        for s in range(2):
            pr = probs[s]
            pr.a_hi, pr.a_lo = a_ops[s].ptrs()
            pr.b_hi, pr.b_lo = b_ops[s].ptrs()
            pr.bias = bias[s].data_ptr() if bias is not None else None
            pr.c = c[s] if c is not None else None
            pr.c_lo = c_lo[s] if c_lo is not None else None
            pr.targets = targets.data_ptr() if targets is not None else None
            pr.ce_part = ce[s].data_ptr() if ce is not None else None
        if self.prof is not None:
            st = torch.cuda.ExternalStream(stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.call("zo2_gemm", probs, 2, M, N, K, epi, stream)
            e1.record(st)
            # algorithmic work of this launch: 2 problems x 2MNK flops
            self.prof.append(("gemm", 2 * 2.0 * M * N * K, e0, e1))
            return
        _lib.call("zo2_gemm", probs, 2, M, N, K, epi, stream)

    def embed_forward(self, table: torch.Tensor, base: int, update: bool, d_g, lr: float,
                      lrs_seed: int, eps: float, rs_seed: int, seq: int, stream) -> None:
        spec = self.spec
        _lib.call("zo2_embed_dual", self.ids.data_ptr(), self.T, seq, spec.dim, spec.vocab,
                  spec.seq_len, table.data_ptr(), base, int(update),
                  d_g.data_ptr() if d_g is not None else None, lr, lrs_seed, eps, rs_seed,
                  self.h[0].data_ptr(), self.h[1].data_ptr(), stream)

    def block_forward(self, stream, set_idx: int = 0) -> None:
        spec = self.spec
        d, T, H = spec.dim, self.T, spec.n_heads
        V, Wm = self.sets[set_idx]
        for s in range(2):
            hi, lo = self.xop[s].ptrs()
            _lib.call("zo2_layernorm", self.h[s].data_ptr(), T, d, V["ln1_g"][s].data_ptr(),
                      V["ln1_b"][s].data_ptr(), hi, lo, stream)
        # qkv = x @ W_qkv + b, emitted directly as the attention's bf16 planes
        self._gemm(self.xop, Wm["qkv_w"], V["qkv_b"], [o.hi.data_ptr() for o in self.qkv],
                   [o.lo.data_ptr() for o in self.qkv] if self.split else None,
                   T, 3 * d, d, _lib.EPI_OPERAND, stream)
        for s in range(2):
            hi, lo = self.ctx[s].ptrs()
            qh, ql = self.qkv[s].ptrs()
            _lib.call("zo2_attention", qh, ql, self.B, spec.seq_len, H, spec.head_dim, hi, lo,
                      stream)
        self._gemm(self.ctx, Wm["attn_out_w"], V["attn_out_b"],
                   [t.data_ptr() for t in self.h], None, T, d, d, _lib.EPI_RESIDUAL, stream)
        for s in range(2):
            hi, lo = self.xop[s].ptrs()
            _lib.call("zo2_layernorm", self.h[s].data_ptr(), T, d, V["ln2_g"][s].data_ptr(),
                      V["ln2_b"][s].data_ptr(), hi, lo, stream)
        self._gemm(self.xop, Wm["mlp_in_w"], V["mlp_in_b"],
                   [o.hi.data_ptr() for o in self.mid],
                   [o.lo.data_ptr() for o in self.mid] if self.split else None,
                   T, 4 * d, d, _lib.EPI_GELU, stream)
        self._gemm(self.mid, Wm["mlp_out_w"], V["mlp_out_b"],
                   [t.data_ptr() for t in self.h], None, T, d, 4 * d, _lib.EPI_RESIDUAL, stream)

    def head_forward(self, stream) -> None:
        """logits = h @ W^T (model.py:301) -> CE partials -> per-sign token sums."""
        spec = self.spec
        d, T = spec.dim, self.T
        # the head GEMM reads h as an A operand: convert residual stream to planes
        for s in range(2):
            hi, lo = self.xop[s].ptrs()
            _lib.call("zo2_to_operand", self.h[s].data_ptr(), T * d, hi, lo, stream)
        self._gemm(self.xop, self.head_op, None, None, None, T, spec.vocab, d, _lib.EPI_CE,
                   stream, targets=self.targets, ce=self.ce_part)
        _lib.call("zo2_ce_reduce", self.ce_all.data_ptr(), T, self.n_tiles_v, 2,
                  self.ce_all.shape[1], self.d_ce_work.data_ptr(), self.d_sums.data_ptr(),
                  stream)


class F64Forward:
    """arith=f64 (the reference's default, harness/config.py:53): the forward
    of one perturbation sign in IEEE binary64 (csrc/zo2_f64.cu), reading the
    module's bucket in place.  The engine perturbs the bucket around the two
    forwards exactly as the reference does (+eps, -2eps, +eps with zo2_axpy_z,
    zo2_engine.py:183-204), so the weights each forward sees are the
    reference's W +- eps z bit for bit; only summation orders differ."""

    arith = "f64"

    def __init__(self, spec: ModelSpec, batch_size: int, device):
        self.spec, self.B = spec, int(batch_size)
        self.dev = torch.device(device)
        d, V = spec.dim, spec.vocab
        T = self.T = self.B * spec.seq_len

        def buf(n):
            return torch.empty(n, dtype=torch.float64, device=self.dev)
        self.h = [buf(T * d) for _ in range(2)]
        self.x, self.qkv, self.ctx, self.mid = buf(T * d), buf(T * 3 * d), buf(T * d), buf(T * 4 * d)
        self.logits, self.row = buf(T * V), buf(T)
        self.d_sums = torch.zeros(2, dtype=torch.float64, device=self.dev)
        # tied head: the embedding's perturbed tok_emb of each sign (model.py:367-369)
        self.stash = [buf(V * d) for _ in range(2)] if spec.tie_lm_head else None
        self.ids = torch.empty(T, dtype=torch.int64, device=self.dev)
        self.targets = torch.empty(T, dtype=torch.int64, device=self.dev)
        self.prof: list | None = None
        self._off = {sg.name: sg.offset for sg in segments(block_layout(spec))}

    @staticmethod
    def estimate_nbytes(spec: ModelSpec, batch_size: int) -> int:
        d, V, T = spec.dim, spec.vocab, int(batch_size) * spec.seq_len
        n = 2 * T * d + T * (d + 3 * d + d + 4 * d) + T * V + T
        n += 2 * V * d if spec.tie_lm_head else 0
        return 8 * n + 2 * T * 8

    def nbytes(self) -> dict[str, int]:
        act = sum(t.numel() * 8 for t in self.h + [self.x, self.qkv, self.ctx, self.mid,
                                                    self.logits, self.row])
        ops = sum(t.numel() * 8 for t in self.stash) if self.stash else 0
        return {"activations": act, "operands": ops, "io": 2 * self.T * 8}

    def forward(self, module: str, bucket: torch.Tensor, sign: int, stream) -> None:
        """Forward of `module` for one sign from its (perturbed) f64 bucket."""
        spec = self.spec
        d, V, T = spec.dim, spec.vocab, self.T
        if module == EMBED_ID:
            p = bucket.data_ptr()
            _lib.call("zo2_f64_embed", self.ids.data_ptr(), T, spec.seq_len, d, p,
                      p + V * d * 8, self.h[sign].data_ptr(), stream)
            if self.stash is not None:
                self.stash[sign].copy_(bucket[:V * d])
        elif module == HEAD_ID:
            w = self.stash[sign] if self.stash is not None else bucket
            _lib.call("zo2_f64_gemm", self.h[sign].data_ptr(), w.data_ptr(), 1, None,
                      self.logits.data_ptr(), T, V, d, _lib.F64_EPI_STORE, stream)
            _lib.call("zo2_f64_ce", self.logits.data_ptr(), self.targets.data_ptr(), T, V,
                      self.row.data_ptr(), self.d_sums[sign:].data_ptr(), stream)
        else:
            self._block(bucket.data_ptr(), sign, stream)

    def _block(self, base: int, sign: int, stream) -> None:
        spec = self.spec
        d, T, H = spec.dim, self.T, spec.n_heads
        o = {k: base + v * 8 for k, v in self._off.items()}
        h, x = self.h[sign].data_ptr(), self.x.data_ptr()
        qkv, ctx, mid = self.qkv.data_ptr(), self.ctx.data_ptr(), self.mid.data_ptr()
        gemm, E = _lib.call, _lib
        _lib.call("zo2_f64_layernorm", h, T, d, o["ln1_g"], o["ln1_b"], x, stream)
        gemm("zo2_f64_gemm", x, o["qkv_w"], 0, o["qkv_b"], qkv, T, 3 * d, d, E.F64_EPI_STORE,
             stream)
        _lib.call("zo2_f64_attention", qkv, self.B, spec.seq_len, H, spec.head_dim, ctx, stream)
        gemm("zo2_f64_gemm", ctx, o["attn_out_w"], 0, o["attn_out_b"], h, T, d, d,
             E.F64_EPI_RESIDUAL, stream)
        _lib.call("zo2_f64_layernorm", h, T, d, o["ln2_g"], o["ln2_b"], x, stream)
        gemm("zo2_f64_gemm", x, o["mlp_in_w"], 0, o["mlp_in_b"], mid, T, 4 * d, d,
             E.F64_EPI_GELU, stream)
        gemm("zo2_f64_gemm", mid, o["mlp_out_w"], 0, o["mlp_out_b"], h, T, d, 4 * d,
             E.F64_EPI_RESIDUAL, stream)
