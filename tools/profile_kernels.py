"""Launch each hot kernel once at the cfg2 (OPT-1.3B, 16x512) shapes, for
`ncu --set full` captures (tools only; not part of the product path).
PK_DIM selects another width (heads = dim/128 from 4096 up, as OPT)."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_12668_b200.model import DualForward, ModelSpec  # noqa: E402

_D = int(os.environ.get("PK_DIM", "2048"))
if os.environ.get("PK_RASTER"):  # "cta,pair" group heights (zo2_set_gemm_raster)
    from paper_2503_12668_b200 import _lib as _L
    _L.call("zo2_set_gemm_raster", *(int(x) for x in os.environ["PK_RASTER"].split(",")))
_SPEC = (1, _D, _D // 128 if _D >= 4096 else _D // 64, 50272, 512)


def main(arith="f32"):
    spec = ModelSpec(*_SPEC)
    fwd = DualForward(spec, 16, arith, "cuda", 1)
    for t in fwd.h:
        t.normal_()
    vec, mat = fwd.sets[0]
    for pair in list(vec.values()):
        for t in pair:
            t.normal_()
    for pair in mat.values():
        for o in pair:
            o.hi.normal_()
            if o.lo is not None:
                o.lo.normal_(0, 1e-3)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        fwd.block_forward(s, 0)
    torch.cuda.synchronize()




def k2(arith="f32"):
    """One K2 (update + perturb, transposed operands) over a cfg2 block."""
    from paper_2503_12668_b200 import _lib
    from paper_2503_12668_b200.model import module_size
    _lib.call("zo2_set_rng_mode", 1 if os.environ.get("ZO2_RNG") == "fast" else 0)
    spec = ModelSpec(*_SPEC)
    fwd = DualForward(spec, 16, arith, "cuda", 1)
    n = module_size(spec, "block.0")
    arena = torch.randn(n, device="cuda") * 0.02
    d_g = torch.tensor([1.5], dtype=torch.float64, device="cuda")
    descs = fwd.block_descs(0)
    s = torch.cuda.current_stream().cuda_stream
    for j in range(2):
        _lib.call("zo2_update_perturb", arena.data_ptr(), _lib.F32, n, 103_000_000, 1,
                  d_g.data_ptr(), 1e-7, 11 + j, 1, 1e-3, 12 + j, descs, len(descs), None, s)
    torch.cuda.synchronize()


def head(arith="f32"):
    """Head GEMM with the fused cross-entropy epilogue (K7) + CE reduce."""
    spec = ModelSpec(*_SPEC)
    fwd = DualForward(spec, 16, arith, "cuda", 1)
    for t in fwd.h:
        t.normal_()
    for o in fwd.head_op:
        o.hi.normal_(0, 0.02)
        if o.lo is not None:
            o.lo.normal_(0, 1e-5)
    fwd.targets.random_(0, spec.vocab)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        fwd.head_forward(s)
    torch.cuda.synchronize()


def embed(arith="f32"):
    """Embedding gather with the on-the-fly update + perturbation (K8)."""
    spec = ModelSpec(*_SPEC)
    fwd = DualForward(spec, 16, arith, "cuda", 1)
    table = torch.randn((spec.vocab + spec.seq_len) * spec.dim, device="cuda") * 0.02
    fwd.ids.random_(0, spec.vocab)
    d_g = torch.tensor([1.5], dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for j in range(2):
        fwd.embed_forward(table, 0, True, d_g, 1e-7, 11 + j, 1e-3, 12 + j, spec.seq_len, s)
    torch.cuda.synchronize()


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "fwd"
    arith = sys.argv[2] if len(sys.argv) > 2 else "f32"
    {"k2": k2, "head": head, "embed": embed}.get(what, main)(arith)
