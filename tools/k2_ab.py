"""A/B timing of K2 (tools only): ZO2_LIB_PATH selects the library, ZO2_RNG
the z generator; K2_ARENA=f32|bf16 and K2_DIM set the arena format (bf16 =
codec arena with bf16 operands, the AMP configurations) and the width."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_12668_b200 import _lib  # noqa: E402
from paper_2503_12668_b200.model import DualForward, ModelSpec, module_size  # noqa: E402

_lib.call("zo2_set_rng_mode", 1 if os.environ.get("ZO2_RNG") == "fast" else 0)
_lib.call("zo2_set_k2_variant", int(os.environ.get("K2_VARIANT", "0")))
arena_fmt = os.environ.get("K2_ARENA", "f32")
dim = int(os.environ.get("K2_DIM", "2048"))
spec = ModelSpec(1, dim, dim // 128 if dim >= 4096 else dim // 64, 50272, 512)
fwd = DualForward(spec, 1, "f32" if arena_fmt == "f32" else "bf16", "cuda", 1)
n = module_size(spec, "block.0")
w = torch.randn(n, device="cuda") * 0.02
if arena_fmt == "f32":
    arena, code = w, _lib.F32
else:
    tdt = torch.float16 if arena_fmt == "f16" else torch.bfloat16
    arena, code = w.to(tdt).view(torch.int16), (_lib.F16 if arena_fmt == "f16" else _lib.BF16)
d_g = torch.tensor([1.5], dtype=torch.float64, device="cuda")
counts = torch.zeros(2, dtype=torch.int64, device="cuda")
descs = fwd.block_descs(0)
s = torch.cuda.current_stream().cuda_stream


def run():
    _lib.call("zo2_update_perturb", arena.data_ptr(), code, n, 103_000_000, 1,
              d_g.data_ptr(), 1e-7, 11, 1, 1e-3, 12, descs, len(descs), counts.data_ptr(), s)


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
R = 10
for _ in range(R):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
fb = ctypes.c_uint64(0)
_lib.call("zo2_k2c_fallbacks", ctypes.byref(fb), 1)
print(f"fallbacks per run {fb.value / (R + 3):.0f} of {n} ({fb.value / (R + 3) / n:.2e}) ", end="")
print(f"variant={os.environ.get('K2_VARIANT', '0')} rng={os.environ.get('ZO2_RNG', 'exact')} arena={arena_fmt} "
      f"d={dim} K2 block ms {ms:.3f}  Gz/s {2 * n / ms / 1e6:.1f}")
