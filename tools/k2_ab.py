"""A/B timing of K2 variants (tools only): ZO2_LIB_PATH selects the library."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2503_12668_b200 import _lib  # noqa: E402
from paper_2503_12668_b200.model import DualForward, ModelSpec, module_size  # noqa: E402

import os
_lib.call("zo2_set_rng_mode", 1 if os.environ.get("ZO2_RNG") == "fast" else 0)
spec = ModelSpec(1, 2048, 32, 50272, 512)
fwd = DualForward(spec, 1, "f32", "cuda", 1)
n = module_size(spec, "block.0")
arena = torch.randn(n, device="cuda") * 0.02
d_g = torch.tensor([1.5], dtype=torch.float64, device="cuda")
descs = fwd.block_descs(0)
s = torch.cuda.current_stream().cuda_stream
for j in range(3):
    _lib.call("zo2_update_perturb", arena.data_ptr(), _lib.F32, n, 103_000_000, 1,
              d_g.data_ptr(), 1e-7, 11, 1, 1e-3, 12, descs, len(descs), None, s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
R = 10
for j in range(R):
    _lib.call("zo2_update_perturb", arena.data_ptr(), _lib.F32, n, 103_000_000, 1,
              d_g.data_ptr(), 1e-7, 11, 1, 1e-3, 12, descs, len(descs), None, s)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
print(f"{_lib.LIB_PATH.split('/')[-1]} rng={os.environ.get('ZO2_RNG', 'exact')} K2 block ms {ms:.3f}  Gz/s {2 * n / ms / 1e6:.1f}")
