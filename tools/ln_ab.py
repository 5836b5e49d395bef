"""LayerNorm timing at cfg2/cfg3 shapes (tools only): achieved HBM GB/s."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_12668_b200 import _lib  # noqa: E402

for T, d, split in ((8192, 2048, True), (8192, 4096, False), (8192, 7168, False)):
    x = torch.randn(T, d, device="cuda")
    g, b = torch.randn(d, device="cuda"), torch.randn(d, device="cuda")
    hi = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    lo = torch.empty_like(hi) if split else None
    s = torch.cuda.current_stream().cuda_stream
    args = (x.data_ptr(), T, d, g.data_ptr(), b.data_ptr(), hi.data_ptr(),
            lo.data_ptr() if split else None, s)
    for _ in range(3):
        _lib.call("zo2_layernorm", *args)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        _lib.call("zo2_layernorm", *args)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    nbytes = T * d * 4 + T * d * 2 * (2 if split else 1)
    print(f"LN T={T} d={d} split={split}: {ms * 1e3:.1f} us  {nbytes / ms / 1e6:.0f} GB/s")
