"""A/B timing of K5 attention at the cfg2 (hd 64, split) and cfg3 (hd 128,
bf16) shapes (tools only; ZO2_LIB_PATH selects the library)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_12668_b200 import _lib  # noqa: E402

import os
_lib.call("zo2_set_attention_variant", int(os.environ.get("ZO2_ATTN_VARIANT", "0")))
SHAPES = ((16, 512, 32, 64, True), (16, 512, 32, 128, False))
if os.environ.get("ATTN_SHAPES"):  # e.g. "4,2048,32,64,1;16,512,32,64,1"
    SHAPES = tuple(tuple(int(x) for x in t.split(",")) for t in os.environ["ATTN_SHAPES"].split(";"))
for B, S, H, hd, split in SHAPES:
    split = bool(split)
    d = H * hd
    T = B * S
    qh = torch.randn(T, 3 * d, device="cuda").to(torch.bfloat16)
    ql = (torch.randn(T, 3 * d, device="cuda") * 1e-3).to(torch.bfloat16) if split else None
    oh = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    ol = torch.empty(T, d, device="cuda", dtype=torch.bfloat16) if split else None
    s = torch.cuda.current_stream().cuda_stream
    args = (qh.data_ptr(), ql.data_ptr() if split else None, B, S, H, hd, oh.data_ptr(),
            ol.data_ptr() if split else None, s)
    for _ in range(3):
        _lib.call("zo2_attention", *args)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        _lib.call("zo2_attention", *args)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    fl = 2 * 2 * B * H * S * S * hd / 2  # causal useful FLOPs (QK^T + PV)
    print(f"variant={os.environ.get('ZO2_ATTN_VARIANT', '0')} hd={hd} split={split}: {ms * 1e3:.1f} us  "
          f"{fl / ms / 1e9:.0f} TFLOP/s causal-useful")
