"""Host-link rate with the GPU busy (tools only): full-duplex 1.2 GB pinned
copies (one stream per direction) alone, beside a loop of OPT-30B mlp_out
GEMMs, and beside a loop of K2c launches on an OPT-30B block.  One JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2503_12668_b200 import _lib  # noqa: E402
from paper_2503_12668_b200.model import DualForward, ModelSpec, module_size  # noqa: E402

dev = torch.device("cuda", 0)
N = 1233125376
h_up = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h_dn = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d_up = torch.empty(N, dtype=torch.uint8, device=dev)
d_dn = torch.empty(N, dtype=torch.uint8, device=dev)
su, sd, sk = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)

# GEMM load: mlp_out at cfg4 shapes, both signs
T, D = 8192, 7168
probs = (_lib.GemmProblem * 2)()
keep = []
for p in range(2):
    a = torch.randn(T, 4 * D, device=dev).to(torch.bfloat16)
    b = (torch.randn(D, 4 * D, device=dev) * 0.02).to(torch.bfloat16)
    bias = torch.zeros(D, device=dev)
    c = torch.zeros(T, D, device=dev)
    keep += [a, b, bias, c]
    probs[p].a_hi, probs[p].b_hi, probs[p].a_lo, probs[p].b_lo = a.data_ptr(), b.data_ptr(), None, None
    probs[p].bias, probs[p].c = bias.data_ptr(), c.data_ptr()

# K2c load: one OPT-30B block, bf16 arena
spec = ModelSpec(1, D, 56, 50272, 512)
fwd = DualForward(spec, 1, "bf16", "cuda", 1)
n = module_size(spec, "block.0")
arena = (torch.randn(n, device=dev) * 0.02).to(torch.bfloat16).view(torch.int16)
d_g = torch.tensor([1.5], dtype=torch.float64, device=dev)
counts = torch.zeros(2, dtype=torch.int64, device=dev)
descs = fwd.block_descs(0)


def load(kind, reps):
    s = sk.cuda_stream
    for _ in range(reps):
        if kind == "gemm":
            _lib.call("zo2_gemm", probs, 2, T, D, 4 * D, _lib.EPI_RESIDUAL, s)
        elif kind == "k2":
            _lib.call("zo2_update_perturb", arena.data_ptr(), _lib.BF16, n, 103_000_000, 1,
                      d_g.data_ptr(), 1e-7, 11, 1, 1e-3, 12, descs, len(descs), counts.data_ptr(), s)


def duplex(kind):
    best = (0.0, 0.0)
    for _ in range(3):
        torch.cuda.synchronize()
        load(kind, 40 if kind == "gemm" else (12 if kind == "k2" else 0))
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        with torch.cuda.stream(su):
            e[0].record(su)
            d_up.copy_(h_up, non_blocking=True)
            e[1].record(su)
        with torch.cuda.stream(sd):
            e[2].record(sd)
            h_dn.copy_(d_dn, non_blocking=True)
            e[3].record(sd)
        torch.cuda.synchronize()
        up = N / (e[0].elapsed_time(e[1]) * 1e-3) / 1e9
        dn = N / (e[2].elapsed_time(e[3]) * 1e-3) / 1e9
        best = max(best, (up, dn))
    return {"h2d_gbs": best[0], "d2h_gbs": best[1]}


print(json.dumps({"idle": duplex(None), "beside_gemm": duplex("gemm"), "beside_k2c": duplex("k2")}))
