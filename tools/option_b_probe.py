"""North-star option (b) -- regenerate z inside the GEMM prologue instead of
materialising W+-eps z once per block (K2) -- priced with MEASURED generator
rates (tools only).

In a weight-stationary-free GEMM (C = A W^T, A = [T, K] activations, W =
[N, K]) every W tile is consumed once per M tile, so regenerating z in the
prologue costs ceil(T / BM) draws per weight per step (both signs share one
z), against 1 draw (+1 for the deferred update) when K2 materialises the
operands.  This script times the standalone generators (the fast Philox4x32
+ erfinv z, and the exact reference z) on 2^30 draws and prints, per OPT
geometry, the prologue draw count per block, its time at the measured rate
(a LOWER bound: the real prologue also forms W+-eps z, converts to bf16 and
stores to shared memory), and the block's GEMM time at the sustained bf16
peak.  Output: one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2503_12668_b200 import _lib  # noqa: E402

N = 1 << 30
out = torch.empty(N, dtype=torch.float32, device="cuda")
out64 = torch.empty(N // 8, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def rate(fn, n):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return n * reps / (e0.elapsed_time(e1) / 1e3)


fast = rate(lambda: _lib.call("zo2_z_fill_fast", out.data_ptr(), N, 7, 1, 0, s), N)
exact = rate(lambda: _lib.call("zo2_z_fill", out64.data_ptr(), N // 8, 7, 1, 0, s), N // 8)
peak = 1392.6e12
try:
    peak = json.load(open("MEASURED_PEAKS.json")).get("bf16_tflops_sustained", 1392.6) * 1e12
except Exception:  # noqa: BLE001
    pass
rows = []
for name, d, T in (("cfg2 OPT-1.3B", 2048, 8192), ("cfg3 OPT-6.7B", 4096, 8192),
                   ("cfg4 OPT-30B", 7168, 8192), ("cfg5 OPT-175B", 12288, 8192)):
    w = 12 * d * d                       # block matrices (qkv 3d^2, out d^2, mlp 8d^2)
    regen = -(-T // 256)                 # CTA-pair M tile of 256 rows
    gemm_s = 2 * 2 * T * w / peak        # both signs
    rows.append({"config": name, "weights": w, "regen_per_weight": regen,
                 "prologue_draws": w * regen,
                 "prologue_ms_fast_lower_bound": 1e3 * w * regen / fast,
                 "prologue_ms_exact_lower_bound": 1e3 * w * regen / exact,
                 "k2_draws": 2 * w, "k2_ms_at_fast_rate": 1e3 * 2 * w / fast,
                 "gemm_ms_at_peak": 1e3 * gemm_s})
print(json.dumps({"probe": "option_b", "fast_gdraws_per_s": fast / 1e9,
                  "exact_gdraws_per_s": exact / 1e9, "rows": rows}))
