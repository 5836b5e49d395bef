"""GEMM tile-raster sweep at the OPT-30B (cfg4) block shapes, T = 16 x 512
(tools only).  For each raster group height it launches the four block
GEMMs (both signs, bf16) and prints the CUDA-event time per launch.  Run it
under `ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct
--clock-control none` for the DRAM bytes of each launch (launch order:
gm-major, shapes in SHAPES order, REPS launches each)."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2503_12668_b200 import _lib  # noqa: E402

D = int(os.environ.get("RS_DIM", "7168"))
T = int(os.environ.get("RS_T", "8192"))
GMS = [int(x) for x in os.environ.get("RS_GMS", "1,2,4,8,16,32").split(",")]
REPS = int(os.environ.get("RS_REPS", "3"))
SHAPES = {"qkv": (3 * D, D, _lib.EPI_STORE), "out": (D, D, _lib.EPI_RESIDUAL),
          "mlp_in": (4 * D, D, _lib.EPI_GELU), "mlp_out": (D, 4 * D, _lib.EPI_RESIDUAL)}
only = os.environ.get("RS_SHAPES")
if only:
    SHAPES = {k: v for k, v in SHAPES.items() if k in only.split(",")}
s = torch.cuda.current_stream().cuda_stream
dev = torch.device("cuda", 0)


def problem(N, K, epi):
    probs = (_lib.GemmProblem * 2)()
    keep = []
    for p in range(2):
        a = torch.randn(T, K, device=dev).to(torch.bfloat16)
        b = (torch.randn(N, K, device=dev) * 0.02).to(torch.bfloat16)
        bias = torch.zeros(N, device=dev)
        keep += [a, b, bias]
        pr = probs[p]
        pr.a_hi, pr.b_hi, pr.a_lo, pr.b_lo = a.data_ptr(), b.data_ptr(), None, None
        pr.bias = bias.data_ptr()
        if epi == _lib.EPI_GELU:
            c = torch.empty(T, N, dtype=torch.bfloat16, device=dev)
            pr.c, pr.c_lo = c.data_ptr(), None
        else:
            c = torch.zeros(T, N, device=dev)
            pr.c = c.data_ptr()
        keep.append(c)
    return probs, keep


probs = {k: problem(*v) for k, v in SHAPES.items()}
for gm in GMS:
    _lib.call("zo2_set_gemm_raster", 12, gm)
    line = [f"gm={gm:3d}"]
    for k, (N, K, epi) in SHAPES.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        _lib.call("zo2_gemm", probs[k][0], 2, T, N, K, epi, s)
        e0.record()
        for _ in range(REPS - 1):
            _lib.call("zo2_gemm", probs[k][0], 2, T, N, K, epi, s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / max(1, REPS - 1)
        tf = 2 * 2 * T * N * K / (ms / 1e3) / 1e12
        line.append(f"{k} {ms:.3f} ms {tf:.0f} TF/s")
    print("  ".join(line), flush=True)
_lib.call("zo2_set_gemm_raster", 0, 0)
