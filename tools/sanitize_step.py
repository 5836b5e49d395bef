"""compute-sanitizer target (tools only): two pipelined ZO2 steps of a
reduced-depth model at a production width, two operand sets, so K2 of block
i+1 co-runs with the tcgen05 GEMMs / attention of block i -- the configuration
in which smaller GEMM staging budgets once hung (zo2_gemm_sm100.cu).

  SAN_DIM (4096) SAN_BLOCKS (2) SAN_BATCH (2) SAN_ARITH (bf16) SAN_STEPS (2)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2503_12668_b200.data import gen_synthetic  # noqa: E402
from paper_2503_12668_b200.engine import TransformerWorkload, ZOConfig, Zo2Engine  # noqa: E402
from paper_2503_12668_b200.model import ModelSpec  # noqa: E402
from paper_2503_12668_b200.numerics import RngState  # noqa: E402
from paper_2503_12668_b200.runtime import OffloadRuntime, init_params  # noqa: E402

d = int(os.environ.get("SAN_DIM", "4096"))
nb = int(os.environ.get("SAN_BLOCKS", "2"))
B = int(os.environ.get("SAN_BATCH", "2"))
arith = os.environ.get("SAN_ARITH", "bf16")
steps = int(os.environ.get("SAN_STEPS", "2"))
V = int(os.environ.get("SAN_VOCAB", "50272"))
codec = "bf16" if arith == "bf16" else None
spec = ModelSpec(nb, d, d // 128 if d >= 4096 else d // 64, V, 512)
params = init_params(spec, RngState(5), codec=codec, device=torch.device("cuda", 0))
rt = OffloadRuntime(params, k_slots=3, codec=codec)
eng = Zo2Engine(TransformerWorkload(params, arith), ZOConfig(1e-3, 1e-5, steps, 5), rt,
                operand_sets=2)
ds = gen_synthetic(V, 512, 8, RngState(5), "affine", B)
for j in range(steps):
    eng.step_async(j, ds.batch(np.arange(B) + j))
gs = eng.drain()
eng.finalize()
torch.cuda.synchronize()
print("sanitize_step ok: operand_sets", eng.operand_sets, "g", gs)
