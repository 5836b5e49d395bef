"""Data parallelism for the ZO2 step.

The path shards over the batch: every rank draws z from the same (seed, step,
offset) stream and applies the same g, so weights stay bit-identical without
any parameter traffic; the only exchange is the two f64 cross-entropy sums
(sum over tokens of l+ and l-), all-reduced before g is formed.  Summing
numerators (not averaging per-rank means) keeps the single-process mean
semantics of model.py:313 up to reduction order.

These helpers are what the engine and bench.py call; they work with any
torch.distributed backend (NCCL on B200 -- the all-reduce is enqueued on the
compute stream -- and gloo on CPU for the multi-process tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .engine import batch_for_step


def shard_indices(seed: int, step_index: int, n_samples: int, per_rank_batch: int,
                  rank: int, world: int) -> np.ndarray:
    """Rank `rank`'s contiguous slice of the global batch batch_for_step(seed, j,
    n, per_rank_batch * world) (zo_ref.py:49-56)."""
    idx = batch_for_step(seed, step_index, n_samples, per_rank_batch * world)
    return idx[rank * per_rank_batch:(rank + 1) * per_rank_batch]


def allreduce_loss_sums(sums: torch.Tensor, group=None) -> torch.Tensor:
    """In-place SUM all-reduce of the [l+ sum, l- sum] f64 pair.  It runs at
    every world size once data parallel is enabled (at world 1 it is the
    identity, but the collective -- NCCL on the compute stream -- still
    executes, so a single-GPU box exercises the multi-rank code path)."""
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    return sums


def projected_gradient(sums, tokens_total: int, eps: float) -> tuple[float, float, float]:
    """Host statement of K10 (zo2_form_g): l+- = sums / count, g = (l+ - l-) / 2eps."""
    lp = float(sums[0]) / tokens_total
    lm = float(sums[1]) / tokens_total
    return lp, lm, (lp - lm) / (2.0 * eps)
