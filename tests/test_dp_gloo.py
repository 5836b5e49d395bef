"""Data-parallel host logic with a real 2-process torch.distributed group (gloo
on CPU): batch sharding + the loss-sum all-reduce reproduce the single-process
global-batch losses and g.  The per-rank forward here is the
CPU oracle (test infrastructure); on B200 the same helpers run with NCCL."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, store, out):
    # file rendezvous: no fixed TCP port that another job could hold
    dist.init_process_group("gloo", init_method=f"file://{store}", rank=rank, world_size=world)
    from oracle import zo2_oracle as O
    from paper_2503_12668_b200.parallel import (allreduce_loss_sums, projected_gradient,
                                                shard_indices)
    spec = O.Spec(2, 32, 4, 64, 16)
    seed, eps, B = 3, 1e-3, 2
    tok, tgt = O.gen_synthetic(spec.vocab, spec.seq_len, 32, seed)
    p = O.init_params(spec, seed)
    off = O.offsets(spec)
    s = O.derive_step_seed(seed, 0)
    idx = shard_indices(seed, 0, 32, B, rank, world)
    sums = []
    for coef in (eps, -2 * eps):
        for m, flat in p.items():
            O.axpy_z(flat, coef, s, off[m])
        h = O.fwd_embed(spec, p["embed"], tok[idx])
        for i in range(spec.n_blocks):
            h = O.fwd_block(spec, p[f"block.{i}"], h)
        logits = (h @ p["head"].reshape(spec.vocab, spec.dim).T).astype(np.float64)
        lse = logits.max(-1) + np.log(np.exp(logits - logits.max(-1, keepdims=True)).sum(-1))
        picked = np.take_along_axis(logits, tgt[idx][..., None], -1)[..., 0]
        sums.append(float((lse - picked).sum()))
    t = torch.tensor(sums, dtype=torch.float64)
    allreduce_loss_sums(t)
    out[rank] = projected_gradient(t.tolist(), B * spec.seq_len * world, eps)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_matches_global_batch():
    from oracle import zo2_oracle as O
    world = 2
    fd, store = tempfile.mkstemp(prefix="zo2_gloo_store_")
    os.close(fd)
    os.unlink(store)
    mgr = mp.Manager()
    out = mgr.dict()
    try:
        mp.spawn(_worker, args=(world, store, out), nprocs=world, join=True)
    finally:
        if os.path.exists(store):
            os.unlink(store)
    assert out[0] == out[1]                      # every rank forms the same g
    spec = O.Spec(2, 32, 4, 64, 16)
    tok, tgt = O.gen_synthetic(spec.vocab, spec.seq_len, 32, 3)
    idx = O.batch_for_step(3, 0, 32, 2 * world)
    eng = O.MeZO(spec, O.init_params(spec, 3), 1e-3, 1e-3, 3)
    g = eng.step(tok[idx], tgt[idx], 0)
    lp, lm, g_dp = out[0]
    assert abs(lp - eng.losses[0]) < 1e-12 * abs(lp)
    assert abs(lm - eng.losses_minus[0]) < 1e-12 * abs(lm)
    assert abs(g_dp - g) <= 1e-12 / (2e-3) * 10
