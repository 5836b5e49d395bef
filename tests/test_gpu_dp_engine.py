"""Data parallel through the real engine.

* NCCL at world size 1: the only multi-GPU code paths this box can execute on
  its single GPU -- the loss-sum all-reduce on the compute stream and the
  in-place `all_gather_into_tensor` of sharded arena transfers -- run through
  NCCL and must leave the step bit-identical to the engine without data
  parallel.
* Two ranks (gloo, sharing one GPU) each running the real engine on half the
  global batch must reproduce the one-rank engine on the whole global batch:
  per-token losses are row-independent, so only the order of the f64 loss-sum
  reduction differs (losses within 1e-12 relative, g within the propagated
  bound), and the final parameters agree to the last few ulps.
"""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SPEC = (3, 64, 4, 128, 32)
SEED, STEPS, EPS, LR = 11, 3, 1e-3, 1e-3


def _engine(codec=None, batch=2):
    from paper_2503_12668_b200.engine import TransformerWorkload, ZOConfig, Zo2Engine
    from paper_2503_12668_b200.model import ModelSpec
    from paper_2503_12668_b200.numerics import RngState
    from paper_2503_12668_b200.runtime import OffloadRuntime, init_params
    spec = ModelSpec(*SPEC)
    params = init_params(spec, RngState(SEED), codec=codec)
    rt = OffloadRuntime(params, k_slots=3, codec=codec)
    eng = Zo2Engine(TransformerWorkload(params, "f32"), ZOConfig(EPS, LR, STEPS, SEED), rt)
    return spec, rt, eng


def _dataset(spec, batch):
    from paper_2503_12668_b200.data import gen_synthetic
    from paper_2503_12668_b200.numerics import RngState
    return gen_synthetic(spec.vocab, spec.seq_len, 16, RngState(SEED), "affine", batch)


def _run_steps(eng, ds, batch, rank, world):
    from paper_2503_12668_b200.parallel import shard_indices
    from paper_2503_12668_b200.runtime import params_digest
    for j in range(STEPS):
        eng.step(ds.batch(shard_indices(SEED, j, ds.n_samples, batch, rank, world)), j)
    final = eng.finalize()
    torch.cuda.synchronize()
    return {"losses": list(eng.losses), "losses_minus": list(eng.losses_minus),
            "gs": list(eng.gs), "digest": params_digest(final), "params": final.to_numpy()}


def _worker(rank, world, store, backend, codec, q):
    try:
        import torch.distributed as dist
        torch.cuda.set_device(0)
        kw = {"device_id": torch.device("cuda", 0)} if backend == "nccl" else {}
        dist.init_process_group(backend, init_method=f"file://{store}", rank=rank,
                                world_size=world, **kw)
        spec, rt, eng = _engine(codec)
        sharded = eng.enable_data_parallel(shard_transfers=(backend == "nccl"))
        out = _run_steps(eng, _dataset(spec, 2), 2, rank, world)
        out.update(sharded=sharded, backend=dist.get_backend(),
                   up_bytes=rt.log.wire_bytes("upload"))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as e:  # surface the failure instead of a queue timeout
        import traceback
        q.put((rank, {"error": f"{e!r}\n{traceback.format_exc()}"}))


def _spawn(world, backend, codec=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    fd, store = tempfile.mkstemp(prefix="zo2_dp_engine_")
    os.close(fd)
    os.unlink(store)
    ps = [ctx.Process(target=_worker, args=(r, world, store, backend, codec, q))
          for r in range(world)]
    for p in ps:
        p.start()
    try:
        res = dict(q.get(timeout=300) for _ in ps)
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
        if os.path.exists(store):
            os.unlink(store)
    for r, out in res.items():
        assert "error" not in out, f"rank {r}: {out['error']}"
    return res


def _single(codec=None, batch=2):
    spec, rt, eng = _engine(codec)
    out = _run_steps(eng, _dataset(spec, batch), batch, 0, 1)
    out["up_bytes"] = rt.log.wire_bytes("upload")
    return out


@pytest.mark.parametrize("codec", [None, "bf16"])
def test_nccl_world1_bit_identical(cuda, codec):
    """The NCCL branches (loss all-reduce on the compute stream, in-place arena
    all-gather) execute and change nothing."""
    dp = _spawn(1, "nccl", codec)[0]
    ref = _single(codec)
    assert dp["backend"] == "nccl" and dp["sharded"]
    assert dp["losses"] == ref["losses"] and dp["gs"] == ref["gs"]
    assert dp["digest"] == ref["digest"]
    assert dp["up_bytes"] == ref["up_bytes"]


def test_two_rank_engine_matches_global_batch(cuda):
    """2 ranks x batch 2 (real engine, gloo all-reduce) == 1 rank x batch 4."""
    two = _spawn(2, "gloo")
    one = _single(batch=4)
    assert two[0]["gs"] == two[1]["gs"] and two[0]["digest"] == two[1]["digest"]
    for key in ("losses", "losses_minus"):
        np.testing.assert_allclose(two[0][key], one[key], rtol=1e-12, atol=0)
    for j in range(STEPS):
        dl = (abs(two[0]["losses"][j] - one["losses"][j])
              + abs(two[0]["losses_minus"][j] - one["losses_minus"][j]))
        assert abs(two[0]["gs"][j] - one["gs"][j]) <= dl / (2 * EPS) + 1e-12 * abs(one["gs"][j])
    # the same z and (up to the reduction order of g) the same updates
    for m, ref in one["params"].items():
        got = two[0]["params"][m]
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-6 * max(1.0, float(np.abs(ref).max())),
                                   err_msg=m)
