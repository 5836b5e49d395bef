"""Data parallel with node-wide shared host masters and sharded transfers
(runtime.SharedHostMasters / OffloadRuntime.enable_sharding):
two ranks (gloo, sharing one GPU) must produce exactly what two ranks with
private masters and full-block transfers produce -- same losses, same g,
bit-identical final parameters -- while each moves half the PCIe bytes."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, store, sharded, codec, q):
    try:
        q.put((rank, _body(rank, world, store, sharded, codec)))
    except Exception as e:  # surface the failure instead of a queue timeout
        import traceback
        q.put((rank, {"error": f"{e!r}\n{traceback.format_exc()}"}))


def _body(rank, world, store, sharded, codec):
    import torch.distributed as dist
    from paper_2503_12668_b200.data import gen_synthetic
    from paper_2503_12668_b200.engine import TransformerWorkload, ZOConfig, Zo2Engine
    from paper_2503_12668_b200.model import ModelSpec, block_id, module_size
    from paper_2503_12668_b200.numerics import CODEC_FORMATS, ElemFormat, RngState
    from paper_2503_12668_b200.parallel import shard_indices
    from paper_2503_12668_b200.runtime import (_TORCH_STORAGE, OffloadRuntime,
                                               SharedHostMasters, init_params, params_digest)
    torch.cuda.set_device(0)
    # file rendezvous: no TCP port to race for between the probe and the bind
    dist.init_process_group("gloo", init_method=f"file://{store}", rank=rank,
                            world_size=world)
    spec = ModelSpec(3, 64, 4, 128, 32)
    seed, steps, B = 11, 3, 2
    shm = None
    if sharded:
        name = [f"zo2_test_{os.path.basename(store)}" if rank == 0 else None]
        dist.broadcast_object_list(name, src=0)
        sdt = _TORCH_STORAGE[CODEC_FORMATS[codec] if codec else ElemFormat.F32]
        n = module_size(spec, block_id(0))
        if rank == 0:
            shm = SharedHostMasters(name[0], spec.n_blocks, n, sdt, owner=True)
            params = init_params(spec, RngState(seed), codec=codec, host_masters=shm)
            dist.barrier()
        else:
            dist.barrier()
            shm = SharedHostMasters(name[0], spec.n_blocks, n, sdt, owner=False)
            params = init_params(spec, RngState(seed), codec=codec, host_masters=shm)
    else:
        params = init_params(spec, RngState(seed), codec=codec)
    rt = OffloadRuntime(params, k_slots=3, codec=codec)
    eng = Zo2Engine(TransformerWorkload(params, "f32"), ZOConfig(1e-3, 1e-3, steps, seed), rt)
    got_sharded = eng.enable_data_parallel(shard_transfers=sharded)
    ds = gen_synthetic(spec.vocab, spec.seq_len, 16, RngState(seed), "affine", B)
    for j in range(steps):
        eng.step(ds.batch(shard_indices(seed, j, ds.n_samples, B, rank, world)), j)
    final = eng.finalize()
    torch.cuda.synchronize()
    out = {"losses": eng.losses, "gs": eng.gs, "digest": params_digest(final),
           "sharded": got_sharded, "up_bytes": rt.log.wire_bytes("upload")}
    dist.barrier()
    if shm is not None:
        shm.close()
    dist.destroy_process_group()
    return out


def _run(sharded, codec=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    fd, store = tempfile.mkstemp(prefix="zo2_dp_store_")
    os.close(fd)
    os.unlink(store)  # the FileStore creates it
    ps = [ctx.Process(target=_worker, args=(r, 2, store, sharded, codec, q)) for r in range(2)]
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


@pytest.mark.parametrize("codec", [None, "bf16"])
def test_sharded_transfers_match_replicated(cuda, codec):
    rep = _run(False, codec)
    sh = _run(True, codec)
    for r in (0, 1):
        assert sh[r]["sharded"] and not rep[r]["sharded"]
        assert sh[r]["losses"] == rep[r]["losses"] and sh[r]["gs"] == rep[r]["gs"]
        assert sh[r]["digest"] == rep[r]["digest"]
        assert sh[r]["up_bytes"] * 2 == rep[r]["up_bytes"]
    # both ranks hold the same model
    assert sh[0]["digest"] == sh[1]["digest"] and np.isfinite(sh[0]["gs"]).all()
