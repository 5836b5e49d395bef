"""Device side of rng = "fast" (csrc/zo2_rng_fast.h): z probe, the fused
update/perturb kernel and a teacher-forced toy run against the oracle's
numpy restatement -- bit-exact, the same checks as the exact mode."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def L():
    from paper_2503_12668_b200 import _lib
    return _lib


def stream():
    return torch.cuda.current_stream().cuda_stream


@pytest.fixture
def fast_mode():
    L().call("zo2_set_rng_mode", 1)
    yield
    L().call("zo2_set_rng_mode", 0)


def test_z_fill_fast_matches_oracle(cuda, oracle):
    for seed, st, ctr, n in ((7, 0, 0, 3_000_001), (2**63 + 5, 0, 2**40 + 3, 10_007)):
        out = torch.empty(n, dtype=torch.float32, device=cuda)
        L().call("zo2_z_fill_fast", out.data_ptr(), n, seed, st, ctr, stream())
        ref = oracle.fast_gauss(seed, st, ctr, n)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("layout", ["linear", "transposed"])
def test_update_perturb_fast_bit_exact(cuda, oracle, fast_mode, layout):
    _l = L()
    rows, cols, base, lrs, rs, eps, lr, g = 72, 200, 4096, 11, 22, 1e-3, 1e-3, -1.25
    n = rows * cols
    w = (np.random.default_rng(2).standard_normal(n) * 0.05).astype(np.float32)
    dev = torch.from_numpy(w.copy()).to(cuda)
    d_g = torch.tensor([g], dtype=torch.float64, device=cuda)
    segs = (_l.SegmentDesc * 1)()
    s = segs[0]
    s.offset, s.rows, s.cols = 0, rows, cols
    if layout == "transposed":
        ph, mh, pl, ml = (torch.empty(n, dtype=torch.bfloat16, device=cuda) for _ in range(4))
        s.out_kind = _l.OUT_SPLIT_T
        s.out_plus, s.out_minus, s.out_plus_lo, s.out_minus_lo = (
            ph.data_ptr(), mh.data_ptr(), pl.data_ptr(), ml.data_ptr())
    else:
        plus, minus = (torch.empty(n, dtype=torch.float32, device=cuda) for _ in range(2))
        s.out_kind = _l.OUT_F32
        s.out_plus, s.out_minus = plus.data_ptr(), minus.data_ptr()
    _l.call("zo2_update_perturb", dev.data_ptr(), _l.F32, n, base, 1, d_g.data_ptr(), lr, lrs, 1,
            eps, rs, segs, 1, None, stream())
    ref = w.copy()
    oracle.axpy_z_fast(ref, -(lr * g), lrs, base)
    oracle.axpy_z_fast(ref, eps, rs, base)
    wp = ref.copy()
    oracle.axpy_z_fast(ref, -2.0 * eps, rs, base)
    wm = ref.copy()
    oracle.axpy_z_fast(ref, eps, rs, base)
    assert np.array_equal(dev.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    if layout == "linear":
        assert np.array_equal(plus.cpu().numpy(), wp) and np.array_equal(minus.cpu().numpy(), wm)
    else:
        refT = torch.from_numpy(wp.reshape(rows, cols).T.copy()).to(torch.bfloat16)
        assert torch.equal(ph.cpu().view(-1), refT.view(-1))


def test_toy_teacher_forced_fast_rng(cuda, golden, oracle):
    """The toy of test_gpu_engine.py with rng = "fast": the B200 deferred ZO2
    engine against the oracle's MeZO driven by the same fast direction."""
    from paper_2503_12668_b200.data import gen_synthetic
    from paper_2503_12668_b200.engine import (TransformerWorkload, ZOConfig, Zo2Engine,
                                              batch_for_step)
    from paper_2503_12668_b200.model import ModelSpec
    from paper_2503_12668_b200.numerics import RngState
    from paper_2503_12668_b200.runtime import OffloadRuntime, init_params
    G = golden("toy.json")
    spec = ModelSpec(*G["spec"])
    steps = 4
    params = init_params(spec, RngState(G["seed"]))
    eng = Zo2Engine(TransformerWorkload(params, "f32"), ZOConfig(G["eps"], G["lr"], steps, G["seed"]),
                    OffloadRuntime(params, k_slots=3), rng="fast")
    ospec = oracle.Spec(*G["spec"])
    ref = oracle.MeZO(ospec, oracle.init_params(ospec, G["seed"]), G["eps"], G["lr"], G["seed"],
                      rng="fast")
    ds = gen_synthetic(spec.vocab, spec.seq_len, G["n_samples"], RngState(G["seed"]), "affine",
                       G["batch_size"])
    for j in range(steps):
        tok, tgt = ds.batch(batch_for_step(G["seed"], j, ds.n_samples, ds.batch_size))
        g_ref = ref.step(tok, tgt, j)
        eng.step((tok, tgt), j)
        assert abs(eng.losses[-1] - ref.losses[-1]) <= 1e-5 * abs(ref.losses[-1])
        eng.force_pending(g_ref)
    final = eng.finalize().to_numpy()
    for m, flat in ref.p.items():
        assert np.array_equal(final[m].view(np.uint32), flat.view(np.uint32)), m
    # and the fast direction really differs from the reference's
    assert eng.losses[0] != G["runs"]["f32"]["l_plus"][0]
