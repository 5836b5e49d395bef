"""Reference parity for the AMP configurations 3-5 at full width.

Known answers: tests/golden/amp.json, written by tests/golden/make_amp_golden.py
from the REFERENCE itself (zo2lab's Zo2Engine over its OffloadRuntime with the
wire codec; harness/config.py:112-113 pins f32 arithmetic under a codec and
runtime.py:145-199 encodes the host master).  Full OPT width, reduced depth
(BASELINE.md §3): cfg3 = 2 blocks at d 4096 / 32 heads with the bf16 wire,
cfg4 = 1 block at d 7168 / 56 heads (bf16 wire), cfg5 = 1 block at
d 12288 / 96 heads (f16 wire); V 50272, S 512, batch 2, two steps + finalize.

  * arith=f32 (the reference's AMP arithmetic): l+/l- within 1e-5 relative,
    g inside the propagated bound, and -- with the reference's g loaded
    (teacher forcing) -- every module's final bytes SHA-256-identical to the
    reference's, the same wire bytes and the same conversion counters.
  * arith=bf16 (the bench's compute): l+/l- within the north star's 1e-2
    relative, g inside the propagated bound, teacher-forced final parameters
    still identical (the update path is arithmetic-independent).
"""
import hashlib

import pytest
import torch

pytestmark = pytest.mark.gpu

TAGS = ["cfg3_2blk", "cfg4_1blk", "cfg5_1blk"]
RTOL = {"f32": 1e-5, "bf16": 1e-2}


def _run(golden, tag, arith):
    from paper_2503_12668_b200.data import gen_synthetic
    from paper_2503_12668_b200.engine import (TransformerWorkload, ZOConfig, Zo2Engine,
                                              batch_for_step)
    from paper_2503_12668_b200.model import ModelSpec
    from paper_2503_12668_b200.numerics import RngState
    from paper_2503_12668_b200.runtime import OffloadRuntime, init_params, params_digest
    K = golden("amp.json")[tag]
    spec = ModelSpec(*K["spec"])
    params = init_params(spec, RngState(K["seed"]), codec=K["codec"])
    rt = OffloadRuntime(params, k_slots=K["k_slots"], codec=K["codec"])
    eng = Zo2Engine(TransformerWorkload(params, arith),
                    ZOConfig(K["eps"], K["lr"], K["steps"], K["seed"]), rt,
                    overlap=K["overlap"])
    ds = gen_synthetic(spec.vocab, spec.seq_len, K["n_samples"], RngState(K["seed"]), "affine",
                       K["batch_size"])
    rtol = RTOL[arith]
    for j in range(K["steps"]):
        idx = batch_for_step(K["seed"], j, ds.n_samples, ds.batch_size)
        assert idx.tolist() == K["batches"][j]
        g = eng.step(ds.batch(idx), j)
        lp, lm = eng.losses[-1], eng.losses_minus[-1]
        dlp, dlm = abs(lp - K["l_plus"][j]), abs(lm - K["l_minus"][j])
        assert dlp <= rtol * abs(K["l_plus"][j]), (tag, arith, j, lp, K["l_plus"][j])
        assert dlm <= rtol * abs(K["l_minus"][j]), (tag, arith, j, lm, K["l_minus"][j])
        assert abs(g - K["g"][j]) <= (dlp + dlm) / (2 * K["eps"]) + 1e-12, (g, K["g"][j])
        eng.force_pending(K["g"][j])
    final = eng.finalize()
    flats = final.to_numpy()
    bad = [m for m, h in K["module_digests"].items()
           if hashlib.sha256(flats[m].tobytes()).hexdigest() != h]
    assert bad == [], f"{tag}/{arith}: modules differ from the reference: {bad}"
    assert params_digest(final) == K["digest"]
    assert rt.log.wire_bytes("upload") == K["wire_up"]
    assert [rt.conversion.nan_count, rt.conversion.saturated_count] == K["conversion"]
    del eng, rt, params, final, flats
    torch.cuda.empty_cache()


@pytest.mark.parametrize("tag", TAGS)
def test_amp_f32_arith_reference_kat(cuda, golden, tag):
    _run(golden, tag, "f32")


@pytest.mark.parametrize("tag", TAGS)
def test_amp_bf16_arith_reference_kat(cuda, golden, tag):
    _run(golden, tag, "bf16")


def test_amp_kats_are_reference_generated(golden):
    """The fixture carries the reference's provenance fields (wire codec with
    f32 arithmetic, the configuration geometry of BASELINE configs 3-5)."""
    A = golden("amp.json")
    assert A["cfg3_2blk"]["spec"][1:3] == [4096, 32] and A["cfg3_2blk"]["codec"] == "bf16"
    assert A["cfg4_1blk"]["spec"][1:3] == [7168, 56] and A["cfg4_1blk"]["codec"] == "bf16"
    assert A["cfg5_1blk"]["spec"][1:3] == [12288, 96] and A["cfg5_1blk"]["codec"] == "f16"
    assert all(A[t]["arith"] == "f32" for t in TAGS)
