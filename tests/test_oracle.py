"""Pin the CPU oracle against fixtures generated from the reference itself
(tests/golden/make_golden.py): RNG, codecs, and a 10-step toy run."""
import numpy as np
import pytest


def test_raw_u64_matches_reference(oracle, golden):
    for c in golden("rng.json")["raw"]:
        got = oracle.raw_u64(c["seed"], c["stream"], c["counter"], c["n"])
        assert [int(x) for x in got] == c["out"]


def test_gaussian_fill_bit_exact(oracle, golden):
    g = golden("rng.json")
    for c in g["gauss"]:
        z = oracle.gauss(c["seed"], c["stream"], c["counter"], c["n"])
        assert [int(x) for x in z.view(np.uint64)] == c["bits"]
    b = g["bulk"]
    z = oracle.gauss(b["seed"], b["stream"], b["counter"], b["n"])
    assert int(np.sum(z.view(np.uint64), dtype=np.uint64)) == b["sum_bits_mod64"]


def test_known_answers_from_survey(oracle):
    z = oracle.gauss(7, 0, 0, 4)
    assert z.tolist() == [1.1362472746449774, -0.5377773613536538, -0.20164360050307614,
                          -0.23941410786242195]
    assert oracle.derive_step_seed(1234, 0) == 0x182AAE38CFCCB83F
    assert oracle.derive_step_seed(1, 0) == 0x5692161D100B05E5


def test_step_seeds(oracle, golden):
    for c in golden("rng.json")["seeds"]:
        assert oracle.derive_step_seed(c["base"], c["j"]) == c["out"]


def test_fill_split_law(oracle):
    # a fill of n followed by m equals a fill of n+m (numerics.py:174-176)
    a = oracle.gauss(5, 0, 3, 11)
    b = np.concatenate([oracle.gauss(5, 0, 3, 4), oracle.gauss(5, 0, 7, 7)])
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("fmt", ["bf16", "f16", "f8"])
def test_codecs_match_reference(oracle, golden, fmt):
    g = golden("codecs.npz")
    bits, nan, sat = oracle.encode(g["x"], fmt)
    assert np.array_equal(bits, g[f"{fmt}_bits"])
    assert [nan, sat] == g[f"{fmt}_counts"].tolist()
    dec = oracle.decode(bits, fmt)
    ref = g[f"{fmt}_dec"]
    same = (dec.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(dec) & np.isnan(ref))
    assert same.all()


def test_e4m3_table(oracle, golden):
    codes = np.arange(256, dtype=np.uint8)
    dec = oracle.decode(codes, "f8").astype(np.float64)
    ref = golden("codecs.npz")["e4m3_table"]
    assert np.array_equal(np.isnan(dec), np.isnan(ref))
    assert np.array_equal(dec[~np.isnan(dec)], ref[~np.isnan(ref)])


def _toy(oracle, golden):
    G = golden("toy.json")
    spec = oracle.Spec(*G["spec"])
    tok, tgt = oracle.gen_synthetic(spec.vocab, spec.seq_len, G["n_samples"], G["seed"])
    return G, spec, tok, tgt


def test_toy_init_and_mezo_run_bit_exact(oracle, golden):
    G, spec, tok, tgt = _toy(oracle, golden)
    z = golden("toy_f32.npz")
    p = oracle.init_params(spec, G["seed"])
    for m in p:
        assert np.array_equal(p[m], z["init::" + m]), m
    eng = oracle.MeZO(spec, p, G["eps"], G["lr"], G["seed"])
    R = G["runs"]["f32"]
    for j in range(G["steps"]):
        idx = oracle.batch_for_step(G["seed"], j, G["n_samples"], G["batch_size"])
        assert idx.tolist() == R["batches"][j]
        eng.step(tok[idx], tgt[idx], j)
    assert eng.losses == R["l_plus"] and eng.losses_minus == R["l_minus"]
    for m in p:
        assert np.array_equal(p[m], z["final::" + m]), m


def test_toy_deferred_zo2_equals_mezo(oracle, golden):
    """SPEC C1: deferred block-wise updates give the monolithic result bit-exactly."""
    G, spec, tok, tgt = _toy(oracle, golden)
    z = golden("toy_f32.npz")
    p = oracle.init_params(spec, G["seed"])
    eng = oracle.Zo2Sequential(spec, p, G["eps"], G["lr"], G["seed"])
    for j in range(G["steps"]):
        idx = oracle.batch_for_step(G["seed"], j, G["n_samples"], G["batch_size"])
        eng.step(tok[idx], tgt[idx], j)
    eng.finalize()
    for m in p:
        assert np.array_equal(p[m], z["final::" + m]), m


def test_perturb_restore_drift_bounded(oracle):
    # +eps, -2eps, +eps returns within 4 ulp of the largest intermediate
    # (test_zo_ref.py:32-47)
    w = (np.random.default_rng(0).standard_normal(10000) * 0.02).astype(np.float32)
    w0 = w.copy()
    eps = 1e-3
    for c in (eps, -2 * eps, eps):
        oracle.axpy_z(w, c, 77, 0)
    z = oracle.gauss(77, 0, 0, w.size)
    inter = np.maximum(np.abs(w0), np.abs(w0) + eps * np.abs(z)).astype(np.float32)
    assert np.max(np.abs(w - w0) / np.spacing(inter)) <= 4.0


def test_gauss_at_matches_fill(oracle):
    """Sampled-position z (used by the whole-block K2 checks) equals the
    sequential fill at the same positions, across Philox block boundaries."""
    n, ctr = 4099, 2**40 + 3
    full = oracle.gauss(77, 0, ctr, n)
    idx = np.random.default_rng(0).choice(n, 600, replace=False).astype(np.uint64)
    assert np.array_equal(oracle.gauss_at(77, 0, ctr, idx).view(np.uint64),
                          full[idx.astype(np.int64)].view(np.uint64))
    w = np.random.default_rng(1).standard_normal(n).astype(np.float32)
    seq = w.copy()
    oracle.axpy_z(seq, -3e-3, 77, ctr)
    at = oracle.axpy_z_at(w[idx.astype(np.int64)], idx, -3e-3, 77, ctr)
    assert np.array_equal(at.view(np.uint32), seq[idx.astype(np.int64)].view(np.uint32))
