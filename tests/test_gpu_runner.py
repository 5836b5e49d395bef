"""MeZO engine (RefEngine drop-in), tied LM head, execute_run artifacts and the
reference's reproducibility / digest-invariance laws (test_harness.py:158-177)."""
import csv

import pytest

pytestmark = pytest.mark.gpu


def _toy_batches(golden, name="toy.json"):
    from paper_2503_12668_b200.data import gen_synthetic
    from paper_2503_12668_b200.engine import batch_for_step
    from paper_2503_12668_b200.numerics import RngState
    G = golden(name)
    ds = gen_synthetic(G["spec"][3], G["spec"][4], G["n_samples"], RngState(G["seed"]),
                       "affine", G["batch_size"])
    return G, [ds.batch(batch_for_step(G["seed"], j, ds.n_samples, ds.batch_size))
               for j in range(G["steps"])]


def test_mezo_engine_matches_reference_bit_exact(cuda, golden):
    from paper_2503_12668_b200.engine import MeZOEngine, TransformerWorkload, ZOConfig
    from paper_2503_12668_b200.model import ModelSpec
    from paper_2503_12668_b200.numerics import RngState
    from paper_2503_12668_b200.runtime import init_params, params_digest
    G, batches = _toy_batches(golden)
    R = G["runs"]["f32"]
    params = init_params(ModelSpec(*G["spec"]), RngState(G["seed"]))
    eng = MeZOEngine(TransformerWorkload(params), ZOConfig(G["eps"], G["lr"], G["steps"],
                                                           G["seed"]))
    for j, b in enumerate(batches):
        eng.step(b, j)
        assert abs(eng.losses[-1] - R["l_plus"][j]) <= 1e-5 * abs(R["l_plus"][j])
        eng._engine.force_pending(R["g"][j])
    assert params_digest(eng.params) == R["digest"]
    assert eng.runtime.log.wire_bytes() == 0          # nothing crosses PCIe


def test_tied_head_teacher_forced(cuda, golden):
    from paper_2503_12668_b200.engine import TransformerWorkload, ZOConfig, Zo2Engine
    from paper_2503_12668_b200.model import ModelSpec
    from paper_2503_12668_b200.numerics import RngState
    from paper_2503_12668_b200.runtime import OffloadRuntime, init_params, params_digest
    G, batches = _toy_batches(golden, "tied.json")
    spec = ModelSpec(*G["spec"], tie_lm_head=True)
    params = init_params(spec, RngState(G["seed"]))
    eng = Zo2Engine(TransformerWorkload(params), ZOConfig(G["eps"], G["lr"], G["steps"],
                                                          G["seed"]),
                    OffloadRuntime(params, k_slots=3), overlap=False)
    for j, b in enumerate(batches):
        eng.step(b, j)
        assert abs(eng.losses[-1] - G["l_plus"][j]) <= 1e-5 * abs(G["l_plus"][j])
        assert abs(eng.losses_minus[-1] - G["l_minus"][j]) <= 1e-5 * abs(G["l_minus"][j])
        eng.force_pending(G["g"][j])
    assert params_digest(eng.finalize()) == G["digest"]


def test_execute_run_artifacts_reproducible_and_schedule_invariant(cuda, tmp_path):
    from paper_2503_12668_b200.config import RunConfig
    from paper_2503_12668_b200.runner import SUMMARY_COLUMNS, execute_run
    base = dict(steps=4, n_blocks=4, seed=99)
    r1 = execute_run(RunConfig(output_dir=str(tmp_path / "a"), **base))
    r2 = execute_run(RunConfig(output_dir=str(tmp_path / "b"), **base))
    assert r1.final_digest == r2.final_digest and r1.losses == r2.losses
    for f in ("metrics.json", "timeline.jsonl", "transfers.jsonl", "summary.csv"):
        assert (tmp_path / "a" / f).exists()
    with open(tmp_path / "a" / "summary.csv") as fh:
        assert next(csv.reader(fh)) == SUMMARY_COLUMNS
    assert r1.uploads == r1.offloads == 4 * 4
    for kw in (dict(overlap=True, arena_slots=4), dict(overlap=False, arena_slots=1),
               dict(overlap=False, arena_slots=2), dict(engine="mezo")):
        r = execute_run(RunConfig(**base, **kw), write_artifacts=False)
        assert r.final_digest == r1.final_digest, kw
        assert r.losses == r1.losses, kw


def test_capacity_error(cuda):
    from paper_2503_12668_b200.config import RunConfig
    from paper_2503_12668_b200.errors import CapacityError
    from paper_2503_12668_b200.runner import execute_run
    with pytest.raises(CapacityError):
        execute_run(RunConfig(steps=1, device_capacity_bytes=1e5), write_artifacts=False)
