"""RunConfig keys, validation and key=value parsing (harness/config.py:44-206)."""
import pytest

from paper_2503_12668_b200.config import RunConfig, build_config, parse_config_text
from paper_2503_12668_b200.errors import UsageError


def test_defaults_and_overrides(tmp_path):
    p = tmp_path / "run.cfg"
    p.write_text("# toy\nn_blocks = 6\ncodec=bf16\narith = bf16\ncost.flops_per_sec = 1e12\n")
    cfg = build_config(str(p), {"--steps": "7", "update-mode": "naive"}
                       if False else {"steps": "7", "update-mode": "naive"})
    assert (cfg.n_blocks, cfg.codec, cfg.arith, cfg.steps, cfg.update_mode) == (
        6, "bf16", "bf16", 7, "naive")
    assert cfg.cost.flops_per_sec == 1e12
    flat = cfg.to_flat()
    assert build_config(None, flat).to_flat() == flat


@pytest.mark.parametrize("bad", [{"engine": "x"}, {"backend": "mpi"}, {"codec": "f4"},
                                 {"arith": "f16"}, {"arena_slots": "2"}, {"steps": "0"},
                                 {"n_samples": "0"}, {"nope": "1"}, {"cost.nope": "1"},
                                 {"overlap": "maybe"}, {"ranks": "0"}])
def test_bad_keys_raise_usage_error(bad):
    with pytest.raises(UsageError):
        build_config(None, bad)


def test_parse_errors():
    with pytest.raises(UsageError):
        parse_config_text("no equals sign here")
    with pytest.raises(UsageError):
        build_config("/nonexistent/file.cfg")


def test_model_spec_from_preset():
    cfg = RunConfig(preset="opt-1.3b", seq_len=512)
    s = cfg.model_spec()
    assert (s.n_blocks, s.dim, s.n_heads, s.vocab, s.seq_len) == (24, 2048, 32, 50272, 512)


def test_reference_defaults_and_aliases():
    """The reference's default arith (f64), its f64 -> f32 switch under a codec
    (harness/config.py:112-113) and its backends accepted as cuda aliases."""
    assert RunConfig().arith == "f64"
    assert RunConfig(codec="bf16").arith == "f32"
    assert RunConfig(codec="bf16", arith="bf16").arith == "bf16"
    with pytest.warns(UserWarning):
        cfg = build_config(None, {"backend": "threaded"})
    assert cfg.backend == "cuda"
    with pytest.warns(UserWarning):
        assert build_config(None, {"backend": "simulated"}).backend == "cuda"
