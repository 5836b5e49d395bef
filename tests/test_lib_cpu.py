"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host restatement of the generator (the same source
the sm_100a kernels compile) matches the reference fixtures bit for bit."""
import re

import numpy as np
import pytest

from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "zo2b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(zo2_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    import ctypes
    from paper_2503_12668_b200 import _lib
    lib = _lib.load()
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _lib.EXPORTED, f"{name} missing from the ctypes signature table"
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        getattr(raw, name)


def test_host_rng_matches_reference(golden):
    from paper_2503_12668_b200.numerics import RngState, gaussian_fill, raw_uint64
    g = golden("rng.json")
    for c in g["raw"]:
        out, st = raw_uint64(RngState(c["seed"], c["stream"], c["counter"]), c["n"])
        assert [int(x) for x in out] == c["out"]
        assert st.counter == (c["counter"] + c["n"]) % 2**64
    for c in g["gauss"]:
        z, _ = gaussian_fill(RngState(c["seed"], c["stream"], c["counter"]), c["n"])
        assert [int(x) for x in z.view(np.uint64)] == c["bits"]
    b = g["bulk"]
    z, _ = gaussian_fill(RngState(b["seed"], b["stream"], b["counter"]), b["n"])
    assert int(np.sum(z.view(np.uint64), dtype=np.uint64)) == b["sum_bits_mod64"]


def test_host_rng_equals_oracle_on_random_states(oracle):
    from paper_2503_12668_b200.numerics import RngState, gaussian_fill
    rng = np.random.default_rng(3)
    for _ in range(6):
        s, c = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**44))
        z, _ = gaussian_fill(RngState(s, 0, c), 200_000)
        ref = oracle.gauss(s, 0, c, 200_000)
        assert np.array_equal(z.view(np.uint64), ref.view(np.uint64))


def test_derive_step_seed(golden):
    from paper_2503_12668_b200.numerics import derive_step_seed
    for c in golden("rng.json")["seeds"]:
        assert derive_step_seed(c["base"], c["j"]) == c["out"]


def test_status_codes_map_to_reference_exceptions():
    from paper_2503_12668_b200 import _lib
    from paper_2503_12668_b200.errors import (CapacityError, NonFiniteLossError,
                                              SchedulingContractError, StateCorruptionError,
                                              UsageError)
    for rc, exc in ((1, UsageError), (3, CapacityError), (4, SchedulingContractError),
                    (5, StateCorruptionError), (6, NonFiniteLossError), (2, RuntimeError)):
        with pytest.raises(exc):
            _lib.check(rc, "x")
    _lib.check(0)


def test_argument_errors_raise_without_gpu():
    """Validation happens before any device work, so it is testable here."""
    from paper_2503_12668_b200 import _lib
    from paper_2503_12668_b200.errors import UsageError
    with pytest.raises(UsageError):
        _lib.call("zo2_encode", None, None, 99, 10, None, None)
    with pytest.raises(UsageError):
        _lib.call("zo2_update_perturb", 1, 1, 4, 0, 1, None, 0.1, 0, 1, 1e-3, 0, None, 0,
                  None, None)


def test_host_side_controls_without_gpu():
    """The host-only entry points of the C ABI: version, launch counter, the
    z-generator switch and the tuning setters with their argument checks."""
    from paper_2503_12668_b200 import _lib
    from paper_2503_12668_b200.errors import UsageError
    lib = _lib.load()
    assert lib.zo2_version() >= 1
    n0 = lib.zo2_launch_count()
    assert lib.zo2_launch_count() == n0  # no device work happens here
    mode = lib.zo2_rng_mode()
    try:
        for m in (1, 0):
            _lib.call("zo2_set_rng_mode", m)
            assert lib.zo2_rng_mode() == m
        with pytest.raises(UsageError):
            _lib.call("zo2_set_rng_mode", 2)
        assert b"zo2_set_rng_mode" in lib.zo2_last_error()
    finally:
        _lib.call("zo2_set_rng_mode", mode)
    for fn, good, bad in (("zo2_set_k2_ctas_per_sm", (0, 1, 32), (-1, 33)),
                          ("zo2_set_attention_variant", (0, 1), (-1, 2)),
                          ("zo2_set_gemm_variant", (0, 1, 2), (-1, 3))):
        for v in bad:
            with pytest.raises(UsageError):
                _lib.call(fn, v)
        for v in good:
            _lib.call(fn, v)
        _lib.call(fn, good[0])
    for bad in ((-1, 8), (12, -1), (1025, 8)):
        with pytest.raises(UsageError):
            _lib.call("zo2_set_gemm_raster", *bad)
    _lib.call("zo2_set_gemm_raster", 0, 0)
