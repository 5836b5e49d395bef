"""rng = "fast": the GPU-cost Gaussian direction (csrc/zo2_rng_fast.h).

Not the reference's stream (that is rng = "exact", bit-exact with numpy's
Philox4x64 + scipy ndtri, tests/test_oracle.py); this checks that
  * the library's host restatement and the oracle's numpy restatement agree
    bit for bit (every step is one IEEE binary32 operation);
  * it is a standard normal: quantiles within 2e-6 of scipy's ndtri for the
    same uniform, moments of 10^6 draws;
  * streams / seeds / positions decorrelate.
The device kernels are checked against the same restatement in
tests/test_gpu_rng_fast.py.
"""
import ctypes

import numpy as np
import pytest
from scipy.special import ndtri


def _host_fast(seed, stream, counter, n):
    from paper_2503_12668_b200 import _lib
    out = np.empty(n, np.float32)
    _lib.call("zo2_host_z_fill_fast", out.ctypes.data_as(ctypes.c_void_p), n, seed, stream,
              counter)
    return out


@pytest.mark.parametrize("seed,stream,counter,n", [(7, 0, 0, 100_000), (2**63 + 5, 0, 2**40 + 3, 9_999),
                                                   (0x182AAE38CFCCB83F, 1, 17, 4096)])
def test_host_restatement_matches_oracle(oracle, seed, stream, counter, n):
    got = _host_fast(seed, stream, counter, n)
    ref = oracle.fast_gauss(seed, stream, counter, n)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_fast_direction_is_standard_normal(oracle):
    r = oracle.fast_raw(20240601, 0, 0, 1_000_000)
    z = oracle.fast_gauss_from_raw(r).astype(np.float64)
    u = ((r >> 9).astype(np.float64) + 0.5) * 2.0**-23
    assert np.max(np.abs(z - ndtri(u))) < 2e-6
    assert abs(z.mean()) < 4e-3 and abs(z.var() - 1.0) < 6e-3
    kurt = ((z - z.mean()) ** 4).mean() / z.var() ** 2
    assert abs(kurt - 3.0) < 0.03
    # extreme raw values stay finite and symmetric
    ext = oracle.fast_gauss_from_raw(np.array([0, 2**32 - 1], np.uint32))
    assert np.all(np.isfinite(ext)) and ext[0] == -ext[1] and ext[1] > 5.0


def test_streams_and_positions_decorrelate(oracle):
    a = oracle.fast_gauss(1, 0, 0, 200_000).astype(np.float64)
    b = oracle.fast_gauss(2, 0, 0, 200_000).astype(np.float64)
    c = oracle.fast_gauss(1, 1, 0, 200_000).astype(np.float64)
    d = oracle.fast_gauss(1, 0, 1, 200_000).astype(np.float64)
    for x in (b, c):
        assert abs(np.corrcoef(a, x)[0, 1]) < 0.01
    assert np.array_equal(a[1:], d[:-1])  # counter shifts the position


def test_rng_config_key(tmp_path):
    from paper_2503_12668_b200.config import RunConfig
    from paper_2503_12668_b200.errors import UsageError
    assert RunConfig(rng="fast").rng == "fast"
    with pytest.raises(UsageError):
        RunConfig(rng="mt19937")
