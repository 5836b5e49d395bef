"""Host-side numeric substrate, mirroring zo2lab numerics.py.

RngState / derive_step_seed / stream ids / ElemFormat keep the reference's
names and semantics (numerics.py:42-190).  The generator itself lives in the
C-ABI library: raw_uint64 and gaussian_fill here call its host restatement
(same source as the sm_100a kernels, csrc/zo2_rng.h), and the device kernels
(zo2_z_fill / zo2_update_perturb) regenerate the identical sequence on the GPU.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib

_MASK64 = (1 << 64) - 1

PERTURB_STREAM = 0   # numerics.py:42
BATCH_STREAM = 1     # numerics.py:43
INIT_STREAM = 2      # numerics.py:44
DATA_STREAM = 3      # numerics.py:45


class ElemFormat(Enum):
    """numerics.py:48-84; `code` is the C-ABI ZO2_* format id."""

    F64 = ("f64", 8, _lib.F64)
    F32 = ("f32", 4, _lib.F32)
    F16 = ("f16", 2, _lib.F16)
    BF16 = ("bf16", 2, _lib.BF16)
    F8E4M3 = ("f8e4m3", 1, _lib.F8E4M3)

    def __init__(self, tag: str, nbytes: int, code: int):
        self.tag = tag
        self.bytes_per_elem = nbytes
        self.code = code

    @property
    def is_arithmetic(self) -> bool:
        return self in (ElemFormat.F64, ElemFormat.F32)

    @property
    def storage_dtype(self) -> np.dtype:
        return {ElemFormat.F64: np.dtype(np.float64), ElemFormat.F32: np.dtype(np.float32),
                ElemFormat.F16: np.dtype(np.float16), ElemFormat.BF16: np.dtype(np.uint16),
                ElemFormat.F8E4M3: np.dtype(np.uint8)}[self]

    @classmethod
    def from_tag(cls, tag: str) -> "ElemFormat":
        for fmt in cls:
            if fmt.tag == tag:
                return fmt
        raise ValueError(f"unknown element format tag: {tag!r}")


CODEC_FORMATS = {"f16": ElemFormat.F16, "bf16": ElemFormat.BF16, "f8": ElemFormat.F8E4M3}


@dataclass(frozen=True)
class RngState:
    """24-byte capturable generator state (numerics.py:140-158)."""

    seed: int
    stream: int = 0
    counter: int = 0

    def __post_init__(self):
        object.__setattr__(self, "seed", int(self.seed) & _MASK64)
        object.__setattr__(self, "stream", int(self.stream) & _MASK64)
        object.__setattr__(self, "counter", int(self.counter) & _MASK64)

    def advanced(self, n: int) -> "RngState":
        return RngState(self.seed, self.stream, self.counter + int(n))


@dataclass
class ConversionSummary:
    """NaN / saturation tallies of the wire codecs (numerics.py:210-217)."""

    nan_count: int = 0
    saturated_count: int = 0

    def add(self, nans: int, saturated: int) -> None:
        self.nan_count += int(nans)
        self.saturated_count += int(saturated)


def derive_step_seed(base_seed: int, step_index: int) -> int:
    """splitmix64 per-step seed (numerics.py:185-190)."""
    return int(_lib.load().zo2_host_derive_step_seed(int(base_seed) & _MASK64,
                                                     int(step_index) & _MASK64))


def raw_uint64(state: RngState, n: int) -> tuple[np.ndarray, RngState]:
    """n Philox4x64-10 draws at absolute positions (numerics.py:161-168)."""
    if n < 1:
        raise ValueError(f"draw count must be >= 1, got {n}")
    out = np.empty(int(n), dtype=np.uint64)
    _lib.call("zo2_host_raw_u64", out.ctypes.data, int(n), state.seed, state.stream,
              state.counter)
    return out, state.advanced(n)


def gaussian_fill(state: RngState, n: int) -> tuple[np.ndarray, RngState]:
    """n standard normals by inverse CDF, one draw each (numerics.py:171-182)."""
    if n < 1:
        raise ValueError(f"draw count must be >= 1, got {n}")
    out = np.empty(int(n), dtype=np.float64)
    _lib.call("zo2_host_gaussian_fill", out.ctypes.data, int(n), state.seed, state.stream,
              state.counter)
    return out, state.advanced(n)
