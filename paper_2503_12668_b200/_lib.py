"""ctypes binding of the sm_100a C-ABI library (include/zo2b200.h).

The library is built in-tree (paper_2503_12668_b200/_lib/libzo2b200.so) by
build.py / __graft_entry__.build().  There is no fallback: if the library is
missing, importing the engine raises ImportError naming the build command.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int32, c_uint32, c_uint64, c_void_p

from .errors import (CapacityError, NonFiniteLossError, SchedulingContractError,
                     StateCorruptionError, UsageError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ZO2_LIB_PATH") or os.path.join(_HERE, "_lib", "libzo2b200.so")

ZO2_OK, ZO2_E_ARG, ZO2_E_CUDA, ZO2_E_CAPACITY = 0, 1, 2, 3
ZO2_E_SCHED, ZO2_E_STATE, ZO2_E_NONFINITE, ZO2_E_UNSUPPORTED = 4, 5, 6, 7

F64, F32, F16, BF16, F8E4M3 = 0, 1, 2, 3, 4

OUT_NONE, OUT_F32, OUT_BF16_T, OUT_SPLIT_T, OUT_BF16, OUT_SPLIT = 0, 1, 2, 3, 4, 5
EPI_STORE, EPI_RESIDUAL, EPI_GELU, EPI_CE, EPI_OPERAND = 0, 1, 2, 3, 4
F64_EPI_STORE, F64_EPI_GELU, F64_EPI_RESIDUAL = 0, 1, 2
CE_PARTS = 148


class SegmentDesc(ctypes.Structure):
    _fields_ = [("offset", c_uint64), ("rows", c_uint32), ("cols", c_uint32),
                ("out_kind", c_int32), ("pad_", c_int32),
                ("out_plus", c_void_p), ("out_minus", c_void_p),
                ("out_plus_lo", c_void_p), ("out_minus_lo", c_void_p)]


class GemmProblem(ctypes.Structure):
    _fields_ = [("a_hi", c_void_p), ("a_lo", c_void_p), ("b_hi", c_void_p), ("b_lo", c_void_p),
                ("bias", c_void_p), ("c", c_void_p), ("c_lo", c_void_p),
                ("targets", c_void_p), ("ce_part", c_void_p)]


_SIGS = {
    "zo2_last_error": (ctypes.c_char_p, []),
    "zo2_version": (c_int, []),
    "zo2_launch_count": (c_uint64, []),
    "zo2_z_fill": (c_int, [c_void_p, c_uint64, c_uint64, c_uint64, c_uint64, c_void_p]),
    "zo2_raw_fill": (c_int, [c_void_p, c_uint64, c_uint64, c_uint64, c_uint64, c_void_p]),
    "zo2_host_raw_u64": (c_int, [c_void_p, c_uint64, c_uint64, c_uint64, c_uint64]),
    "zo2_host_gaussian_fill": (c_int, [c_void_p, c_uint64, c_uint64, c_uint64, c_uint64]),
    "zo2_host_derive_step_seed": (c_uint64, [c_uint64, c_uint64]),
    "zo2_init_normal": (c_int, [c_void_p, c_int, c_uint64, c_double, c_uint64, c_uint64,
                                c_void_p]),
    "zo2_fill_const": (c_int, [c_void_p, c_int, c_uint64, c_double, c_void_p]),
    "zo2_axpy_z": (c_int, [c_void_p, c_int, c_uint64, c_double, c_uint64, c_uint64, c_uint64,
                           c_void_p]),
    "zo2_update_perturb": (c_int, [c_void_p, c_int, c_uint64, c_uint64, c_int, c_void_p,
                                   c_double, c_uint64, c_int, c_double, c_uint64,
                                   POINTER(SegmentDesc), c_int, c_void_p, c_void_p]),
    "zo2_set_k2_ctas_per_sm": (c_int, [c_int]),
    "zo2_set_rng_mode": (c_int, [c_int]),
    "zo2_set_k2_variant": (c_int, [c_int]),
    "zo2_zapprox_bound_probe": (c_int, [c_void_p, c_void_p]),
    "zo2_k2c_fallbacks": (c_int, [POINTER(c_uint64), c_int]),
    "zo2_host_register": (c_int, [c_void_p, c_uint64]),
    "zo2_host_unregister": (c_int, [c_void_p]),
    "zo2_rng_mode": (c_int, []),
    "zo2_z_fill_fast": (c_int, [c_void_p, c_uint64, c_uint64, c_uint64, c_uint64, c_void_p]),
    "zo2_host_z_fill_fast": (c_int, [c_void_p, c_uint64, c_uint64, c_uint64, c_uint64]),
    "zo2_encode": (c_int,[c_void_p, c_void_p, c_int, c_uint64, c_void_p, c_void_p]),
    "zo2_decode": (c_int, [c_void_p, c_void_p, c_int, c_uint64, c_void_p]),
    "zo2_form_g": (c_int, [c_void_p, c_double, c_double, c_void_p, c_void_p, c_void_p]),
    "zo2_embed_dual": (c_int, [c_void_p, c_uint64, c_uint32, c_uint32, c_uint32, c_uint32,
                               c_void_p, c_uint64, c_int, c_void_p, c_double, c_uint64,
                               c_double, c_uint64, c_void_p, c_void_p, c_void_p]),
    "zo2_layernorm": (c_int, [c_void_p, c_uint64, c_uint32, c_void_p, c_void_p, c_void_p,
                              c_void_p, c_void_p]),
    "zo2_to_operand": (c_int, [c_void_p, c_uint64, c_void_p, c_void_p, c_void_p]),
    "zo2_gemm": (c_int, [POINTER(GemmProblem), c_int, c_uint32, c_uint32, c_uint32, c_int,
                         c_void_p]),
    "zo2_gemm_tile_n": (c_int, [c_int]),
    "zo2_set_gemm_variant": (c_int, [c_int]),
    "zo2_set_gemm_raster": (c_int, [c_int, c_int]),
    "zo2_set_attention_variant": (c_int, [c_int]),
    "zo2_ce_reduce": (c_int, [c_void_p, c_uint32, c_uint32, c_int, c_uint64, c_void_p,
                              c_void_p, c_void_p]),
    "zo2_attention": (c_int, [c_void_p, c_void_p, c_uint32, c_uint32, c_uint32, c_uint32,
                              c_void_p,
                              c_void_p, c_void_p]),
    "zo2_f64_gemm": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_uint64, c_uint64,
                             c_uint64, c_int, c_void_p]),
    "zo2_f64_layernorm": (c_int, [c_void_p, c_uint64, c_uint32, c_void_p, c_void_p, c_void_p,
                                  c_void_p]),
    "zo2_f64_embed": (c_int, [c_void_p, c_uint64, c_uint32, c_uint32, c_void_p, c_void_p,
                              c_void_p, c_void_p]),
    "zo2_f64_attention": (c_int, [c_void_p, c_uint32, c_uint32, c_uint32, c_uint32, c_void_p,
                                  c_void_p]),
    "zo2_f64_ce": (c_int, [c_void_p, c_void_p, c_uint64, c_uint32, c_void_p, c_void_p,
                           c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load() -> ctypes.CDLL:
    """Load the library once; raise ImportError if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (nvcc, sm_100a); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    """Map a ZO2_E_* status onto the reference's exception taxonomy."""
    if rc == ZO2_OK:
        return
    msg = (load().zo2_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == ZO2_E_ARG:
        raise UsageError(text)
    if rc == ZO2_E_CAPACITY:
        raise CapacityError(text)
    if rc == ZO2_E_SCHED:
        raise SchedulingContractError(text)
    if rc == ZO2_E_STATE:
        raise StateCorruptionError(text)
    if rc == ZO2_E_NONFINITE:
        raise NonFiniteLossError(text)
    raise RuntimeError(f"zo2 CUDA failure ({rc}) {text}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
