"""B200-native (sm_100a) ZO2 zeroth-order fine-tuning step.

Drop-in for the hot path of zo2lab (arXiv 2503.12668 reproduction): same
engine / runtime / config surface, arithmetic in a C-ABI CUDA library
(include/zo2b200.h, built in-tree as _lib/libzo2b200.so).  There is no CPU
fallback: the library must be built (build.py) and a GPU present to step.
"""
from . import _lib
from .errors import (CapacityError, NonFiniteLossError, SchedulingContractError,
                     StateCorruptionError, UsageError)
from .model import (EMBED_ID, HEAD_ID, ModelSpec, block_id, block_layout, embed_layout,
                    head_layout, module_order, param_count, rng_offsets)
from .numerics import (BATCH_STREAM, DATA_STREAM, INIT_STREAM, PERTURB_STREAM,
                       ConversionSummary, ElemFormat, RngState, derive_step_seed,
                       gaussian_fill, raw_uint64)

__all__ = [
    "CapacityError", "NonFiniteLossError", "SchedulingContractError", "StateCorruptionError",
    "UsageError", "EMBED_ID", "HEAD_ID", "ModelSpec", "block_id", "block_layout",
    "embed_layout", "head_layout", "module_order", "param_count", "rng_offsets",
    "BATCH_STREAM", "DATA_STREAM", "INIT_STREAM", "PERTURB_STREAM", "ConversionSummary",
    "ElemFormat", "RngState", "derive_step_seed", "gaussian_fill", "raw_uint64",
]
