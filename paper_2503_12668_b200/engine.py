"""ZO2 and MeZO engines on B200 (drop-in for zo2lab zo2_engine.py / zo_ref.py).

Zo2Engine keeps the reference's constructor, step/finalize/train contract and
bookkeeping (RngStateManager FIFO, PendingGradient gate, DAG validation,
zo2_engine.py:38-345); the arithmetic runs in the sm_100a library:

  per module (zo2_engine.py:183-204 dual_forward), one compute-stream task:
    K2  zo2_update_perturb: deferred update with lrs (gated on g != 0), then
        +eps / -2eps / +eps with rs, emitting W+-eps z as GEMM operands and
        leaving the restored weights in the arena (codec-encoded if active)
    forward kernels for both signs (model.DualForward)
  head: fused head GEMM + CE partials, CE reduce, K10 forms g on device; the
  next step's K2 reads g from HBM, so no host round trip sits between steps'
  kernels -- the host only reads (l+, l-, g) back for the returned value.
Upload / offload run on their own streams (scheduler.enqueue_dag).
"""
from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import (NonFiniteLossError, SchedulingContractError, StateCorruptionError,
                     UsageError)
from .model import (EMBED_ID, HEAD_ID, DualForward, F64Forward, ModelSpec, module_order,
                    module_size, rng_offsets)
from .numerics import (BATCH_STREAM, PERTURB_STREAM, ElemFormat, RngState, derive_step_seed,
                       raw_uint64)
from .runtime import ModelParams, OffloadRuntime
from .scheduler import (CudaLanes, Lane, build_iteration_dag, build_prepare_dag, ckey,
                        close_step, cross_step_edges, enqueue_dag, okey, pkey, ukey,
                        validate_timeline)


# markers for update coefficients resolved when the iteration's g is known
_G_PREV, _G_CUR = object(), object()

# z generator per engine (zo2b200.h zo2_set_rng_mode): "exact" is the
# reference's stream (numerics.py:161-182), "fast" the GPU-cost Philox4x32
# direction; the mode is process-wide in the library and set before every
# enqueue, so engines with different modes can share a process.
RNG_MODES = {"exact": 0, "fast": 1}


@dataclass(frozen=True)
class ZOConfig:
    """zo_ref.py:29-42."""

    eps: float
    lr: float
    steps: int
    seed: int

    def __post_init__(self):
        if self.eps <= 0:
            raise ValueError("eps must be > 0")
        if self.lr <= 0:
            raise ValueError("lr must be > 0")
        if self.steps < 1:
            raise ValueError("steps must be >= 1")


def step_perturb_state(seed: int, step_index: int) -> RngState:
    """zo_ref.py:45-46."""
    return RngState(derive_step_seed(seed, step_index), PERTURB_STREAM, 0)


def batch_for_step(seed: int, step_index: int, n_samples: int, batch_size: int) -> np.ndarray:
    """zo_ref.py:49-56: batch indices from the BATCH stream."""
    if n_samples < 1:
        raise ValueError("cannot sample from an empty dataset")
    raw, _ = raw_uint64(RngState(derive_step_seed(seed, step_index), BATCH_STREAM, 0),
                        batch_size)
    return (raw % np.uint64(n_samples)).astype(np.int64)


@dataclass
class PendingGradient:
    """zo2_engine.py:38-51: one scalar, valid iff g != 0."""

    g: float = 0.0
    valid: bool = False

    def set(self, g: float) -> None:
        self.g = float(g)
        self.valid = g != 0.0

    def clear(self) -> None:
        self.g = 0.0
        self.valid = False


@dataclass
class _RsbEntry:
    step: int
    module: str
    state: RngState


class RngStateManager:
    """zo2_engine.py:61-110 (rsb FIFO + lrs_map); misalignment is fatal."""

    def __init__(self, seed: int):
        self.seed = seed
        self.rsb: deque[_RsbEntry] = deque()
        self.lrs_map: dict[str, RngState] = {}
        self.storage: dict[int, RngState] = {}
        self.current_seed: int | None = None

    def begin_iteration(self, step_seed: int) -> None:
        self.current_seed = step_seed
        self.set_state(step_seed, RngState(step_seed, PERTURB_STREAM, 0))

    def set_state(self, seed: int, state: RngState) -> None:
        self.storage[seed] = state

    def get_state(self, seed: int | None = None) -> RngState:
        return self.storage[self.current_seed if seed is None else seed]

    def push_rs(self, step: int, module: str, state: RngState) -> None:
        self.rsb.append(_RsbEntry(step, module, state))
        self.lrs_map[module] = state

    def _pop(self, module: str) -> RngState:
        e = self.rsb.popleft()
        if e.module != module:
            raise StateCorruptionError(f"rsb misaligned: expected {module}, found {e.module} "
                                       f"from step {e.step}")
        return e.state

    def pop_backlog(self, module: str, current_step: int) -> RngState | None:
        if self.rsb and self.rsb[0].step < current_step:
            return self._pop(module)
        return None

    def pop_current(self, module: str, current_step: int) -> RngState:
        if not self.rsb or self.rsb[0].step != current_step:
            raise StateCorruptionError(f"no state recorded for {module} in step {current_step}")
        return self._pop(module)


@dataclass
class ModuleHandle:
    module: str
    size: int
    transferable: bool


class TransformerWorkload:
    """Adapter the engines drive (model.py:335-393 surface): module sequence and
    shapes; the forward itself runs in DualForward on the device."""

    def __init__(self, params: ModelParams, arith: str = "f32"):
        self.params = params
        self.spec: ModelSpec = params.spec
        self.arith = arith

    def modules(self) -> list[ModuleHandle]:
        return [ModuleHandle(m, module_size(self.spec, m), m not in (EMBED_ID, HEAD_ID))
                for m in module_order(self.spec)]

    @property
    def tied_stash_bytes(self) -> int:
        return 0  # the tied head reads the embedding's W+- operands directly

    def activation_bytes(self, module: str, batch_size: int) -> int:
        width = self.spec.vocab if module == HEAD_ID else self.spec.dim
        return batch_size * self.spec.seq_len * width * 4


class _DeviceStep:
    """Shared device state of both engines: dual forward, scalars, pinned I/O."""

    def __init__(self, spec: ModelSpec, arith: str, device, operand_sets: int = 1):
        self.spec, self.arith, self.device = spec, arith, torch.device(device)
        self.operand_sets = operand_sets
        self.fwd: DualForward | None = None
        self.d_out = torch.zeros(3, dtype=torch.float64, device=self.device)  # l+, l-, g
        self.d_flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.h_out = torch.zeros(4, dtype=torch.float64, pin_memory=True)
        self.h_tok = None
        self.offsets = rng_offsets(spec)

    def ensure(self, batch_size: int) -> DualForward:
        if self.fwd is None or self.fwd.B != batch_size:
            self.fwd = None
            torch.cuda.empty_cache()
            if self.arith == "f64":
                self.fwd = F64Forward(self.spec, batch_size, self.device)
            else:
                self.fwd = DualForward(self.spec, batch_size, self.arith, self.device,
                                       self.operand_sets)
            T = self.fwd.T
            # a ring of pinned staging buffers: step_async may enqueue several
            # iterations before the first one's token copy has executed
            self.h_tok_ring = [torch.empty(2, T, dtype=torch.int64, pin_memory=True)
                               for _ in range(4)]
            self.h_tok_ev = [None] * len(self.h_tok_ring)
            self.h_tok_i = 0
            self.h_tok = self.h_tok_ring[0]
        return self.fwd

    def stage_batch(self, batch, stream: torch.cuda.Stream) -> tuple[int, int]:
        tokens, targets = (np.asarray(x) for x in batch)
        if tokens.ndim != 2 or tokens.shape != targets.shape:
            raise ValueError(f"tokens {tokens.shape} / targets {targets.shape} must be (B, S)")
        if tokens.shape[1] > self.spec.seq_len:
            raise ValueError(f"tokens shape {tokens.shape} invalid for seq_len {self.spec.seq_len}")
        if tokens.shape[1] != self.spec.seq_len:
            raise ValueError("the B200 forward requires full-length sequences (S == seq_len)")
        if tokens.size and (tokens.min() < 0 or tokens.max() >= self.spec.vocab):
            raise ValueError("token id out of range")
        # the CE epilogue only records a target logit for 0 <= target < vocab:
        # refuse instead of silently forming a wrong loss (and a wrong g)
        if targets.size and (targets.min() < 0 or targets.max() >= self.spec.vocab):
            raise ValueError(f"target id out of range [0, {self.spec.vocab})")
        fwd = self.ensure(tokens.shape[0])
        i = self.h_tok_i = (self.h_tok_i + 1) % len(self.h_tok_ring)
        if self.h_tok_ev[i] is not None:
            self.h_tok_ev[i].synchronize()  # its previous copy has been read
        self.h_tok = self.h_tok_ring[i]
        self.h_tok[0].numpy()[:] = tokens.reshape(-1)
        self.h_tok[1].numpy()[:] = targets.reshape(-1)
        with torch.cuda.stream(stream):
            fwd.ids.copy_(self.h_tok[0], non_blocking=True)
            fwd.targets.copy_(self.h_tok[1], non_blocking=True)
            ev = self.h_tok_ev[i] = torch.cuda.Event()
            ev.record(stream)
        return tokens.shape[0], tokens.shape[1]

    def read_out(self, stream: torch.cuda.Stream) -> None:
        with torch.cuda.stream(stream):
            self.h_out[:3].copy_(self.d_out, non_blocking=True)
            self.h_out[3:4].copy_(self.d_flag.to(torch.float64), non_blocking=True)


class Zo2Engine:
    """Block-offloaded dual-forward optimizer on B200 (zo2_engine.py:113-345)."""

    def __init__(self, workload: TransformerWorkload, cfg: ZOConfig, runtime: OffloadRuntime,
                 *, overlap: bool = True, backend: str = "cuda", update_mode: str = "deferred",
                 cost=None, trace=None, validate: bool = True, prepare_lane: bool = True,
                 operand_sets: int | None = None, rng: str = "exact",
                 pipeline_steps: bool = True):
        if update_mode not in ("deferred", "naive"):
            raise ValueError(f"unknown update_mode {update_mode!r}")
        if rng not in RNG_MODES:
            raise ValueError(f"unknown rng {rng!r} (one of {tuple(RNG_MODES)})")
        self.rng = rng
        if overlap and runtime.k_slots < 3:
            raise ValueError("overlap requires at least 3 arena slots")
        if backend != "cuda":
            raise ValueError("this engine runs on the 'cuda' backend only")
        if workload.arith == "f64":
            # the reference's default arithmetic: f64 buckets, perturbed in place
            # around two f64 forwards (no operand emission, so no prepare lane)
            if runtime.codec is not None:
                raise UsageError("arith f64 with a wire codec: the reference runs codecs with "
                                 "f32 arithmetic (harness/config.py:112-113)")
            if runtime.wire_fmt is not ElemFormat.F64:
                raise UsageError("arith f64 needs f64 parameters: "
                                 "init_params(spec, state, ElemFormat.F64)")
            prepare_lane = False
        self.workload, self.cfg, self.runtime = workload, cfg, runtime
        self.overlap, self.backend, self.update_mode = overlap, backend, update_mode
        self.cost, self.trace, self.validate = cost, trace, validate
        self.mgr = RngStateManager(cfg.seed)
        self.pending = PendingGradient()
        self.losses: list[float] = []
        self.losses_minus: list[float] = []
        self.gs: list[float] = []
        self.timelines = []
        self._handles = {h.module: h for h in workload.modules()}
        self._order = [h.module for h in workload.modules()]
        self._blocks = [m for m in self._order if self._handles[m].transferable]
        self.prepare_lane = prepare_lane
        # operand sets: 2 lets K2 of block i+1 run beside the forward of block i
        # (None = 2 unless the device capacity only admits one set)
        self._sets_auto = operand_sets is None and prepare_lane and update_mode == "deferred"
        if prepare_lane and update_mode == "deferred":
            self.operand_sets = 2 if operand_sets is None else int(operand_sets)
        else:
            self.operand_sets = 1
        self.lanes = CudaLanes(runtime.device)
        self.dev = _DeviceStep(workload.spec, workload.arith, runtime.device, self.operand_sets)
        self._set_k2_grid()
        self._booked: dict[str, int] = {}  # DevicePool booking of self.dev.fwd
        self._booked_fwd = None
        self._async: list = []
        # cross-step pipelining: the previous iteration
        # whose tail the next one overlaps instead of a full step barrier
        self.pipeline_steps = pipeline_steps
        self._prev_enq = None
        # per-iteration (l+, l-, g, flag) of step_async until drain()
        self._hist = torch.zeros(1024, 4, dtype=torch.float64, device=runtime.device)
        # data parallel: loss sums are all-reduced before g is formed (K10)
        self.dist_group = None
        self.world = 1
        # trace (zo2_engine.py:156-159): events of an enqueued iteration are
        # buffered and delivered by _finish, once the g their update
        # coefficients depend on is known; _g_last is the g the next deferred
        # update applies.  trace_update_same_step (MeZOEngine): report each
        # step's update at that step's end, in RefEngine order (zo_ref.py:97-112)
        self._tev: list = []
        self._g_last = 0.0
        self.trace_update_same_step = False

    def _set_k2_grid(self) -> None:
        # K2 grid from occupancy (0) also beside the forward: measured faster
        # than capping it at 1-2 CTAs per SM (tools/ab_sets.sh)
        import os
        conc = int(os.environ.get("ZO2_K2_CONCURRENT_CTAS", "0"))
        _lib.call("zo2_set_k2_ctas_per_sm", conc if self.operand_sets >= 2 else 0)

    def _choose_operand_sets(self, batch_size: int) -> None:
        """Auto mode: drop to one operand set when two would not fit the
        device capacity (DevicePool, runtime.py:94-142)."""
        if not self._sets_auto:
            return
        fwd = self.dev.fwd
        if fwd is not None and fwd.B == batch_size:
            return
        pool = self.runtime.pool
        need = DualForward.estimate_nbytes(self.workload.spec, batch_size,
                                           self.workload.arith, 2)
        # the current forward's booking is released when it is rebuilt
        booked = sum(self._booked.values())
        sets = 2 if pool.used - booked + need <= pool.capacity else 1
        if sets != self.operand_sets:
            self.operand_sets = sets
            self.dev.operand_sets = sets
            self.dev.fwd = None
            self._set_k2_grid()

    def enable_data_parallel(self, group=None, shard_transfers: bool = False) -> bool:
        """Shard the batch over torch.distributed ranks: every rank perturbs with
        the same seed and applies the same g; only the two f64 loss sums cross
        NVLink (one NCCL all-reduce per step on the compute stream).

        shard_transfers (node-wide shared masters, runtime.SharedHostMasters):
        each rank also moves only its 1/world slice of every block over PCIe and
        completes the arena with an NVLink all-gather.  Returns whether the
        transfers are sharded."""
        import torch.distributed as dist
        self.dist_group = group or dist.group.WORLD
        self.world = dist.get_world_size(self.dist_group)
        sharded = False
        if shard_transfers and not getattr(self.runtime, "resident", False):
            sharded = self.runtime.enable_sharding(dist.get_rank(self.dist_group), self.world)
        params = getattr(self.runtime, "params", None)
        if (self.world > 1 and getattr(params, "shared_masters", False) and not sharded
                and not getattr(self.runtime, "resident", False)):
            # every rank would upload and offload whole blocks of one shared
            # copy: a rank running ahead would hand the next one already
            # updated weights.  One writer per byte needs sharded transfers.
            raise UsageError("node-shared host masters need sharded transfers "
                             "(enable_data_parallel(shard_transfers=True), block size "
                             "divisible by the world size and a working in-place "
                             "all-gather); use per-rank masters otherwise")
        return sharded

    # -- bookkeeping of one module visit (zo2_engine.py:187-203) -------------
    def _visit(self, module: str, step: int) -> tuple[RngState, RngState | None, bool]:
        rs = self.mgr.get_state()
        if rs.counter != self.dev.offsets[module]:
            raise StateCorruptionError(f"rs counter {rs.counter} != bucket offset of {module}")
        lrs = self.mgr.pop_backlog(module, step)
        update = self.pending.valid
        if update and lrs is None:
            raise StateCorruptionError(f"pending update for {module} but no saved state (lrs)")
        self.mgr.push_rs(step, module, rs)
        size = self._handles[module].size
        if size:
            if update and not self.trace_update_same_step:
                self._emit("update", module, _G_PREV, lrs)
            self._emit_perturbs(module, rs)
        self.mgr.set_state(rs.seed, rs.advanced(size))
        return rs, lrs, update

    def _emit(self, op: str, module: str, coef, state: RngState | None) -> None:
        """Buffer one trace event of the iteration being enqueued; coef may be
        _G_PREV / _G_CUR (resolved in _finish to -(lr*g) of the previous /
        this iteration)."""
        if self.trace is not None and state is not None:
            self._tev.append((op, module, coef, (state.seed, state.stream, state.counter)))

    def _emit_perturbs(self, module: str, rs: RngState) -> None:
        """The three perturbation passes of one module visit (zo2_engine.py:
        195-202): +eps, -2eps, +eps, all from the same state."""
        eps = self.cfg.eps
        for c in (eps, -2.0 * eps, eps):
            self._emit("perturb", module, c, rs)

    def _deliver(self, events, g: float | None) -> None:
        """Resolve and hand an iteration's buffered events to the trace callback
        in enqueue order; g None (non-finite losses): no update of this step."""
        if self.trace is None:
            return
        lr = self.cfg.lr
        for op, module, coef, st in events:
            if coef is _G_PREV:
                if self._g_last == 0.0:  # gated off on the device (g == 0)
                    continue
                coef = -(lr * self._g_last)
            elif coef is _G_CUR:
                if g is None:
                    continue
                coef = -(lr * g)
            self.trace({"op": op, "module": module, "coef": coef, "state": st})

    def _k2(self, buf: torch.Tensor, fmt_code: int, module: str, update: int, lrs_seed: int,
            perturb: bool, rs_seed: int, descs, stream) -> None:
        n = self._handles[module].size
        if n == 0:
            return
        prof = self.dev.fwd.prof if self.dev.fwd is not None else None
        if prof is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        _lib.call("zo2_update_perturb", buf.data_ptr(), fmt_code, n, self.dev.offsets[module],
                  int(update), self.dev.d_out[2:].data_ptr(), self.cfg.lr, lrs_seed,
                  int(perturb), self.cfg.eps, rs_seed, descs, len(descs),
                  self.runtime.d_conv.data_ptr(), stream.cuda_stream)
        if prof is not None:
            e1.record(stream)
            # work unit: Gaussian draws regenerated (update pass + perturb pass)
            prof.append(("k2", float(n * ((1 if update else 0) + (1 if perturb else 0))), e0, e1))

    # -- per-module compute tasks -------------------------------------------
    def _bookkeep(self, module: str, step: int):
        if self.update_mode == "naive":
            rs = self.mgr.get_state()
            self.mgr.push_rs(step, module, rs)
            if self._handles[module].size:
                self._emit_perturbs(module, rs)
            self.mgr.set_state(rs.seed, rs.advanced(self._handles[module].size))
            return rs, 0, False
        rs, lrs, update = self._visit(module, step)
        return rs, (lrs.seed if lrs is not None else 0), update

    def _set_of(self, module: str) -> int:
        return self._blocks.index(module) % self.operand_sets

    def _prepare(self, module: str, step: int, stream: torch.cuda.Stream) -> None:
        """P task (prepare lane): K2 for a block or the head."""
        fwd = self.dev.fwd
        rs, lrs_seed, update = self._bookkeep(module, step)
        if module == HEAD_ID:
            self._k2(self.runtime.persistent[HEAD_ID], _lib.F32, module, update, lrs_seed, True,
                     rs.seed, fwd.head_descs(), stream)
        else:
            slot = self.runtime.slot_for(self._blocks.index(module))
            self._k2(self.runtime.slot_bucket(slot), self.runtime.wire_fmt.code, module, update,
                     lrs_seed, True, rs.seed, fwd.block_descs(self._set_of(module)), stream)

    def _forward(self, module: str, stream: torch.cuda.Stream) -> None:
        """C task of the prepare DAG (compute lane): forward from W+- operands."""
        fwd = self.dev.fwd
        s = stream.cuda_stream
        if module == HEAD_ID:
            self._head_tail(fwd, stream)
        else:
            fwd.block_forward(s, self._set_of(module))

    def _head_tail(self, fwd, stream) -> None:
        fwd.head_forward(stream.cuda_stream)
        self._form_g(fwd, stream)

    def _form_g(self, fwd, stream) -> None:
        """Loss sums (all-reduced under data parallel) -> l+, l-, g on device."""
        s = stream.cuda_stream
        if self.dist_group is not None:
            from .parallel import allreduce_loss_sums
            with torch.cuda.stream(stream):
                allreduce_loss_sums(fwd.d_sums, self.dist_group)
        _lib.call("zo2_form_g", fwd.d_sums.data_ptr(), float(fwd.T * self.world),
                  self.cfg.eps, self.dev.d_out.data_ptr(), self.dev.d_flag.data_ptr(), s)

    def _compute(self, module: str, step: int, seq: int, stream: torch.cuda.Stream) -> None:
        """Reference-shaped C task: K2 and forward of one module on one lane
        (the embedding always; every module in naive update mode)."""
        if self.workload.arith == "f64":
            self._compute_f64(module, step, stream)
            return
        fwd = self.dev.fwd
        rs, lrs_seed, update = self._bookkeep(module, step)
        s = stream.cuda_stream
        if module == EMBED_ID:
            table = self.runtime.persistent[EMBED_ID]
            fwd.embed_forward(table, self.dev.offsets[EMBED_ID], update,
                              self.dev.d_out[2:], self.cfg.lr, lrs_seed, self.cfg.eps, rs.seed,
                              seq, s)
            self._k2(table, _lib.F32, module, update, lrs_seed, True, rs.seed,
                     fwd.embed_descs(), stream)
        elif module == HEAD_ID:
            self._k2(self.runtime.persistent[HEAD_ID], _lib.F32, module, update, lrs_seed, True,
                     rs.seed, fwd.head_descs(), stream)
            self._head_tail(fwd, stream)
        else:
            slot = self.runtime.slot_for(self._blocks.index(module))
            self._k2(self.runtime.slot_bucket(slot), self.runtime.wire_fmt.code, module, update,
                     lrs_seed, True, rs.seed, fwd.block_descs(0), stream)
            fwd.block_forward(s, 0)

    def _compute_f64(self, module: str, step: int, stream: torch.cuda.Stream) -> None:
        """arith=f64: the reference's dual_forward verbatim (zo2_engine.py:
        183-204) on the device -- deferred update (K2, gated on g != 0 on
        device), then +eps / forward(+) / -2eps / forward(-) / +eps in place on
        the f64 bucket, each pass one zo2_axpy_z over the module's z."""
        fwd = self.dev.fwd
        rs, lrs_seed, update = self._bookkeep(module, step)
        rt = self.runtime
        if module in (EMBED_ID, HEAD_ID):
            buf = rt.persistent[module]
        else:
            buf = rt.slot_bucket(rt.slot_for(self._blocks.index(module)))
        n = self._handles[module].size
        s = stream.cuda_stream
        if n and update:
            self._k2(buf, _lib.F64, module, 1, lrs_seed, False, 0, self._update_descs(module),
                     stream)
        off, eps = self.dev.offsets[module], self.cfg.eps

        def axpy(coef):
            if n:
                _lib.call("zo2_axpy_z", buf.data_ptr(), _lib.F64, n, coef, rs.seed, rs.stream,
                          off, s)
        axpy(eps)
        fwd.forward(module, buf, 0, s)
        axpy(-2.0 * eps)
        fwd.forward(module, buf, 1, s)
        axpy(eps)
        if module == HEAD_ID:
            self._form_g(fwd, stream)

    @staticmethod
    def _fmt_of(t: torch.Tensor) -> int:
        return _lib.F64 if t.dtype == torch.float64 else _lib.F32

    def _naive_update(self, module: str, step: int, stream: torch.cuda.Stream) -> None:
        """zo2_engine.py:251-260: update after g with the same-step state (no gate)."""
        rs = self.mgr.pop_current(module, step)
        if self._handles[module].size == 0:
            return
        self._emit("update", module, _G_CUR, rs)
        if module in (EMBED_ID, HEAD_ID):
            buf = self.runtime.persistent[module]
            code = self._fmt_of(buf)
        else:
            buf = self.runtime.slot_bucket(self.runtime.slot_for(self._blocks.index(module)))
            code = self.runtime.wire_fmt.code
        descs = self._update_descs(module)
        self._k2(buf, code, module, 2, rs.seed, False, 0, descs, stream)

    def _update_descs(self, module: str):
        from .model import module_layout, segments
        segs = segments(module_layout(self.workload.spec, module))
        arr = (_lib.SegmentDesc * len(segs))()
        for k, sg in enumerate(segs):
            arr[k].offset = sg.offset
            arr[k].rows = 1 if len(sg.shape) == 1 else sg.shape[0]
            arr[k].cols = sg.shape[-1]
            arr[k].out_kind = _lib.OUT_NONE
        return arr

    def _book_pool(self, fwd: DualForward) -> None:
        """Book the dual forward's device working set in the DevicePool; a
        rebuilt forward (new batch size or operand sets) replaces the booking."""
        if self._booked_fwd is fwd:
            return
        pool = self.runtime.pool
        for cat, nb in self._booked.items():
            pool.free(cat, nb)
        self._booked, self._booked_fwd = {}, None
        for cat, nb in fwd.nbytes().items():
            pool.alloc(cat, nb)
            self._booked[cat] = nb
        self._booked_fwd = fwd

    # -- one iteration (zo2_engine.py:264-316) --------------------------------
    def step(self, batch, step_index: int) -> float:
        """Reference contract: enqueue the whole iteration, synchronise, return g."""
        enq, dag, recs, events = self._enqueue(batch, step_index)
        self.dev.read_out(self.lanes[Lane.COMPUTE])
        self.lanes.synchronize()
        lp, lm, g, flag = (float(x) for x in self.dev.h_out.tolist())
        return self._finish(step_index, enq, dag, recs, lp, lm, g, flag, events)

    def step_async(self, step_index: int, batch=None) -> None:
        """Enqueue one iteration without waiting (device-resident batch when
        `batch` is None).  The next iteration's deferred update reads g from
        HBM and is gated on g != 0 on the device; drain() synchronises and
        performs the per-step checks of step()."""
        enq, dag, recs, events = self._enqueue(batch, step_index)
        slot = len(self._async)
        if slot >= self._hist.shape[0]:
            raise RuntimeError("too many outstanding async steps; call drain()")
        with torch.cuda.stream(self.lanes[Lane.COMPUTE]):
            self._hist[slot, :3].copy_(self.dev.d_out)
            self._hist[slot, 3:4].copy_(self.dev.d_flag.to(torch.float64))
        self._async.append((step_index, enq, dag, recs, events))
        if self.update_mode != "naive":
            self.pending.valid, self.pending.g = True, float("nan")  # resolved on device

    def drain(self) -> list[float]:
        """Synchronise and run the per-step checks of every iteration enqueued
        by step_async, in order.  If one of them fails (non-finite losses, a
        scheduling violation) the error names that step; the iterations queued
        after it already ran with g = 0 on the device (K10 zeroes g on a
        non-finite loss, so their deferred updates were gated off) and are
        discarded, and the pending gradient is cleared to match the device."""
        self.lanes.synchronize()
        hist = self._hist[: len(self._async)].cpu().tolist()
        gs = []
        entries, self._async = self._async, []
        try:
            for (j, enq, dag, recs, events), (lp, lm, g, flag) in zip(entries, hist):
                gs.append(self._finish(j, enq, dag, recs, lp, lm, g, flag, events))
        except Exception:
            self.pending.clear()
            self._g_last = 0.0
            self.dev.d_out[2].zero_()
            self._prev_enq = None
            raise
        return gs

    def _finish(self, step_index, enq, dag, recs, lp, lm, g, flag, events=()) -> float:
        timeline = enq.timeline()
        self.runtime.commit_records(timeline, recs)
        if flag != 0.0 or not (math.isfinite(lp) and math.isfinite(lm)):
            self._deliver(events, None)
            raise NonFiniteLossError(f"step {step_index}: l+={lp}, l-={lm}")
        if self.validate:
            bad = validate_timeline(timeline, dag, tol=2e-6)
            if bad:
                raise SchedulingContractError("; ".join(str(v) for v in bad[:5]))
        self.timelines.append((step_index, timeline))
        self._deliver(events, g)
        if self.update_mode == "naive":
            self.pending.clear()
            self._g_last = 0.0
        else:
            self.pending.set(g)
            self._g_last = g
        self.losses.append(lp)
        self.losses_minus.append(lm)
        self.gs.append(g)
        return g

    def _enqueue(self, batch, step_index: int):
        cfg, rt = self.cfg, self.runtime
        _lib.call("zo2_set_rng_mode", RNG_MODES[self.rng])
        rt.current_step = step_index
        self.mgr.begin_iteration(derive_step_seed(cfg.seed, step_index))
        comp = self.lanes[Lane.COMPUTE]
        if batch is not None:
            self._choose_operand_sets(int(np.asarray(batch[0]).shape[0]))
            _, seq = self.dev.stage_batch(batch, comp)
        elif self.dev.fwd is None:
            raise ValueError("step_async(batch=None) needs a batch staged by an earlier step")
        else:
            seq = self.workload.spec.seq_len
        self._book_pool(self.dev.fwd)
        naive = self.update_mode == "naive"
        wire = {b: rt.block_nbytes for b in self._blocks}
        fns = {ckey(m): (lambda st, m=m: self._compute(m, step_index, seq, st))
               for m in self._order}
        if naive or not self.prepare_lane:
            dag = build_iteration_dag(self._blocks, k_slots=rt.k_slots, overlap=self.overlap,
                                      naive_update=naive, wire_bytes=wire,
                                      embed_id=self._order[0], head_id=self._order[-1])
        else:
            dag = build_prepare_dag(self._blocks, k_slots=rt.k_slots, overlap=self.overlap,
                                    wire_bytes=wire, operand_sets=self.operand_sets,
                                    embed_id=self._order[0], head_id=self._order[-1])
            for m in self._order[1:]:
                fns[pkey(m)] = lambda st, m=m: self._prepare(m, step_index, st)
                fns[ckey(m)] = lambda st, m=m: self._forward(m, st)
        for i, b in enumerate(self._blocks):
            slot = rt.slot_for(i)
            fns[ukey(b)] = lambda st, b=b, slot=slot: rt.upload(b, slot, step_index, st, ukey(b))
            fns[okey(b)] = lambda st, b=b, slot=slot: rt.offload(b, slot, step_index, st, okey(b))
            if naive:
                fns[ukey(b, 2)] = (lambda st, b=b, slot=slot:
                                   rt.upload(b, slot, step_index, st, ukey(b, 2)))
                fns[okey(b, 2)] = (lambda st, b=b, slot=slot:
                                   rt.offload(b, slot, step_index, st, okey(b, 2)))
        if naive:
            for m in self._order:
                fns[ckey(m, 2)] = lambda st, m=m: self._naive_update(m, step_index, st)
        carry = None if naive or not self.prepare_lane else self._carry()
        prev = self._prev_enq
        enq = enqueue_dag(dag, self.lanes, fns, carry=carry,
                          base=None if prev is None else prev.origin_event)
        close_step(self.lanes)
        self._prev_enq = enq if (self.pipeline_steps and not naive and self.prepare_lane) else None
        expected = 0 if naive else len(self._order)
        if len(self.mgr.rsb) != expected:
            raise StateCorruptionError(f"rsb holds {len(self.mgr.rsb)} entries, "
                                       f"expected {expected}")
        if self.trace_update_same_step and not naive:
            for e in self.mgr.rsb:  # this iteration's states, module order
                if self._handles[e.module].size:
                    self._emit("update", e.module, _G_CUR, e.state)
        events, self._tev = self._tev, []
        return enq, dag, rt.take_records(), events

    def _carry(self):
        """Cross-step edges replacing the per-step barrier (None: barrier);
        see scheduler.cross_step_edges."""
        prev = self._prev_enq
        if prev is None:
            return None
        edges = cross_step_edges(self._blocks, self._order[-1], self.runtime.k_slots)
        return {k: [prev.end_event(p) for p in ps] for k, ps in edges.items()}

    def force_pending(self, g: float) -> None:
        """Parity hook: replace the pending projected gradient with an
        externally supplied value (e.g. the reference's g for this step), so the
        next step's deferred update -- and finalize -- use exactly it."""
        self.pending.set(g)
        self._g_last = float(g)
        self.dev.d_out[2].fill_(float(g))
        torch.cuda.synchronize(self.runtime.device)

    def finalize(self) -> ModelParams:
        """Drain the last pending update (zo2_engine.py:318-336); idempotent."""
        if self._async:  # iterations enqueued by step_async: check them first
            self.drain()
        rt = self.runtime
        shard = getattr(rt, "shard", None)
        if shard is not None and self.pending.valid:
            # node-shared masters: every rank's last offloads must have landed
            # before any rank reads a whole block back
            import torch.distributed as dist
            torch.cuda.synchronize(rt.device)
            dist.barrier(group=shard[2])
        if self.pending.valid:
            _lib.call("zo2_set_rng_mode", RNG_MODES[self.rng])
            comp = self.lanes[Lane.COMPUTE]
            for module in self._order:
                h = self._handles[module]
                if h.size == 0:
                    continue
                lrs = self.mgr.lrs_map.get(module)
                if lrs is None:
                    raise StateCorruptionError(f"finalize: no lrs for {module}")
                if self.trace is not None and not self.trace_update_same_step:
                    self.trace({"op": "update", "module": module,
                                "coef": -(self.cfg.lr * self.pending.g),
                                "state": (lrs.seed, lrs.stream, lrs.counter)})
                descs = self._update_descs(module)
                if h.transferable and getattr(rt, "resident", False):
                    # resident blocks (MeZO): the 'host master' is the device bucket
                    self._k2(rt.masters[module], rt.wire_fmt.code, module, 1, lrs.seed, False, 0,
                             descs, comp)
                elif h.transferable:
                    slot = 0
                    with torch.cuda.stream(comp):
                        rt.slots[slot].copy_(rt.masters[module], non_blocking=True)
                    self._k2(rt.slots[slot], rt.wire_fmt.code, module, 1, lrs.seed, False, 0,
                             descs, comp)
                    with torch.cuda.stream(comp):
                        if shard is None:
                            rt.masters[module].copy_(rt.slots[slot], non_blocking=True)
                        else:
                            # write back only this rank's shard: another rank
                            # may already have updated its own shard in the
                            # shared master, so the rest of this copy may hold
                            # a twice-updated region
                            lo, hi = shard[3], shard[4]
                            rt.masters[module][lo:hi].copy_(rt.slots[slot][lo:hi],
                                                         non_blocking=True)
                    comp.synchronize()
                else:
                    self._k2(rt.persistent[module], self._fmt_of(rt.persistent[module]), module,
                             1, lrs.seed, False, 0, descs, comp)
            comp.synchronize()
            if shard is not None:
                import torch.distributed as dist
                dist.barrier(group=shard[2])  # all shards written before export
        self.pending.clear()
        self._g_last = 0.0
        self.mgr.rsb.clear()
        self._prev_enq = None
        return rt.export_params()

    def train(self, dataset, steps: int | None = None) -> list[float]:
        steps = self.cfg.steps if steps is None else steps
        for j in range(steps):
            idx = batch_for_step(self.cfg.seed, j, dataset.n_samples, dataset.batch_size)
            self.step(dataset.batch(idx), j)
        self.finalize()
        return self.losses


class MeZOEngine:
    """All-resident MeZO engine, drop-in for zo_ref.RefEngine (zo_ref.py:82-121):
    step(batch, j) -> g, .losses, .params, .train(dataset).

    The arithmetic per parameter is the reference's (+eps, -2eps, +eps, then
    -lr*g along the same z); the update is folded into the next step's fused
    K2 pass exactly as the ZO2 engine does (SPEC C1: bit-identical result) and
    is drained whenever .params is read, so the observable state after every
    step equals RefEngine's."""

    def __init__(self, workload: TransformerWorkload, cfg: ZOConfig, trace=None, *,
                 device="cuda", capacity_bytes: float = float("inf"), rng: str = "exact"):
        from .runtime import ResidentRuntime
        self.workload, self.cfg, self.trace = workload, cfg, trace
        self.runtime = ResidentRuntime(workload.params, capacity_bytes=capacity_bytes,
                                       device=device)
        k = self.runtime.k_slots
        self._engine = Zo2Engine(workload, cfg, self.runtime, overlap=k >= 3, trace=trace, rng=rng)
        # RefEngine reports each step's update at the end of that step
        self._engine.trace_update_same_step = True

    @property
    def losses(self) -> list[float]:
        return self._engine.losses

    @property
    def gs(self) -> list[float]:
        return self._engine.gs

    @property
    def timelines(self):
        return self._engine.timelines

    def step(self, batch, step_index: int) -> float:
        return self._engine.step(batch, step_index)

    @property
    def params(self) -> ModelParams:
        return self._engine.finalize()

    def train(self, dataset, steps: int | None = None) -> list[float]:
        steps = self.cfg.steps if steps is None else steps
        for j in range(steps):
            idx = batch_for_step(self.cfg.seed, j, dataset.n_samples, dataset.batch_size)
            self.step(dataset.batch(idx), j)
        return self.losses


RefEngine = MeZOEngine
