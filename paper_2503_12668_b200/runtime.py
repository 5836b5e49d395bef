"""Two-tier memory for the B200 offload step (replaces zo2lab runtime.py).

Host tier: one pinned (cudaHostAlloc) master per transformer block, in the
wire format: the arithmetic format (f32) or, with a codec, the low-bit
encoding (runtime.py:145-199 HostBlockStore; "the full-precision
copy exists only on the device").  Device tier: K reusable arenas in the same
wire format plus the resident embedding and LM head in f32 (runtime.py:228-247).
Upload / offload are cudaMemcpyAsync on the upload / offload streams; the
codec is applied on device inside the fused update/perturb kernel (K2), so
the wire carries exactly `wire bytes` and nothing is staged on the host.

Accounting (DevicePool, runtime.py:94-142) books every real device allocation
by category and enforces device_capacity_bytes (CapacityError).
"""
from __future__ import annotations

import hashlib
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import CapacityError, SchedulingContractError
from .model import (EMBED_ID, HEAD_ID, ModelSpec, block_id, init_module_,
                    module_size)
from .numerics import CODEC_FORMATS, ConversionSummary, ElemFormat, RngState

_TORCH_STORAGE = {ElemFormat.F64: torch.float64, ElemFormat.F32: torch.float32,
                  ElemFormat.F16: torch.int16, ElemFormat.BF16: torch.int16,
                  ElemFormat.F8E4M3: torch.uint8}


@dataclass
class TransferRecord:
    module: str
    direction: str
    bytes_wire: int
    fmt_wire: ElemFormat
    t_start: float
    t_end: float
    step: int = 0

    def to_json(self) -> dict:
        return {"module": self.module, "direction": self.direction,
                "bytes_wire": self.bytes_wire, "fmt_wire": self.fmt_wire.tag,
                "t_start": self.t_start, "t_end": self.t_end, "step": self.step}


class TransferLog:
    """Append-only transfer log (runtime.py:44-69)."""

    def __init__(self):
        self._records: list[TransferRecord] = []
        self._lock = threading.Lock()

    def append(self, rec: TransferRecord) -> None:
        with self._lock:
            self._records.append(rec)

    def records(self) -> list[TransferRecord]:
        with self._lock:
            return list(self._records)

    def counts(self) -> dict[tuple[str, str], int]:
        out: dict[tuple[str, str], int] = {}
        for r in self.records():
            out[(r.module, r.direction)] = out.get((r.module, r.direction), 0) + 1
        return out

    def wire_bytes(self, direction: str | None = None) -> int:
        return sum(r.bytes_wire for r in self.records()
                   if direction is None or r.direction == direction)


class DevicePool:
    """Byte accountant with capacity enforcement (runtime.py:94-142)."""

    def __init__(self, capacity_bytes: float = float("inf")):
        self.capacity = capacity_bytes
        self._used: dict[str, int] = {}
        self.peak_used = 0
        self._lock = threading.Lock()

    def alloc(self, category: str, nbytes: int) -> None:
        if nbytes < 0:
            raise ValueError("allocation size must be >= 0")
        with self._lock:
            used = sum(self._used.values()) + nbytes
            if used > self.capacity:
                raise CapacityError(f"alloc {nbytes} B for {category}: {used} B exceeds "
                                    f"capacity {self.capacity} B")
            self._used[category] = self._used.get(category, 0) + nbytes
            self.peak_used = max(self.peak_used, used)

    def free(self, category: str, nbytes: int) -> None:
        with self._lock:
            have = self._used.get(category, 0)
            if nbytes > have:
                raise ValueError(f"freeing {nbytes} B from {category}, only {have} B live")
            self._used[category] = have - nbytes

    @property
    def used(self) -> int:
        with self._lock:
            return sum(self._used.values())

    def breakdown(self) -> dict[str, int]:
        with self._lock:
            return dict(self._used)


class ModelParams:
    """Parameter buckets of one model: embedding and head resident on device
    (f32), blocks as pinned host f32 masters (model.py:158-181 layout)."""

    def __init__(self, spec: ModelSpec, embedding: torch.Tensor, blocks: list[torch.Tensor],
                 lm_head: torch.Tensor, fmt: ElemFormat = ElemFormat.F32):
        self.spec, self.embedding, self.blocks, self.lm_head, self.fmt = (
            spec, embedding, blocks, lm_head, fmt)
        self.block_codec: ElemFormat | None = None  # blocks already hold wire-format bits
        self.init_conversion = None
        self.shared_masters = False  # blocks are views of a node-wide SharedHostMasters

    def buckets(self) -> list[tuple[str, torch.Tensor]]:
        return ([(EMBED_ID, self.embedding)] +
                [(block_id(i), b) for i, b in enumerate(self.blocks)] + [(HEAD_ID, self.lm_head)])

    def bucket(self, module: str) -> torch.Tensor:
        if module == EMBED_ID:
            return self.embedding
        if module == HEAD_ID:
            return self.lm_head
        return self.blocks[int(module.split(".", 1)[1])]

    def total_params(self) -> int:
        return sum(b.numel() for _, b in self.buckets())

    def to_numpy(self) -> dict[str, np.ndarray]:
        return {m: b.detach().cpu().numpy().copy() for m, b in self.buckets()}

    @classmethod
    def from_numpy(cls, spec: ModelSpec, flats: dict[str, np.ndarray], device="cuda",
                   pin: bool = True) -> "ModelParams":
        """Adopt reference buckets (e.g. zo2lab init_params(...).buckets())."""
        def dev(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(device)
        n = module_size(spec, block_id(0))
        blocks = pinned_blocks(spec.n_blocks, n, torch.float32) if pin else []
        for i in range(spec.n_blocks):
            t = torch.from_numpy(np.ascontiguousarray(flats[block_id(i)], dtype=np.float32))
            if pin:
                blocks[i].copy_(t)
            else:
                blocks.append(t.clone())
        head = flats.get(HEAD_ID, np.zeros(0, np.float32))
        return cls(spec, dev(flats[EMBED_ID]), blocks, dev(head))


class _PinnedHostArena:
    """Page-locked host memory of EXACT size for the block masters: one plain
    allocation, page-locked with cudaHostRegister (zo2_host_register).
    torch's pinned allocator rounds every allocation up to a power of two, so
    a 1.23 GB OPT-30B bf16 block would take 2 GB of host RAM (96 instead of
    59 GB for the model) -- the difference between fitting and not fitting
    the masters of a large model, or of N data-parallel ranks, in host RAM.
    Same DMA rate as cudaHostAlloc (profiles/r2_link_alloc_probe.json).  Every
    block view carries a reference to the arena, so the range is unregistered
    only after the last view is gone, just before the memory is freed."""

    HUGE = 1 << 21

    def __init__(self, n_blocks: int, block_elems: int, dtype: torch.dtype):
        import mmap
        import os
        esize = torch.empty((), dtype=dtype).element_size()
        self.nbytes = n_blocks * block_elems * esize
        self.registered = False
        self._map = None
        mode = os.environ.get("ZO2_HOST_ALLOC", "hugepage")
        if mode == "torch" or self.nbytes == 0:
            # torch's pinned allocator (power-of-two rounding), for A/B only
            self.flat = torch.empty(n_blocks * block_elems, dtype=dtype,
                                    pin_memory=self.nbytes > 0)
        else:
            # anonymous mapping, 2 MB aligned, transparent huge pages where the
            # kernel grants them: fewer IOMMU / page-table entries per DMA
            self._map = mmap.mmap(-1, self.nbytes + self.HUGE,
                                  flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
            if mode == "hugepage" and hasattr(mmap, "MADV_HUGEPAGE"):
                self._map.madvise(mmap.MADV_HUGEPAGE)
            raw = torch.frombuffer(self._map, dtype=torch.uint8)
            off = (-raw.data_ptr()) % self.HUGE
            self.flat = raw[off:off + self.nbytes].view(dtype)
            _lib.call("zo2_host_register", self.flat.data_ptr(), self.nbytes)
            self.registered = True
        self.ptr = self.flat.data_ptr()
        self.blocks = []
        for i in range(n_blocks):
            b = self.flat[i * block_elems:(i + 1) * block_elems]
            b._zo2_host_arena = self  # keeps the registration alive with the view
            self.blocks.append(b)

    def __del__(self):
        if getattr(self, "registered", False):
            try:
                _lib.call("zo2_host_unregister", self.ptr)
            except Exception:  # noqa: BLE001 -- interpreter shutdown
                pass
            self.registered = False


def pinned_blocks(n_blocks: int, block_elems: int, dtype: torch.dtype) -> list:
    """n_blocks page-locked host tensors of block_elems each (one exact-size
    registered allocation, _PinnedHostArena)."""
    return _PinnedHostArena(n_blocks, block_elems, dtype).blocks


class SharedHostMasters:
    """One node-wide copy of the block masters for data-parallel ranks.

    Every rank holds bit-identical weights (same z, same all-reduced g), so a
    per-rank private master (N x the host RAM, N x the host-DRAM traffic) is
    redundant: the masters live in one POSIX shared-memory file that every
    local rank maps and page-locks (zo2_host_register).  With sharded
    transfers (OffloadRuntime.enable_sharding) rank r uploads and offloads only
    slice r of each block, and the arenas are completed over NVLink; rank r's
    slice of the master is written only by rank r, so no cross-process
    ordering on host memory is needed.  Local rank 0 creates and initialises
    the file (`owner`); SURVEY.md 8(e)."""

    def __init__(self, name: str, n_blocks: int, block_elems: int, dtype: torch.dtype,
                 owner: bool):
        import os
        self.path = f"/dev/shm/{name}"
        self.owner = owner
        esize = torch.empty((), dtype=dtype).element_size()
        total = n_blocks * block_elems
        if owner:
            with open(self.path, "wb") as f:
                f.truncate(total * esize)
        self.flat = torch.from_file(self.path, shared=True, size=total, dtype=dtype)
        self.nbytes = total * esize
        _lib.call("zo2_host_register", self.flat.data_ptr(), self.nbytes)
        self.blocks = [self.flat[i * block_elems:(i + 1) * block_elems] for i in range(n_blocks)]
        self._os = os

    def close(self) -> None:
        if self.flat is not None:
            _lib.call("zo2_host_unregister", self.flat.data_ptr())
            self.flat = None
            self.blocks = []
            if self.owner and self._os.path.exists(self.path):
                self._os.unlink(self.path)


def init_params(spec: ModelSpec, state: RngState, fmt: ElemFormat = ElemFormat.F32,
                device="cuda", pin: bool = True, codec: str | None = None,
                host_masters: "SharedHostMasters | None" = None) -> ModelParams:
    """model.py:198-224 on device: bit-identical buckets, blocks then moved to
    pinned host memory (the offload tier).

    With `codec`, each block is encoded on the device straight into its pinned
    low-bit host master (exactly HostBlockStore's encode at construction,
    runtime.py:154-162) so the f32 block copy never exists on the host --
    required for OPT-30B/175B, whose f32 masters would not fit in host RAM.

    With `host_masters` (data parallel, one copy per node) the blocks are the
    shared file's views; only its owner writes them."""
    if fmt not in (ElemFormat.F32, ElemFormat.F64):
        raise ValueError(f"parameters are f32 (arith f32 / bf16) or f64 (arith f64), "
                         f"not {fmt.tag}")
    cfmt = CODEC_FORMATS[codec] if codec not in (None, "none") else None
    if fmt is ElemFormat.F64 and (cfmt is not None or host_masters is not None):
        raise ValueError("f64 parameters take no wire codec and no shared masters "
                         "(the reference's codecs run with f32 arithmetic)")
    seed = state.seed
    dt = torch.float64 if fmt is ElemFormat.F64 else torch.float32
    emb = torch.empty(module_size(spec, EMBED_ID), dtype=dt, device=device)
    init_module_(spec, EMBED_ID, seed, emb)
    head = torch.empty(module_size(spec, HEAD_ID), dtype=dt, device=device)
    if head.numel():
        init_module_(spec, HEAD_ID, seed, head)
    blocks = []
    n = module_size(spec, block_id(0))
    scratch = torch.empty(n, dtype=dt, device=device)
    conv = torch.zeros(2, dtype=torch.int64, device=device)
    enc = torch.empty(n, dtype=_TORCH_STORAGE[cfmt], device=device) if cfmt else None
    s = torch.cuda.current_stream().cuda_stream
    pool = (pinned_blocks(spec.n_blocks, n, dt if cfmt is None else enc.dtype)
            if pin and host_masters is None else None)
    for i in range(spec.n_blocks):
        if host_masters is not None:
            host = host_masters.blocks[i]
            if not host_masters.owner:
                blocks.append(host)
                continue
        init_module_(spec, block_id(i), seed, scratch)
        if cfmt is None:
            if host_masters is None:
                host = pool[i] if pool is not None else torch.empty(n, dtype=dt)
            host.copy_(scratch)
        else:
            _lib.call("zo2_encode", scratch.data_ptr(), enc.data_ptr(), cfmt.code, n,
                      conv.data_ptr(), s)
            if host_masters is None:
                host = pool[i] if pool is not None else torch.empty(n, dtype=enc.dtype)
            host.copy_(enc.view(host.dtype))
        blocks.append(host)
    torch.cuda.synchronize()
    p = ModelParams(spec, emb, blocks, head, fmt)
    p.block_codec = cfmt
    p.init_conversion = conv
    p.shared_masters = host_masters is not None
    return p


def params_digest(params) -> str:
    """SHA-256 over canonical bucket bytes (metrics.py:20-27); equal digests
    mean identical models.  Accepts our ModelParams or {module: ndarray}."""
    h = hashlib.sha256()
    items = (params.to_numpy().items() if isinstance(params, ModelParams)
             else params.items())
    for module, flat in items:
        flat = np.asarray(flat)
        tag = "f64" if flat.dtype == np.float64 else "f32"
        h.update(module.encode())
        h.update(tag.encode())
        h.update(flat.tobytes())
    return h.hexdigest()


class HostBlockStore:
    """Master copy of one block on the host tier (runtime.py:145-199 surface).

    The bytes are the runtime's pinned master (`runtime.masters[module]`):
    the f32 block itself, or its encoded low-bit copy with a wire codec.
    Transfers move those bytes unchanged (the codec is decoded / re-encoded
    on the device inside K2), so load_into / store_from are plain copies of
    wire-format bytes; apply() edits the master in full precision."""

    def __init__(self, runtime: "OffloadRuntime", module: str):
        self._rt, self.module = runtime, module
        self.codec = runtime.codec

    @property
    def tensor(self) -> torch.Tensor:
        return self._rt.masters[self.module]

    @property
    def nbytes(self) -> int:
        t = self.tensor
        return t.numel() * t.element_size()

    @property
    def wire_fmt(self) -> ElemFormat:
        return self._rt.wire_fmt

    def load_into(self, arena: torch.Tensor) -> None:
        arena.copy_(self.tensor)

    def store_from(self, arena: torch.Tensor) -> None:
        self.tensor.copy_(arena)

    def apply(self, fn) -> None:
        """runtime.py:186-193: fn(flat) mutates the master as an f32 (or f64)
        numpy array; with a codec the master is decoded on the device, edited,
        and re-encoded (conversions counted like every other encode)."""
        rt = self._rt
        torch.cuda.synchronize(rt.device)
        if self.codec is None:
            if self.tensor.device.type == "cpu":
                fn(self.tensor.numpy())
            else:
                flat = self.tensor.cpu().numpy()
                fn(flat)
                self.tensor.copy_(torch.from_numpy(flat))
            return
        s = torch.cuda.current_stream(rt.device).cuda_stream
        enc = self.tensor.to(rt.device)
        wide = torch.empty(enc.numel(), dtype=torch.float32, device=rt.device)
        _lib.call("zo2_decode", enc.data_ptr(), wide.data_ptr(), self.codec.code, enc.numel(), s)
        flat = wide.cpu().numpy()
        fn(flat)
        wide.copy_(torch.from_numpy(flat))
        _lib.call("zo2_encode", wide.data_ptr(), enc.data_ptr(), self.codec.code, enc.numel(),
                  rt.d_conv.data_ptr(), s)
        self.tensor.copy_(enc)
        torch.cuda.synchronize(rt.device)
        nan, sat = (int(x) for x in rt.d_conv.tolist())
        rt.conversion.nan_count, rt.conversion.saturated_count = nan, sat


class OffloadRuntime:
    """Pinned host masters + K device arenas + transfer log + pool, for one run
    (runtime.py:202-304 surface)."""

    shard = None  # (rank, world, group, lo, hi) once enable_sharding() succeeded

    def __init__(self, params: ModelParams, *, k_slots: int = 3, codec: str | None = None,
                 capacity_bytes: float = float("inf"), device="cuda"):
        self.params = params
        self.spec = params.spec
        self.k_slots = int(k_slots)
        self.codec = CODEC_FORMATS[codec] if codec not in (None, "none") else None
        self.wire_fmt = self.codec or params.fmt
        self.device = torch.device(device)
        self.pool = DevicePool(capacity_bytes)
        self.log = TransferLog()
        self.conversion = ConversionSummary()
        self.current_step = 0
        self._block_ids = [block_id(i) for i in range(self.spec.n_blocks)]
        self.block_size = module_size(self.spec, block_id(0)) if self._block_ids else 0
        self.d_conv = torch.zeros(2, dtype=torch.int64, device=self.device)
        sdt = _TORCH_STORAGE[self.wire_fmt]
        # pinned host masters: alias the f32 blocks, or encode them
        self.masters: dict[str, torch.Tensor] = {}
        if params.block_codec is not None and params.block_codec is not self.codec:
            raise ValueError(f"blocks were initialised as {params.block_codec.tag}, runtime "
                             f"codec is {self.codec.tag if self.codec else 'none'}")
        if self.codec is None or params.block_codec is self.codec:
            for i, b in enumerate(self._block_ids):
                self.masters[b] = params.blocks[i]
            if params.init_conversion is not None:
                self.d_conv += params.init_conversion
        else:
            scratch = torch.empty(self.block_size, dtype=torch.float32, device=self.device)
            enc = torch.empty(self.block_size, dtype=sdt, device=self.device)
            s = torch.cuda.current_stream().cuda_stream
            pool = pinned_blocks(len(self._block_ids), self.block_size, sdt)
            for i, b in enumerate(self._block_ids):
                scratch.copy_(params.blocks[i])
                _lib.call("zo2_encode", scratch.data_ptr(), enc.data_ptr(), self.codec.code,
                          self.block_size, self.d_conv.data_ptr(), s)
                host = pool[i]
                host.copy_(enc)
                self.masters[b] = host
            del scratch, enc
            torch.cuda.synchronize()
        # the reference's per-block host stores (runtime.py:145-199) over them
        self.host = {b: HostBlockStore(self, b) for b in self._block_ids}
        # persistent residents: embedding and LM head (f32, never evicted)
        self.persistent = {EMBED_ID: params.embedding, HEAD_ID: params.lm_head}
        for t in self.persistent.values():
            self.pool.alloc("persistent_params", t.numel() * t.element_size())
        # K arenas in wire format
        self.pool.alloc("block_arenas", self.k_slots * self.block_nbytes)
        self.slots = [torch.empty(self.block_size, dtype=sdt, device=self.device)
                      for _ in range(self.k_slots)]
        self._slot_owner: list[str | None] = [None] * self.k_slots
        self._pending_records: list[tuple[TransferRecord, str]] = []

    def enable_sharding(self, rank: int, world: int, group=None) -> bool:
        """Data parallel with node-wide shared masters: rank r moves only slice r
        of every block over PCIe (H2D and D2H) and the arena is completed with
        one NVLink all-gather on the upload lane.  Per-rank
        host-link bytes drop by `world`; every rank's arena still holds the
        whole block, bit-identical across ranks.  Needs block_size % world ==
        0 (d % 8 == 0 and world | 8); returns False (replicated transfers)
        otherwise.  world == 1 is accepted (the all-gather is the identity) so
        the sharded path runs end to end on a single GPU."""
        import torch.distributed as dist
        if world < 1 or self.block_size % world != 0:
            return False
        n = self.block_size // world
        # a communicator of its own: the arena all-gathers queue behind each
        # other, never behind the compute lane's loss all-reduce
        g = dist.new_group(list(range(world))) if group is None else group
        self.shard = (rank, world, g, rank * n, (rank + 1) * n)
        # self-test of the in-place all-gather this path relies on; any
        # backend refusal falls back to replicated full-block transfers
        try:
            probe = torch.full((4 * world,), 0, dtype=torch.uint8, device=self.device)
            probe[4 * rank:4 * rank + 4] = rank + 1
            self._gather_bytes(probe, 4, g)
            torch.cuda.synchronize(self.device)
            want = torch.arange(1, world + 1, device=self.device,
                                dtype=torch.uint8).repeat_interleave(4)
            ok = bool(torch.equal(probe, want))
        except Exception:  # noqa: BLE001 -- any failure means: do not shard
            ok = False
        if not ok:
            self.shard = None
        return ok

    def _gather_bytes(self, full: torch.Tensor, chunk: int, g) -> None:
        import torch.distributed as dist
        rank, world = self.shard[0], self.shard[1]
        mine = full[rank * chunk:(rank + 1) * chunk]
        if dist.get_backend(g) == "nccl":
            dist.all_gather_into_tensor(full, mine, group=g)  # in place
        else:  # gloo (CPU tests / ranks sharing one GPU)
            parts = list(full.chunk(world))
            dist.all_gather(parts, mine.clone(), group=g)

    def _gather(self, slot: int) -> None:
        rank, world, g, lo, hi = self.shard
        esize = self.slots[slot].element_size()
        self._gather_bytes(self.slots[slot].view(torch.uint8), (hi - lo) * esize, g)

    @property
    def block_nbytes(self) -> int:
        return self.block_size * self.wire_fmt.bytes_per_elem

    @property
    def wire_nbytes(self) -> int:
        """Host-link bytes of one block transfer on this rank."""
        if self.shard is None:
            return self.block_nbytes
        return self.block_nbytes // self.shard[1]

    def slot_for(self, block_index: int) -> int:
        return block_index % self.k_slots

    def slot_bucket(self, slot: int) -> torch.Tensor:
        return self.slots[slot]

    def host_param_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.masters.values())

    # -- transfers (enqueue only; times are filled from CUDA events) --------
    def upload(self, module: str, slot: int, step: int, stream: torch.cuda.Stream,
               key: str | None = None) -> TransferRecord:
        """runtime.py:255-270.  Returns the step's TransferRecord; the copy is
        only enqueued on `stream`, so t_start / t_end are stamped with the
        device times of its CUDA events when the step's timeline is committed
        (commit_records) -- the same object, updated in place."""
        if self._slot_owner[slot] is not None:
            raise SchedulingContractError(
                f"upload of {module} into slot {slot} still owned by "
                f"{self._slot_owner[slot]} (scheduler bug)")
        with torch.cuda.stream(stream):
            if self.shard is None:
                self.slots[slot].copy_(self.masters[module], non_blocking=True)
            else:
                lo, hi = self.shard[3], self.shard[4]
                self.slots[slot][lo:hi].copy_(self.masters[module][lo:hi], non_blocking=True)
                self._gather(slot)
        self._slot_owner[slot] = module
        rec = TransferRecord(module, "upload", self.wire_nbytes, self.wire_fmt, 0.0, 0.0, step)
        self._pending_records.append((rec, key or f"U:{module}"))
        return rec

    def offload(self, module: str, slot: int, step: int, stream: torch.cuda.Stream,
                key: str | None = None) -> TransferRecord:
        """runtime.py:272-285; see upload() for the record's timestamps."""
        if self._slot_owner[slot] != module:
            raise SchedulingContractError(
                f"offload of {module} from slot {slot} owned by {self._slot_owner[slot]} "
                f"(scheduler bug)")
        with torch.cuda.stream(stream):
            if self.shard is None:
                self.masters[module].copy_(self.slots[slot], non_blocking=True)
            else:
                lo, hi = self.shard[3], self.shard[4]
                self.masters[module][lo:hi].copy_(self.slots[slot][lo:hi], non_blocking=True)
        self._slot_owner[slot] = None
        rec = TransferRecord(module, "offload", self.wire_nbytes, self.wire_fmt, 0.0, 0.0, step)
        self._pending_records.append((rec, key or f"O:{module}"))
        return rec

    def take_records(self) -> list:
        out, self._pending_records = self._pending_records, []
        return out

    def commit_records(self, timeline, records=None) -> None:
        """Stamp a step's transfer records with device times and log them."""
        ev = timeline.by_key()
        for rec, key in (self.take_records() if records is None else records):
            if key in ev:
                rec.t_start, rec.t_end = ev[key].t_start, ev[key].t_end
            self.log.append(rec)
        nan, sat = (int(x) for x in self.d_conv.tolist())
        self.conversion.nan_count, self.conversion.saturated_count = nan, sat

    def export_params(self) -> ModelParams:
        """Make the model's own buckets reflect the host masters (runtime.py:290-294)."""
        if self.codec is not None:
            scratch = torch.empty(self.block_size, dtype=torch.float32, device=self.device)
            enc = torch.empty(self.block_size, dtype=self.slots[0].dtype, device=self.device)
            s = torch.cuda.current_stream().cuda_stream
            decoded = []
            for i, b in enumerate(self._block_ids):
                enc.copy_(self.masters[b])
                _lib.call("zo2_decode", enc.data_ptr(), scratch.data_ptr(), self.codec.code,
                          self.block_size, s)
                if self.params.block_codec is None:
                    self.params.blocks[i].copy_(scratch)
                else:  # blocks alias the encoded masters: export into fresh f32 copies
                    decoded.append(scratch.cpu())
            if decoded:  # the runtime keeps its encoded masters in self.masters
                self.params.blocks = decoded
                self.params.block_codec = None
            torch.cuda.synchronize()
        return self.params

    def memory_report(self) -> dict:
        return {"device_peak_bytes": self.pool.peak_used,
                "device_used_bytes": self.pool.used,
                "host_param_bytes": self.host_param_bytes(),
                "breakdown": self.pool.breakdown(),
                "conversion": {"nan_count": self.conversion.nan_count,
                               "saturated_count": self.conversion.saturated_count},
                "torch_max_allocated": int(torch.cuda.max_memory_allocated(self.device))}


class ResidentRuntime(OffloadRuntime):
    """All blocks resident in HBM (the MeZO / no-offload configuration, zo_ref.py):
    one f32 device buffer per block serves as its permanent 'arena'; uploads and
    offloads are no-ops, so the same engine and kernels run with zero host
    traffic.  export_params() copies the device buckets back to the host view."""

    resident = True

    def __init__(self, params: ModelParams, *, capacity_bytes: float = float("inf"),
                 device="cuda"):
        self.params = params
        self.spec = params.spec
        self.codec = None
        self.wire_fmt = params.fmt
        self.device = torch.device(device)
        self.pool = DevicePool(capacity_bytes)
        self.log = TransferLog()
        self.conversion = ConversionSummary()
        self.current_step = 0
        self._block_ids = [block_id(i) for i in range(self.spec.n_blocks)]
        self.block_size = module_size(self.spec, block_id(0)) if self._block_ids else 0
        self.k_slots = max(1, len(self._block_ids))
        self.d_conv = torch.zeros(2, dtype=torch.int64, device=self.device)
        self.persistent = {EMBED_ID: params.embedding, HEAD_ID: params.lm_head}
        for t in self.persistent.values():
            self.pool.alloc("persistent_params", t.numel() * t.element_size())
        self.pool.alloc("resident_blocks", len(self._block_ids) * self.block_nbytes)
        self.slots = [b.to(self.device) for b in params.blocks]
        self.masters = {b: self.slots[i] for i, b in enumerate(self._block_ids)}
        self.host = {b: HostBlockStore(self, b) for b in self._block_ids}
        self._slot_owner = [None] * self.k_slots
        self._pending_records = []

    def upload(self, module, slot, step, stream, key=None) -> None:
        pass

    def offload(self, module, slot, step, stream, key=None) -> None:
        pass

    def export_params(self) -> ModelParams:
        torch.cuda.synchronize(self.device)
        for i, t in enumerate(self.slots):
            self.params.blocks[i].copy_(t)
        return self.params
