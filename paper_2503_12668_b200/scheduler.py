"""Per-iteration task DAG over three lanes, executed on three CUDA streams.

The DAG is the reference's scheduling contract (zo2lab scheduler.py:137-216,
Alg. 3 of the paper):

  C(i) after U(i) and C(i-1)      O(i) after C(i) and O(i-1)
  U(i+1) after U(i)               U(i) after O(i-K)   (arena ring of K slots)

plus the naive-update second pass (scheduler.py:166-211) and full
serialisation for overlap=False (scheduler.py:219-236).

B200 execution (replaces the 3 Python threads of scheduler.py:403-447): each
lane is a CUDA stream; tasks are enqueued in topological order, a cross-lane
edge becomes cudaStreamWaitEvent on the predecessor's end event and same-lane
order is stream order.  Every task is bracketed by timing events, so after the
step's synchronisation the same Timeline / validate_timeline checks of the
reference run on device timestamps (no host-side waiting on the hot path).
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field
from enum import Enum
from typing import Callable, Mapping

import torch

from .errors import SchedulingContractError
from .model import EMBED_ID, HEAD_ID


class Lane(Enum):
    COMPUTE = "compute"
    UPLOAD = "upload"
    OFFLOAD = "offload"
    PREPARE = "prepare"   # B200 addition: K2 (update/perturb) beside the GEMMs


@dataclass(frozen=True)
class TaskSpec:
    key: str
    lane: Lane
    module: str
    kind: str        # "dual" | "update" | "upload" | "offload"
    bytes: int = 0
    phase: int = 1


@dataclass
class TaskDag:
    tasks: list[TaskSpec]
    edges: list[tuple[str, str]]

    def __post_init__(self):
        self.by_key = {t.key: t for t in self.tasks}
        if len(self.by_key) != len(self.tasks):
            raise ValueError("duplicate task keys in DAG")
        self._pred: dict[str, list[str]] = {t.key: [] for t in self.tasks}
        self._succ: dict[str, list[str]] = {t.key: [] for t in self.tasks}
        for a, b in self.edges:
            if a not in self.by_key or b not in self.by_key:
                raise ValueError(f"edge ({a}, {b}) references unknown task")
            self._pred[b].append(a)
            self._succ[a].append(b)

    def preds(self, key: str) -> list[str]:
        return self._pred[key]

    def succs(self, key: str) -> list[str]:
        return self._succ[key]

    def lane_tasks(self, lane: Lane) -> list[TaskSpec]:
        return [t for t in self.tasks if t.lane is lane]


@dataclass
class StreamEvent:
    lane: Lane
    key: str
    module: str
    t_start: float
    t_end: float

    @property
    def duration(self) -> float:
        return self.t_end - self.t_start


@dataclass
class Timeline:
    events: list[StreamEvent] = field(default_factory=list)

    @property
    def makespan(self) -> float:
        if not self.events:
            return 0.0
        return max(e.t_end for e in self.events) - min(e.t_start for e in self.events)

    def by_key(self) -> dict[str, StreamEvent]:
        return {e.key: e for e in self.events}

    def lane_busy(self, lane: Lane) -> float:
        return sum(e.duration for e in self.events if e.lane is lane)

    def chrome_trace_rows(self, step: int | None = None) -> list[dict]:
        """Chrome-trace rows, field names as scheduler.py:103-117."""
        tid = {Lane.COMPUTE: 0, Lane.UPLOAD: 1, Lane.OFFLOAD: 2, Lane.PREPARE: 3}
        rows = []
        for e in self.events:
            args = {"block": e.module, "t_start": e.t_start, "t_end": e.t_end}
            if step is not None:
                args["step"] = step
            rows.append({"name": e.key, "cat": e.lane.value, "ph": "X", "pid": 0,
                         "tid": tid[e.lane], "ts": e.t_start * 1e6, "dur": e.duration * 1e6,
                         "args": args})
        return rows


def ckey(m: str, phase: int = 1) -> str:
    return ("C:" if phase == 1 else "C2:") + m


def ukey(m: str, phase: int = 1) -> str:
    return ("U:" if phase == 1 else "U2:") + m


def okey(m: str, phase: int = 1) -> str:
    return ("O:" if phase == 1 else "O2:") + m


def build_iteration_dag(block_ids: list[str], *, k_slots: int = 3, overlap: bool = True,
                        naive_update: bool = False, wire_bytes: Mapping[str, int] | int = 0,
                        embed_id: str = EMBED_ID, head_id: str = HEAD_ID) -> TaskDag:
    """One iteration's DAG (same task keys and edges as scheduler.py:137-216)."""
    if k_slots < 1:
        raise ValueError("k_slots must be >= 1")
    if overlap and k_slots < 3:
        raise ValueError("overlap requires at least 3 arena slots")
    nb = (lambda m: wire_bytes) if isinstance(wire_bytes, int) else (lambda m: int(wire_bytes[m]))
    phases = (1, 2) if naive_update else (1,)
    compute, upload, offload = [], [], []
    for ph in phases:
        kind = "dual" if ph == 1 else "update"
        compute += [TaskSpec(ckey(m, ph), Lane.COMPUTE, m, kind, 0, ph)
                    for m in [embed_id, *block_ids, head_id]]
        upload += [TaskSpec(ukey(b, ph), Lane.UPLOAD, b, "upload", nb(b), ph) for b in block_ids]
        offload += [TaskSpec(okey(b, ph), Lane.OFFLOAD, b, "offload", nb(b), ph)
                    for b in block_ids]
    edges: list[tuple[str, str]] = []
    for chain in (compute, upload, offload):
        edges += [(a.key, b.key) for a, b in zip(chain, chain[1:])]
    n = len(block_ids)
    for i, b in enumerate(block_ids):
        edges.append((ukey(b), ckey(b)))
        edges.append((ckey(b), okey(b)))
        if i >= k_slots:
            edges.append((okey(block_ids[i - k_slots]), ukey(b)))
    if naive_update:
        for i, b in enumerate(block_ids):
            edges += [(okey(b), ukey(b, 2)), (ukey(b, 2), ckey(b, 2)), (ckey(b, 2), okey(b, 2))]
            last_in_slot = ((n - 1 - i) // k_slots) * k_slots + i
            if last_in_slot != i:
                edges.append((okey(block_ids[last_in_slot]), ukey(b, 2)))
            if i >= k_slots:
                edges.append((okey(block_ids[i - k_slots], 2), ukey(b, 2)))
        edges.append((ckey(head_id), ckey(embed_id, 2)))
    dag = TaskDag(compute + upload + offload, edges)
    return dag if overlap else serialize_dag(dag)


def pkey(m: str) -> str:
    return "P:" + m


def build_prepare_dag(block_ids: list[str], *, k_slots: int = 3, overlap: bool = True,
                      wire_bytes: Mapping[str, int] | int = 0, operand_sets: int = 2,
                      embed_id: str = EMBED_ID, head_id: str = HEAD_ID) -> TaskDag:
    """The B200 refinement of the iteration DAG (deferred update mode).

    The reference's compute task C(i) is split in two: P(i) on a PREPARE lane
    runs K2 (deferred update + perturb/restore, emitting W+-eps z operands) and
    C(i) on the COMPUTE lane runs the dual forward from those operands.  Every
    edge is a real data dependency:

      U(i) -> P(i)            arena holds block i
      P(i) -> C(i)            operands of block i are ready
      P(i) -> O(i)            restored (and re-encoded) weights are final, so
                              the arena drains while block i still computes
      C(i-S) -> P(i)          operand set i % S is free again (S sets)
      O(i-K) -> U(i)          arena ring of K slots (scheduler.py:196-197)
      P(head) -> C(head), C(N-1) -> C(head)

    The FP64/INT-bound P(i+1) runs concurrently with the tensor-core C(i)."""
    if k_slots < 1:
        raise ValueError("k_slots must be >= 1")
    if overlap and k_slots < 2:
        raise ValueError("overlap requires at least 2 arena slots on the prepare DAG")
    nb = (lambda m: wire_bytes) if isinstance(wire_bytes, int) else (lambda m: int(wire_bytes[m]))
    compute = ([TaskSpec(ckey(embed_id), Lane.COMPUTE, embed_id, "dual")] +
               [TaskSpec(ckey(b), Lane.COMPUTE, b, "dual") for b in block_ids] +
               [TaskSpec(ckey(head_id), Lane.COMPUTE, head_id, "dual")])
    prepare = ([TaskSpec(pkey(b), Lane.PREPARE, b, "prepare") for b in block_ids] +
               [TaskSpec(pkey(head_id), Lane.PREPARE, head_id, "prepare")])
    upload = [TaskSpec(ukey(b), Lane.UPLOAD, b, "upload", nb(b)) for b in block_ids]
    offload = [TaskSpec(okey(b), Lane.OFFLOAD, b, "offload", nb(b)) for b in block_ids]
    edges: list[tuple[str, str]] = []
    for chain in (compute, prepare, upload, offload):
        edges += [(a.key, b.key) for a, b in zip(chain, chain[1:])]
    for i, b in enumerate(block_ids):
        edges += [(ukey(b), pkey(b)), (pkey(b), ckey(b)), (pkey(b), okey(b))]
        if i >= operand_sets:
            edges.append((ckey(block_ids[i - operand_sets]), pkey(b)))
        if i >= k_slots:
            edges.append((okey(block_ids[i - k_slots]), ukey(b)))
    edges.append((pkey(head_id), ckey(head_id)))
    dag = TaskDag(compute + prepare + upload + offload, edges)
    if overlap:
        return dag
    order: list[str] = [ckey(embed_id)]
    for b in block_ids:
        order += [ukey(b), pkey(b), ckey(b), okey(b)]
    order += [pkey(head_id), ckey(head_id)]
    seen, full = set(), []
    for e in list(dag.edges) + list(zip(order, order[1:])):
        if e not in seen:
            seen.add(e)
            full.append(e)
    return TaskDag(dag.tasks, full)


def serialize_dag(dag: TaskDag) -> TaskDag:
    """Strict per-module U -> C -> O chaining (scheduler.py:219-236)."""
    order: list[str] = []
    for t in dag.lane_tasks(Lane.COMPUTE):
        for k in (ukey(t.module, t.phase), t.key, okey(t.module, t.phase)):
            if k in dag.by_key:
                order.append(k)
    seen, edges = set(), []
    for e in list(dag.edges) + list(zip(order, order[1:])):
        if e not in seen:
            seen.add(e)
            edges.append(e)
    return TaskDag(dag.tasks, edges)


def topological_order(dag: TaskDag) -> list[TaskSpec]:
    """Kahn's algorithm, ties broken by submission order (deterministic)."""
    indeg = {t.key: len(dag.preds(t.key)) for t in dag.tasks}
    rank = {t.key: i for i, t in enumerate(dag.tasks)}
    ready = [(rank[k], k) for k, d in indeg.items() if d == 0]
    heapq.heapify(ready)
    out = []
    while ready:
        _, k = heapq.heappop(ready)
        out.append(dag.by_key[k])
        for s in dag.succs(k):
            indeg[s] -= 1
            if indeg[s] == 0:
                heapq.heappush(ready, (rank[s], s))
    if len(out) != len(dag.tasks):
        raise SchedulingContractError("dependency cycle in task DAG")
    return out


@dataclass
class Violation:
    kind: str
    pred: str
    succ: str
    detail: str

    def __str__(self):
        return f"{self.kind}: {self.pred} -> {self.succ} ({self.detail})"


def validate_timeline(timeline: Timeline, dag: TaskDag, tol: float = 1e-9) -> list[Violation]:
    """Empty iff every edge and lane-FIFO constraint holds (scheduler.py:466-490)."""
    ev = timeline.by_key()
    out = [Violation("missing-event", t.key, t.key, "task produced no timeline event")
           for t in dag.tasks if t.key not in ev]
    for a, b in dag.edges:
        if a in ev and b in ev and ev[b].t_start + tol < ev[a].t_end:
            out.append(Violation("dependency", a, b,
                                 f"succ starts {ev[b].t_start:.9f} before pred ends "
                                 f"{ev[a].t_end:.9f}"))
    for lane in Lane:
        keys = [t.key for t in dag.lane_tasks(lane) if t.key in ev]
        for a, b in zip(keys, keys[1:]):
            if ev[b].t_start + tol < ev[a].t_end:
                out.append(Violation("lane-fifo", a, b, f"{lane.value} lane tasks overlap"))
    return out


# ----------------------------------------------------------------------------
# CUDA-stream executor
# ----------------------------------------------------------------------------

class CudaLanes:
    """The lanes as CUDA streams on one device (compute gets high priority so
    the tensor-core chain is never starved by the prepare lane's kernels)."""

    def __init__(self, device):
        self.device = torch.device(device)
        with torch.cuda.device(self.device):
            self.streams = {Lane.COMPUTE: torch.cuda.Stream(self.device, priority=-1),
                            Lane.UPLOAD: torch.cuda.Stream(self.device),
                            Lane.OFFLOAD: torch.cuda.Stream(self.device),
                            Lane.PREPARE: torch.cuda.Stream(self.device)}
        self._tail: list[torch.cuda.Event] = []

    def __getitem__(self, lane: Lane) -> torch.cuda.Stream:
        return self.streams[lane]

    def synchronize(self) -> None:
        for s in self.streams.values():
            s.synchronize()

    def barrier_in(self) -> None:
        """Every lane waits for the previous iteration's tail on every lane
        (a device-side step barrier: no host synchronisation)."""
        for s in self.streams.values():
            for e in self._tail:
                s.wait_event(e)

    def barrier_out(self) -> None:
        self._tail = []
        for s in self.streams.values():
            e = torch.cuda.Event()
            e.record(s)
            self._tail.append(e)


class EnqueuedStep:
    """Events of one enqueued DAG; timeline() is valid after synchronisation."""

    def __init__(self, dag: TaskDag, origin: torch.cuda.Event,
                 marks: dict[str, tuple[Lane, str, torch.cuda.Event, torch.cuda.Event]],
                 rebase: bool = False, origin_event: torch.cuda.Event | None = None):
        # origin: the timing base; origin_event: this iteration's own start
        # mark on the compute lane (the next pipelined iteration's base)
        self.dag, self.origin, self.marks, self.rebase = dag, origin, marks, rebase
        self.origin_event = origin if origin_event is None else origin_event

    def end_event(self, key: str) -> torch.cuda.Event:
        return self.marks[key][3]

    def timeline(self) -> Timeline:
        evs = []
        for key, (lane, module, s, e) in self.marks.items():
            t0 = self.origin.elapsed_time(s) * 1e-3
            t1 = self.origin.elapsed_time(e) * 1e-3
            evs.append(StreamEvent(lane, key, module, t0, t1))
        if self.rebase and evs:
            t_min = min(e.t_start for e in evs)
            evs = [StreamEvent(e.lane, e.key, e.module, e.t_start - t_min, e.t_end - t_min)
                   for e in evs]
        evs.sort(key=lambda x: (x.t_start, x.key))
        return Timeline(evs)


def cross_step_edges(block_ids: list[str], head_id: str, k_slots: int) -> dict[str, list[str]]:
    """Edges from iteration j to iteration j+1 of the prepare DAG that replace
    the per-step barrier (cross-step pipelining):
    {task of j+1: [tasks of j it waits for]}.  Next to FIFO order on each lane:

      * the arena ring: U(i, j+1), i < K, waits for the offload of the last
        block of iteration j that used slot i % K (slot_for(i) = i % K,
        runtime.py:202-304); blocks i >= K follow through U(i-K.. ) edges;
      * g_j: the first prepare task waits for C(head, j) -- K2 applies the
        deferred update with g_j and rewrites operand sets C(., j) read.

    The compute lane (the embedding updates in place with g_j, the head forms
    g) and the offload lane need nothing beyond FIFO order."""
    n = len(block_ids)
    out: dict[str, list[str]] = {}
    for i in range(min(k_slots, n)):
        last = max(m for m in range(n) if m % k_slots == i % k_slots)
        out[ukey(block_ids[i])] = [okey(block_ids[last])]
    first_p = pkey(block_ids[0]) if n else pkey(head_id)
    out[first_p] = [ckey(head_id)]
    return out


def enqueue_dag(dag: TaskDag, lanes: CudaLanes, task_fns: Mapping[str, Callable],
                after: torch.cuda.Event | None = None,
                carry: Mapping[str, list] | None = None,
                base: torch.cuda.Event | None = None) -> EnqueuedStep:
    """Enqueue every task of `dag` on its lane's stream; returns immediately.

    task_fns[key](stream) enqueues the task's work on `stream`.  `after`
    (optional) is an event every lane waits on first (previous step's tail).

    Without `carry` the iteration starts behind a device-side barrier on the
    previous iteration's tail on every lane (the reference's per-step barrier,
    zo2_engine.py:295).  With `carry` (cross-step pipelining)
    there is no barrier: carry[key] lists the previous iteration's events
    task `key` must wait for, on top of stream order.  `base` is then an event
    known to precede every task of this iteration (the previous iteration's
    origin); timelines are measured from it and shifted to start at 0."""
    if carry is None:
        lanes.barrier_in()
    if after is not None:
        for lane in Lane:
            lanes[lane].wait_event(after)
    origin = torch.cuda.Event(enable_timing=True)
    origin.record(lanes[Lane.COMPUTE])
    if carry is None:
        for lane in (Lane.UPLOAD, Lane.OFFLOAD, Lane.PREPARE):
            lanes[lane].wait_event(origin)
    marks: dict = {}
    for task in topological_order(dag):
        stream = lanes[task.lane]
        for p in dag.preds(task.key):
            plane = dag.by_key[p].lane
            if plane is not task.lane:
                stream.wait_event(marks[p][3])
        if carry is not None:
            for ev in carry.get(task.key, ()):
                stream.wait_event(ev)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        fn = task_fns.get(task.key)
        if fn is not None:
            fn(stream)
        e.record(stream)
        marks[task.key] = (task.lane, task.module, s, e)
    if carry is not None and base is not None:
        return EnqueuedStep(dag, base, marks, rebase=True, origin_event=origin)
    return EnqueuedStep(dag, origin, marks)


def close_step(lanes: CudaLanes) -> None:
    """Mark the end of an enqueued iteration on every lane (see barrier_in)."""
    lanes.barrier_out()
