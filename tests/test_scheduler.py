"""The iteration DAG, its CUDA-stream refinement and the timeline validator
(CPU only; the stream executor itself is exercised by the gpu tests)."""
import itertools

import pytest

from paper_2503_12668_b200.errors import SchedulingContractError
from paper_2503_12668_b200.scheduler import (Lane, StreamEvent, TaskDag, TaskSpec, Timeline,
                                             build_iteration_dag, build_prepare_dag, ckey, okey,
                                             pkey, topological_order, ukey, validate_timeline)


def test_dag_identical_to_reference(golden):
    for c in golden("dags.json"):
        blocks = [f"block.{i}" for i in range(c["n"])]
        d = build_iteration_dag(blocks, k_slots=c["k"], overlap=c["overlap"],
                                naive_update=c["naive"], wire_bytes=7)
        got = [[t.key, t.lane.value, t.module, t.kind, t.bytes, t.phase] for t in d.tasks]
        assert got == c["tasks"]
        assert sorted(map(tuple, d.edges)) == sorted(map(tuple, c["edges"]))


def _simulate(dag, dur):
    """Earliest-start schedule honouring edges and lane FIFO order."""
    end, lane_free, ev = {}, {}, []
    for t in topological_order(dag):
        s = max([end[p] for p in dag.preds(t.key)] + [lane_free.get(t.lane, 0.0)])
        e = s + dur(t)
        end[t.key], lane_free[t.lane] = e, e
        ev.append(StreamEvent(t.lane, t.key, t.module, s, e))
    return Timeline(ev)


@pytest.mark.parametrize("n,k,sets", [(6, 3, 1), (6, 3, 2), (9, 4, 2), (2, 2, 1), (1, 3, 2)])
def test_prepare_dag_keeps_every_data_dependency(n, k, sets):
    blocks = [f"block.{i}" for i in range(n)]
    d = build_prepare_dag(blocks, k_slots=k, operand_sets=sets)
    edges = set(d.edges)
    for i, b in enumerate(blocks):
        assert (ukey(b), pkey(b)) in edges and (pkey(b), ckey(b)) in edges
        assert (pkey(b), okey(b)) in edges          # restored weights -> offload
        if i >= k:
            assert (okey(blocks[i - k]), ukey(b)) in edges   # arena ring
        if i >= sets:
            assert (ckey(blocks[i - sets]), pkey(b)) in edges  # operand sets
    assert (pkey("head"), ckey("head")) in edges
    tl = _simulate(d, lambda t: {"upload": 3.0, "offload": 3.0, "prepare": 1.0}.get(
        t.lane.value, 2.0))
    assert validate_timeline(tl, d) == []
    # arena slot discipline: no two blocks live in one slot at once
    ev = tl.by_key()
    for i, j in itertools.combinations(range(n), 2):
        if i % k == j % k and i < j:
            assert ev[ukey(blocks[j])].t_start >= ev[okey(blocks[i])].t_end


def test_prepare_dag_serialised_without_overlap():
    blocks = ["block.0", "block.1", "block.2"]
    d = build_prepare_dag(blocks, k_slots=1, overlap=False)
    order = [t.key for t in topological_order(d)]
    assert order == ["C:embed", "U:block.0", "P:block.0", "C:block.0", "O:block.0",
                     "U:block.1", "P:block.1", "C:block.1", "O:block.1", "U:block.2",
                     "P:block.2", "C:block.2", "O:block.2", "P:head", "C:head"]


def test_validator_flags_violations():
    d = build_iteration_dag(["block.0", "block.1"], k_slots=3)
    tl = _simulate(d, lambda t: 1.0)
    assert validate_timeline(tl, d) == []
    ev = tl.by_key()
    bad = [StreamEvent(e.lane, e.key, e.module, e.t_start, e.t_end) for e in tl.events]
    for e in bad:
        if e.key == "C:block.0":   # starts before its upload ends
            e.t_start = ev["U:block.0"].t_start
    kinds = {v.kind for v in validate_timeline(Timeline(bad), d)}
    assert "dependency" in kinds
    missing = Timeline([e for e in tl.events if e.key != "O:block.1"])
    assert any(v.kind == "missing-event" for v in validate_timeline(missing, d))


def test_cycle_detected():
    t = [TaskSpec("a", Lane.COMPUTE, "m", "dual"), TaskSpec("b", Lane.COMPUTE, "m", "dual")]
    with pytest.raises(SchedulingContractError):
        topological_order(TaskDag(t, [("a", "b"), ("b", "a")]))


def test_overlap_needs_three_slots():
    with pytest.raises(ValueError):
        build_iteration_dag(["block.0"], k_slots=2, overlap=True)


def test_chrome_trace_rows():
    d = build_prepare_dag(["block.0"], k_slots=3)
    rows = _simulate(d, lambda t: 1e-3).chrome_trace_rows(step=4)
    assert {r["tid"] for r in rows} == {0, 1, 2, 3}
    assert all(r["ph"] == "X" and r["args"]["step"] == 4 for r in rows)


@pytest.mark.parametrize("n,k,sets", [(6, 3, 1), (7, 3, 1), (9, 4, 2), (2, 3, 1), (1, 3, 1),
                                      (5, 2, 1)])
def test_cross_step_edges_keep_every_hazard(n, k, sets):
    """Two pipelined iterations (per-lane FIFO + each DAG + cross_step_edges,
    no barrier) scheduled with random durations never violate a cross-step
    hazard: a slot is re-uploaded only after its previous tenant's offload, a
    block's host master is read only after it was written back, K2 of j+1 runs
    after g_j exists and after C(., j) released the operand sets."""
    import random
    from paper_2503_12668_b200.scheduler import HEAD_ID as head
    from paper_2503_12668_b200.scheduler import cross_step_edges
    blocks = [f"block.{i}" for i in range(n)]
    d = build_prepare_dag(blocks, k_slots=k, operand_sets=sets)
    cross = cross_step_edges(blocks, head, k)

    def tag(key, j):
        return f"{key}@{j}"
    tasks, edges = [], []
    for j in (0, 1):
        tasks += [TaskSpec(tag(t.key, j), t.lane, t.module, t.kind, t.bytes, t.phase)
                  for t in d.tasks]
        edges += [(tag(a, j), tag(b, j)) for a, b in d.edges]
    edges += [(tag(p, 0), tag(c, 1)) for c, ps in cross.items() for p in ps]
    # lane FIFO across the iteration boundary: every task of j on a lane
    # precedes every task of j+1 on it (stream order)
    for lane in Lane:
        t0 = [tag(t.key, 0) for t in topological_order(d) if t.lane is lane]
        t1 = [tag(t.key, 1) for t in topological_order(d) if t.lane is lane]
        if t0 and t1:
            edges.append((t0[-1], t1[0]))
    two = TaskDag(tasks, edges)
    rnd = random.Random(n * 100 + k * 10 + sets)
    for _ in range(20):
        dur = {t.key: rnd.uniform(0.1, 3.0) for t in two.tasks}
        ev = _simulate(two, lambda t: dur[t.key]).by_key()
        for i, b in enumerate(blocks):
            # same slot: every block of j in slot i % k is offloaded before U(i, j+1)
            for m, b2 in enumerate(blocks):
                if m % k == i % k:
                    assert ev[tag(okey(b2), 0)].t_end <= ev[tag(ukey(b), 1)].t_start
            # host master of block b written back (O(b, j)) before read (U(b, j+1))
            assert ev[tag(okey(b), 0)].t_end <= ev[tag(ukey(b), 1)].t_start
            # K2(b, j+1) needs g_j and free operand sets
            assert ev[tag(ckey(head), 0)].t_end <= ev[tag(pkey(b), 1)].t_start
            for b2 in blocks:
                assert ev[tag(ckey(b2), 0)].t_end <= ev[tag(pkey(b), 1)].t_start
        assert ev[tag(ckey(head), 0)].t_end <= ev[tag(pkey(head), 1)].t_start
        # and pipelining does overlap: U(0, j+1) need not wait for C(head, j)
    if n > k:
        dur = {t.key: (5.0 if t.lane is Lane.COMPUTE else 1.0) for t in two.tasks}
        ev = _simulate(two, lambda t: dur[t.key]).by_key()
        assert ev[tag(ukey(blocks[0]), 1)].t_start < ev[tag(ckey(head), 0)].t_end


def test_operand_set_choice_follows_capacity():
    """Host logic of Zo2Engine._choose_operand_sets (CPU): two operand sets
    unless the device capacity only admits one; explicit choices are kept."""
    from types import SimpleNamespace

    from paper_2503_12668_b200.engine import Zo2Engine
    from paper_2503_12668_b200.model import DualForward, ModelSpec
    spec = ModelSpec(2, 64, 4, 96, 32)
    one = DualForward.estimate_nbytes(spec, 4, "f32", 1)
    two = DualForward.estimate_nbytes(spec, 4, "f32", 2)
    assert two > one > 0
    calls = []

    def fake(cap, auto=True, used=1000, booked=0):
        eng = SimpleNamespace(
            _sets_auto=auto, operand_sets=2, _booked={"activations": booked},
            dev=SimpleNamespace(fwd=None, operand_sets=2),
            runtime=SimpleNamespace(pool=SimpleNamespace(used=used, capacity=cap)),
            workload=SimpleNamespace(spec=spec, arith="f32"),
            _set_k2_grid=lambda: calls.append(1))
        Zo2Engine._choose_operand_sets(eng, 4)
        return eng.operand_sets, eng.dev.operand_sets
    assert fake(float("inf")) == (2, 2)
    assert fake(1000 + two) == (2, 2)
    assert fake(1000 + two - 1) == (1, 1)
    assert fake(1000 + one) == (1, 1)
    assert fake(1000 + one, auto=False) == (2, 2)
    # the current forward's own booking does not count against its rebuild
    assert fake(1000 + two, used=1000 + 500, booked=500) == (2, 2)
