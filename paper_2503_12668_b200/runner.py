"""execute_run: one RunConfig in, one MetricsReport + artifacts out
(drop-in for zo2lab harness/runner.py:129-234 with backend = "cuda").

Artifacts per run, as the reference writes them: metrics.json,
timeline.jsonl (Chrome-trace rows from the device timelines), transfers.jsonl
and an appended summary.csv row with the reference's column order
(metrics.py:11-17).  Makespans are the device-measured step spans.
"""
from __future__ import annotations

import csv
import json
import time
from dataclasses import asdict, dataclass, field
from pathlib import Path

import numpy as np

from .config import RunConfig, build_config
from .data import gen_synthetic
from .engine import MeZOEngine, TransformerWorkload, ZOConfig, Zo2Engine, batch_for_step
from .numerics import ElemFormat, RngState
from .runtime import OffloadRuntime, init_params, params_digest

SUMMARY_COLUMNS = [
    "engine", "backend", "overlap", "update_mode", "codec", "arena_slots",
    "n_blocks", "dim", "vocab", "seq_len", "batch_size", "steps", "seed",
    "final_loss", "final_digest", "device_peak_bytes", "host_param_bytes",
    "uploads", "offloads", "wire_bytes_total",
    "tokens_per_sec_incl_warmup", "tokens_per_sec_excl_warmup", "wall_seconds",
]


@dataclass
class MetricsReport:
    """metrics.py:30-74 fields."""

    config: dict
    losses: list[float]
    final_digest: str
    device_peak_bytes: int
    host_param_bytes: int
    memory_breakdown: dict
    uploads: int
    offloads: int
    wire_bytes_up: int
    wire_bytes_down: int
    makespan_total_s: float
    makespan_mean_s: float
    tokens_per_sec_incl_warmup: float
    tokens_per_sec_excl_warmup: float
    wall_seconds: float
    extra: dict = field(default_factory=dict)

    @property
    def final_loss(self) -> float:
        return self.losses[-1] if self.losses else float("nan")

    def to_json(self) -> dict:
        return asdict(self)

    def summary_row(self) -> dict:
        c = self.config
        row = {k: c.get(k) for k in SUMMARY_COLUMNS[:13]}
        row.update({"final_loss": self.final_loss, "final_digest": self.final_digest,
                    "device_peak_bytes": self.device_peak_bytes,
                    "host_param_bytes": self.host_param_bytes,
                    "uploads": self.uploads, "offloads": self.offloads,
                    "wire_bytes_total": self.wire_bytes_up + self.wire_bytes_down,
                    "tokens_per_sec_incl_warmup": self.tokens_per_sec_incl_warmup,
                    "tokens_per_sec_excl_warmup": self.tokens_per_sec_excl_warmup,
                    "wall_seconds": self.wall_seconds})
        return row


def write_jsonl(path, rows) -> None:
    with open(path, "w") as fh:
        for r in rows:
            fh.write(json.dumps(r) + "\n")


def append_summary_row(path: Path, row: dict) -> None:
    new = not Path(path).exists()
    with open(path, "a", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=SUMMARY_COLUMNS)
        if new:
            w.writeheader()
        w.writerow(row)


def execute_run(cfg: RunConfig, write_artifacts: bool = True, device="cuda") -> MetricsReport:
    spec = cfg.model_spec()
    fmt = ElemFormat.F64 if cfg.arith == "f64" else ElemFormat.F32  # runner.py:132
    params = init_params(spec, RngState(cfg.seed), fmt, device=device)
    workload = TransformerWorkload(params, cfg.arith)
    ds = gen_synthetic(cfg.vocab, cfg.seq_len, cfg.n_samples, RngState(cfg.seed), cfg.pattern,
                       cfg.batch_size)
    zo = ZOConfig(eps=cfg.eps, lr=cfg.lr, steps=cfg.steps, seed=cfg.seed)
    tokens_per_step = cfg.batch_size * cfg.seq_len
    if cfg.engine == "mezo":
        engine = MeZOEngine(workload, zo, device=device,
                            capacity_bytes=cfg.device_capacity_bytes, rng=cfg.rng)
        runtime = engine.runtime
    else:
        runtime = OffloadRuntime(params, k_slots=cfg.arena_slots, codec=cfg.codec,
                                 capacity_bytes=cfg.device_capacity_bytes, device=device)
        engine = Zo2Engine(workload, zo, runtime, overlap=cfg.overlap,
                           update_mode=cfg.update_mode, rng=cfg.rng)
    t_run0 = time.perf_counter()
    walls = []
    for j in range(cfg.steps):
        idx = batch_for_step(cfg.seed, j, ds.n_samples, cfg.batch_size)
        t0 = time.perf_counter()
        engine.step(ds.batch(idx), j)
        walls.append(time.perf_counter() - t0)
    final = engine.params if cfg.engine == "mezo" else engine.finalize()
    wall = time.perf_counter() - t_run0
    makespans = [tl.makespan for _, tl in engine.timelines] or walls
    total = sum(makespans)
    tps_incl = cfg.steps * tokens_per_step / total if total > 0 else float("inf")
    tail = total - makespans[0]
    tps_excl = ((cfg.steps - 1) * tokens_per_step / tail
                if cfg.steps > 1 and tail > 0 else tps_incl)
    mem = runtime.memory_report()
    counts = runtime.log.counts()
    report = MetricsReport(
        config=cfg.to_flat(), losses=[float(x) for x in engine.losses],
        final_digest=params_digest(final), device_peak_bytes=int(mem["device_peak_bytes"]),
        host_param_bytes=int(mem["host_param_bytes"]),
        memory_breakdown={k: int(v) for k, v in mem["breakdown"].items()},
        uploads=sum(v for (_, d), v in counts.items() if d == "upload"),
        offloads=sum(v for (_, d), v in counts.items() if d == "offload"),
        wire_bytes_up=runtime.log.wire_bytes("upload"),
        wire_bytes_down=runtime.log.wire_bytes("offload"),
        makespan_total_s=float(total), makespan_mean_s=float(np.mean(makespans)),
        tokens_per_sec_incl_warmup=float(tps_incl), tokens_per_sec_excl_warmup=float(tps_excl),
        wall_seconds=float(wall),
        extra={"gs": [float(g) for g in engine.gs],
               "torch_max_allocated": mem.get("torch_max_allocated"),
               "conversion": mem.get("conversion")})
    if write_artifacts:
        out = cfg.resolved_output_dir()
        out.mkdir(parents=True, exist_ok=True)
        with open(out / "metrics.json", "w") as fh:
            json.dump(report.to_json(), fh, indent=2)
        rows = []
        for j, tl in engine.timelines:
            rows.extend(tl.chrome_trace_rows(j))
        write_jsonl(out / "timeline.jsonl", rows)
        write_jsonl(out / "transfers.jsonl", [r.to_json() for r in runtime.log.records()])
        append_summary_row(out / "summary.csv", report.summary_row())
    return report


def cli_run(config_file: str | None = None, overrides: dict[str, str] | None = None,
            write_artifacts: bool = True) -> MetricsReport:
    return execute_run(build_config(config_file, overrides), write_artifacts=write_artifacts)
