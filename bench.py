#!/usr/bin/env python
"""ZO2 step throughput on B200 (BASELINE.json metric: "ZO step tokens/s
(1/2/4/8 B200) vs PCIe/tensor roofline; H2D GB/s; GPU idle %").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]

Workload (default cfg4 = BASELINE configs[3], the north-star target): OPT-30B
geometry (48 blocks, d 7168, 56 heads, V 50272), per-block offload under an
18 GB HBM cap, bf16 compute with the bf16 wire codec (the reference's AMP
mode), batch 16 x 512 synthetic tokens per rank, random-init weights
(init_params semantics, seed 1), the reference's exact z stream.  One "step"
= one full ZO2 iteration (dual forward of every module with the deferred
ZO-SGD update fused in, all 48 blocks uploaded and offloaded over PCIe).
Each step streams 59 GB of block weights per direction, far larger than the
126 MB L2 (no flush needed).  --config cfg2 (OPT-1.3B, f32 parameters and
wire, bf16x3 split GEMMs) and the others are the secondary lines.

value  device-timed (CUDA events, compute stream, max over ranks) with the
       batch already resident in HBM, steps enqueued asynchronously.
e2e    the public API Zo2Engine.step(batch) per step: pinned H2D of the
       batch, D2H of (l+, l-, g), synchronous (wall clock == device here).
--impl reference  the reference's CPU path (oracle port of zo2lab's step) on
       the host cores, each step a bounded sample scaled to the full step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # the reference's own CPU-runnable case: MeZO, every block resident in HBM
    "cfg1": dict(workload="OPT-125M ZO-SGD (MeZO) fp32, batch 16 x seq 128, no offload",
                 spec=(12, 768, 12, 50272, 128), B=16, arith="f32", codec="none", lr=1e-6,
                 slots=3, resident=True),
    "cfg2": dict(workload="OPT-1.3B ZO2 per-block offload fp32, batch 16 x seq 512",
                 spec=(24, 2048, 32, 50272, 512), B=16, arith="f32", codec="none", lr=1e-7,
                 slots=3),
    "cfg3": dict(workload="OPT-6.7B ZO2 AMP: bf16 compute, bf16 wire, batch 16 x seq 512",
                 spec=(32, 4096, 32, 50272, 512), B=16, arith="bf16", codec="bf16", lr=1e-7,
                 slots=3),
    "cfg3f16": dict(workload="OPT-6.7B ZO2 AMP: bf16 compute, fp16 wire, batch 16 x seq 512",
                    spec=(32, 4096, 32, 50272, 512), B=16, arith="bf16", codec="f16", lr=1e-7,
                    slots=3),
    "cfg4": dict(workload="OPT-30B ZO2 offload, bf16 compute/wire, 18 GB HBM cap, 16 x 512",
                 spec=(48, 7168, 56, 50272, 512), B=16, arith="bf16", codec="bf16", lr=1e-7,
                 slots=3, cap=18e9),
    # OPT-175B: the full 96 blocks need 348 GB of pinned fp16 masters; the GPU
    # boxes of this pool have 196 GB of host RAM, so the bench runs 36 of the 96
    # full-width blocks (130 GB of exact-size page-locked masters) and also
    # reports the full-depth step extrapolated from the measured per-block
    # time (blocks are identical work units)
    "cfg5": dict(workload="OPT-175B geometry ZO2 offload, fp16 host masters, bf16 compute, "
                          "16 x 512, 36 of 96 blocks (host RAM)",
                 spec=(36, 12288, 96, 50272, 512), B=16, arith="bf16", codec="f16", lr=1e-7,
                 slots=3, full_blocks=96),
}
EPS, SEED = 1e-3, 1

_FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(_FALLBACK_PEAKS)
    d["source"] = "fallback (B200_PROFILING.md)"
    return d


# ----------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------
# K2 is bound by instruction issue, not HBM: warp instructions per draw
# (smsp__inst_executed.sum / 2 n draws) from ncu captures of one block:
#   exact, f32 arena (the queued exact kernel with the certified update draw):
#     profiles/r2_ncu_full_k2_exact_f32_cfg2_live.txt, OPT-1.3B, n = 50 358 272
#   exact, codec arena (K2c, the AMP configurations 3-5):
#     profiles/r2_ncu_full_k2_cert_cfg4_live.txt, OPT-30B, n = 616 562 688
#   fast z: profiles/r1_ncu_full_k2_fast.txt, OPT-1.3B
# The blocks are > 97 % of the draws of a step, so the block kernel's figure
# is the one used.
K2_WARP_INST_PER_DRAW = {"exact": 659403050 / (2 * 50358272),
                         "exact_codec": 5385252546 / (2 * 616562688),
                         "fast": 440114924 / (2 * 50358272)}


def k2_issue_roofline(draws, ms, rng, clocks, dev, codec="none"):
    """K2's roofline: one warp instruction per SM sub-partition per clock at
    the SM clock measured during the run; achieved = draws per second."""
    if not ms:
        return None
    import torch
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    key = "exact_codec" if rng == "exact" and codec != "none" else rng
    ipd = K2_WARP_INST_PER_DRAW[key]
    limit = 4 * sms * mhz * 1e6 / ipd / 1e9
    got = draws / (ms * 1e-3) / 1e9
    return {"bound": "issue", "achieved": got, "peak": limit, "unit": "Gdraws/s",
            "frac": got / limit, "warp_inst_per_draw": ipd, "sm_mhz": mhz,
            "note": "peak = 4 SMSPs x SMs x SM clock / warp instructions per draw "
                    "(ncu captures named at K2_WARP_INST_PER_DRAW in bench.py); HBM is "
                    "6-8% utilised", "kernel": "K2c (certified)" if key == "exact_codec" else "K2"}


class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc = index, None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        else:
            # block until the sampler is running (its first line is taken
            # before the timed region and not counted), so short timed regions
            # still get samples
            import select
            if select.select([self.proc.stdout], [], [], 5.0)[0]:
                self.proc.stdout.readline()
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is None:
            return
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 8:
                self.rows.append(f)
        self.after = False
        if not self.rows:
            # timed region shorter than the sampling interval (cfg1): one
            # query right after it, flagged as such in the summary
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=10).stdout
                f = [x.strip() for x in out.strip().split(",")]
                if len(f) >= 8:
                    self.rows.append(f)
                    self.after = True
            except (OSError, subprocess.SubprocessError):
                pass

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[4:8]) if v == "Active"})
        d = {"sm_mhz": statistics.median(sm) if sm else None,
             "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
             "samples": 0 if getattr(self, "after", False) else len(self.rows)}
        if getattr(self, "after", False):
            d["note"] = "timed region shorter than the 100 ms sampling interval: one query right after it"
        return d


# ----------------------------------------------------------------------------
# CPU baseline: the reference's step (oracle port), bounded sample
# ----------------------------------------------------------------------------
_CPU_STATE: dict = {}
CPU_SUB_BATCH = 1


def _cpu_setup(cfg):
    """Reduced-depth reference model at FULL width (1 block, the embedding and
    the head) for the CPU arm.  Setup, not timed: random weights (values do not
    change the work), the wire codec applied once like the reference's
    construction-time encode."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    from oracle import zo2_oracle as O
    key = cfg["workload"]
    if key not in _CPU_STATE:
        nb, d, H, V, S = cfg["spec"]
        spec = O.Spec(1, d, H, V, S)
        pool = ThreadPoolExecutor(os.cpu_count() or 1)
        rng = np.random.default_rng(SEED)
        p = {}
        for m, lay in O.layouts(spec).items():
            n = sum(int(np.prod(sh)) for _, sh in lay)
            p[m] = (rng.standard_normal(n, dtype=np.float32) * np.float32(0.02))
        tok, tgt = O.gen_synthetic(V, S, 4, SEED)
        _CPU_STATE[key] = (spec, p, tok[:CPU_SUB_BATCH], tgt[:CPU_SUB_BATCH], pool)
    return _CPU_STATE[key]


def cpu_reference_step(cfg, j):
    """ONE WHOLE reference ZO2 step (oracle port of zo2lab's deferred step,
    zo2_engine.py:183-204 / :264-316) on this host: embedding, one full-width
    block, head; the deferred update and +eps/-2eps/+eps RNG passes over every
    parameter (all host threads), the wire codec round trip of the block
    (upload decode + offload encode), dual forward at batch CPU_SUB_BATCH x S,
    f64 cross-entropy.  Returns (seconds of the whole reduced step, estimate of
    the full step, breakdown): the full step is extrapolated EXPLICITLY as
    embed + head + n_blocks x block, with the forward phases scaled by
    B / CPU_SUB_BATCH (RNG and codec work do not depend on the batch)."""
    from oracle import zo2_oracle as O
    spec, p, tok, tgt, pool = _cpu_setup(cfg)
    key = ("eng", cfg["workload"])
    if key not in _CPU_STATE:
        codec = cfg["codec"] if cfg["codec"] != "none" else None
        _CPU_STATE[key] = O.Zo2Sequential(spec, p, EPS, cfg["lr"], SEED, pool=pool, codec=codec)
    eng = _CPU_STATE[key]
    eng.t = {}
    t0 = time.perf_counter()
    eng.step(tok, tgt, j)
    measured = time.perf_counter() - t0
    nb, B = cfg["spec"][0], cfg["B"]
    scale = B / CPU_SUB_BATCH
    parts = {}
    for kind in ("embed", "block", "head"):
        rng_s = eng.t.get((kind, "rng"), 0.0) + eng.t.get((kind, "codec"), 0.0)
        fwd_s = eng.t.get((kind, "fwd"), 0.0)
        parts[kind] = {"rng_codec_s": rng_s, "fwd_s": fwd_s,
                       "full_s": rng_s + fwd_s * scale}
    full = parts["embed"]["full_s"] + parts["head"]["full_s"] + nb * parts["block"]["full_s"]
    return measured, full, parts


def cpu_sample_desc(cfg):
    nb, d, H, V, S = cfg["spec"]
    return (f"oracle port of the reference ZO2 step, {os.cpu_count()} host threads: each "
            f"timed step is one WHOLE step of a reduced-depth model at full width (embedding "
            f"{V}+{S}x{d}, 1 of {nb} blocks, head {V}x{d}; deferred update + 3 perturb passes "
            f"over all parameters, block wire codec '{cfg['codec']}', dual forward at batch "
            f"{CPU_SUB_BATCH}x{S}, f64 CE); value = {cfg['B']}x{S} tokens / (embed + head + "
            f"{nb} x block), forward phases x{cfg['B'] // CPU_SUB_BATCH} for batch {cfg['B']}")


def link_probe(dev, nbytes=1 << 30, reps=3):
    """Pinned host <-> device copy rate of this box, both directions at once
    (full duplex, as in the step): best of `reps` 1 GiB copies, CUDA events on
    each copy stream.  The link term of the step roofline uses this capability,
    not the rate the step's own transfers happened to reach."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dbuf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    dbuf2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    su, so = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    best_up = best_dn = 0.0
    for _ in range(reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize(dev)
        with torch.cuda.stream(su):
            ev[0].record(su)
            dbuf.copy_(h, non_blocking=True)
            ev[1].record(su)
        with torch.cuda.stream(so):
            ev[2].record(so)
            h2.copy_(dbuf2, non_blocking=True)
            ev[3].record(so)
        torch.cuda.synchronize(dev)
        best_up = max(best_up, nbytes / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9)
        best_dn = max(best_dn, nbytes / (ev[2].elapsed_time(ev[3]) * 1e-3) / 1e9)
    del h, h2, dbuf, dbuf2
    return best_up, best_dn


def full_depth_estimate(tls, cfg, tokens_step):
    """Step time of the full-depth model from the measured timelines: the
    per-block period (compute-lane start of block i+1 minus that of block i,
    median over the timed steps) x the missing blocks, added to the measured
    step (embedding, head and the measured blocks included)."""
    from paper_2503_12668_b200.scheduler import Lane
    periods, steps = [], []
    for tl in tls:
        cs = sorted((e.t_start, e.module) for e in tl.events
                    if e.lane is Lane.COMPUTE and e.module.startswith("block."))
        periods += [b[0] - a[0] for a, b in zip(cs, cs[1:])]
        steps.append(tl.makespan if hasattr(tl, "makespan") else
                     max(e.t_end for e in tl.events) - min(e.t_start for e in tl.events))
    if not periods:
        return None
    per_block = statistics.median(periods)
    nb, full = cfg["spec"][0], cfg["full_blocks"]
    step = statistics.median(steps) + (full - nb) * per_block
    return {"blocks_measured": nb, "blocks_full": full, "per_block_ms": per_block * 1e3,
            "step_ms": step * 1e3, "tokens_per_s": tokens_step / step}


def run_reference(args, cfg, rank, world):
    """--impl reference: the reference's CPU path on this host (rank 0 only),
    whole reduced-depth steps with an explicit full-depth extrapolation."""
    if rank != 0:
        return
    S = cfg["spec"][4]
    tokens = cfg["B"] * S
    for j in range(args.warmup):
        cpu_reference_step(cfg, j)
    meas, full, parts = [], [], None
    for k in range(args.steps):
        m, f, parts = cpu_reference_step(cfg, args.warmup + k)
        meas.append(m)
        full.append(f)
    step_s = statistics.median(full)
    value = tokens / step_s
    line = {"impl": "reference", "metric": "ZO step tokens/s", "value": value,
            "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(cfg, world),
            "arm": {"impl": "oracle port of zo2lab (numpy + C restatement), CPU",
                    "compute": "f32 forward (numpy BLAS), f64 CE, reference z stream"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": os.cpu_count(),
                             "kind": "port", "sample": cpu_sample_desc(cfg)},
            "extrapolation": {"measured_reduced_step_s": meas,
                              "full_step_s": full, "per_module_last_step": parts,
                              "formula": "embed + head + n_blocks x block, forward x B/sub_batch"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(cfg, world):
    """The workload description both arms print (identical dicts)."""
    nb, d, H, V, S = cfg["spec"]
    return {"workload": cfg["workload"], "model": f"OPT geometry {nb}x{d}, {H} heads, V={V}",
            "global_batch": cfg["B"] * world, "seq_len": S,
            "parallelism": f"dp{world}" if world > 1 else "single",
            "wire": cfg["codec"] if cfg["codec"] != "none" else "f32",
            "l2": "inputs larger than L2 (GBs of weights streamed per step)"}


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
def run_ours(args, cfg, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2503_12668_b200 import _lib
    from paper_2503_12668_b200.data import gen_synthetic
    from paper_2503_12668_b200.engine import TransformerWorkload, ZOConfig, Zo2Engine
    from paper_2503_12668_b200.model import ModelSpec
    from paper_2503_12668_b200.numerics import RngState
    from paper_2503_12668_b200.runtime import OffloadRuntime, init_params
    from paper_2503_12668_b200.scheduler import Lane

    dev = torch.device("cuda", local_rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    _lib.call("zo2_set_gemm_variant", args.gemm_variant)
    nb, d, H, V, S = cfg["spec"]
    spec = ModelSpec(nb, d, H, V, S)
    B = cfg["B"]
    T = B * S
    # with a codec the blocks are encoded on device straight into pinned low-bit
    # masters (no f32 host copy: OPT-30B f32 masters alone exceed host RAM).
    # Data parallel: one node-wide shared copy of the masters (local rank 0
    # creates and fills it), each rank moving only its slice over PCIe.
    shm = None
    use_shm = world > 1 and not args.replicated_masters
    if use_shm:
        from paper_2503_12668_b200.model import block_id, module_size
        from paper_2503_12668_b200.runtime import _TORCH_STORAGE, SharedHostMasters
        from paper_2503_12668_b200.numerics import CODEC_FORMATS, ElemFormat
        sdt = _TORCH_STORAGE[CODEC_FORMATS[cfg["codec"]] if cfg["codec"] != "none"
                             else ElemFormat.F32]
        n_elem = module_size(spec, block_id(0))
        need = nb * n_elem * torch.empty((), dtype=sdt).element_size()
        name = [None, True]
        if rank == 0:
            st = os.statvfs("/dev/shm") if os.path.isdir("/dev/shm") else None
            name = [f"zo2_masters_{os.getpid()}_{int(time.time())}",
                    st is not None and st.f_bavail * st.f_frsize > need * 1.05]
            if not name[1]:
                print(f"bench: /dev/shm cannot hold {need / 1e9:.1f} GB of shared masters; "
                      f"using per-rank masters", file=sys.stderr)
        dist.broadcast_object_list(name, src=0)
        use_shm = bool(name[1])
    if use_shm:
        if rank == 0:
            shm = SharedHostMasters(name[0], nb, n_elem, sdt, owner=True)
            params = init_params(spec, RngState(SEED), device=dev, codec=cfg["codec"],
                                 host_masters=shm)
            dist.barrier()
        else:
            dist.barrier()
            shm = SharedHostMasters(name[0], nb, n_elem, sdt, owner=False)
            params = init_params(spec, RngState(SEED), device=dev, codec=cfg["codec"],
                                 host_masters=shm)
    else:
        params = init_params(spec, RngState(SEED), device=dev, codec=cfg["codec"])
    def make_engine(params):
        if cfg.get("resident"):  # MeZO: blocks live in HBM, transfers are no-ops
            from paper_2503_12668_b200.runtime import ResidentRuntime
            rt = ResidentRuntime(params, device=dev)
        else:
            rt = OffloadRuntime(params, k_slots=args.slots or cfg["slots"], codec=cfg["codec"],
                                capacity_bytes=cfg.get("cap", float("inf")), device=dev)
        eng = Zo2Engine(TransformerWorkload(params, cfg["arith"]),
                        ZOConfig(EPS, cfg["lr"], max(1, args.steps), SEED), rt, validate=True,
                        operand_sets=args.operand_sets, rng=args.rng,
                        pipeline_steps=not args.no_pipeline)
        return rt, eng

    rt, eng = make_engine(params)
    sharded = False
    if world > 1:
        from paper_2503_12668_b200.errors import UsageError
        try:
            sharded = eng.enable_data_parallel(shard_transfers=shm is not None)
        except UsageError as e:  # shared masters but no sharded transfers
            print(f"bench: {e}; using per-rank masters", file=sys.stderr)
            del eng, rt, params
            dist.barrier()
            shm.close()
            shm = None
            params = init_params(spec, RngState(SEED), device=dev, codec=cfg["codec"])
            rt, eng = make_engine(params)
            sharded = eng.enable_data_parallel(shard_transfers=False)
    ds = gen_synthetic(V, S, 64 * world, RngState(SEED), "affine", B)
    from paper_2503_12668_b200.parallel import shard_indices

    def batch(j):
        return ds.batch(shard_indices(SEED, j, ds.n_samples, B, rank, world))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    j = 0
    for _ in range(args.warmup):
        eng.step(batch(j), j)
        j += 1
    torch.cuda.synchronize()

    # ---- value: device-timed, batch resident, async enqueue ----------------
    lib = _lib.load()
    comp = eng.lanes[Lane.COMPUTE]
    eng.dev.fwd.prof = []
    n_tl0 = len(eng.timelines)
    barrier()
    torch.cuda.synchronize()
    l0 = lib.zo2_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev.index) as clk:
        e0.record(comp)
        for k in range(args.steps):
            if len(eng._async) == eng._hist.shape[0]:
                eng.drain()  # more iterations than the result ring holds
            eng.step_async(j + k)
        # the timed region ends when every lane is done (the last offload
        # may trail the compute lane), not just the compute stream
        for st in eng.lanes.streams.values():
            if st is not comp:
                ev = torch.cuda.Event()
                ev.record(st)
                comp.wait_event(ev)
        e1.record(comp)
        eng.drain()
        torch.cuda.synchronize()
    launches = lib.zo2_launch_count() - l0
    barrier()
    j += args.steps
    dev_ms = e0.elapsed_time(e1)
    tls = [tl for _, tl in eng.timelines[n_tl0:]]
    ms = max_over_ranks(dev_ms)
    prof = eng.dev.fwd.prof
    eng.dev.fwd.prof = None
    gemm = [(w, a.elapsed_time(b)) for kind, w, a, b in prof if kind == "gemm"]
    k2 = [(w, a.elapsed_time(b)) for kind, w, a, b in prof if kind == "k2"]
    gemm_flops = sum(w for w, _ in gemm)
    gemm_ms = sum(t for _, t in gemm)
    k2_ms = sum(t for _, t in k2)
    k2_draws = sum(w for w, _ in k2)

    # per-step timeline metrics: H2D GB/s from upload events, GPU idle %
    up = [e for tl in tls for e in tl.events if e.lane is Lane.UPLOAD]
    off = [e for tl in tls for e in tl.events if e.lane is Lane.OFFLOAD]
    # host-link bytes this rank moved per block transfer (1/world of the block
    # with sharded transfers; the upload event also covers the NVLink all-gather)
    h2d_gbs = (sum(rt.wire_nbytes for _ in up) / sum(e.duration for e in up) / 1e9) if up else None
    d2h_gbs = (sum(rt.wire_nbytes for _ in off) / sum(e.duration for e in off) / 1e9) if off else None
    if cfg.get("resident"):
        h2d_gbs = d2h_gbs = None  # no weight traffic
    comp_busy = sum(tl.lane_busy(Lane.COMPUTE) for tl in tls)
    idle_pct = max(0.0, 100.0 * (1.0 - comp_busy / (dev_ms * 1e-3))) if tls else None

    # ---- e2e: public API per step (host batch in, (l+, l-, g) out) ---------
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(args.steps):
        eng.step(batch(j + k), j + k)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    barrier()

    pk = peaks()
    tokens_step = T * world
    value = tokens_step * args.steps / (ms * 1e-3)
    e2e_value = tokens_step * args.steps / e2e_s
    wire_per_dir = 0 if cfg.get("resident") else nb * rt.wire_nbytes
    # step roofline: slower of offloaded bytes at the measured
    # host link and algorithmic GEMM FLOPs at the bf16 tensor peak
    flops_step = 2 * (nb * (24.0 * T * d * d + 4.0 * B * S * S * d) + 2.0 * T * d * V)
    probe_up, probe_dn = link_probe(dev)
    # full duplex: the slower direction binds; the link capability is the better
    # of the probe and what the step's own block copies reached
    link_gbs = max(min(probe_up, probe_dn), min(h2d_gbs or 0.0, d2h_gbs or 0.0))
    t_link = wire_per_dir / (link_gbs * 1e9) if link_gbs else 0.0
    split = cfg["arith"] == "f32"
    # f32-faithful GEMMs run 3 bf16 tensor passes per algorithmic FLOP
    # (hi*hi + hi*lo + lo*hi): their peak is the bf16 dense peak / 3
    passes = 3 if split else 1
    t_tensor = passes * flops_step / (pk["bf16_tflops_sustained"] * 1e12)
    t_roof = max(t_link or 0.0, t_tensor)
    step_s = ms * 1e-3 / args.steps
    gemm_tflops = gemm_flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms else None
    phys = (gemm_tflops or 0.0) * passes
    if phys <= pk["bf16_tflops_sustained"]:
        peak_bf16, peak_src = pk["bf16_tflops_sustained"], pk["source"] + ", sustained"
    else:  # the step's GEMMs beat the 4 s cuBLAS sustained figure: burst binds
        peak_bf16, peak_src = pk["bf16_tflops"], pk["source"] + ", burst (sustained exceeded)"
    traffic, traffic_note = None, None
    tp = os.path.join(ROOT, "profiles", "r2_gemm_traffic.json")
    if os.path.exists(tp):
        tr = json.load(open(tp)).get(args.config)
        if tr:
            traffic = tr["dram_bytes"]
            traffic_note = (f"DRAM bytes of one {tr['kernel']} launch (ncu, {tr['source']}); "
                            f"algorithmic {tr['algorithmic_bytes'] / 1e9:.2f} GB "
                            f"({tr['ratio']:.1f}x)")
    line = {
        "metric": "ZO step tokens/s", "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16x3" if split else "bf16", "data": "synthetic",
        "config": config_dict(cfg, world),
        "arm": {"parallelism_detail": ("shared host masters, sharded PCIe + NVLink all-gather"
                                       if sharded else ("replicated host masters"
                                                        if world > 1 else None)),
                "compute": ("f32 parameters / update / LN / CE; GEMMs as bf16x3 splits "
                            "(hi*hi + hi*lo + lo*hi, ~16-bit operand mantissas, f32 "
                            "accumulate)" if split else
                            "bf16 compute (bf16 GEMM operands, f32 accumulate; f32 "
                            "parameters / update / LN / softmax / residual, CE in f64), "
                            f"{cfg['codec']} wire"),
                "rng": args.rng + (" (reference z stream, bit-exact)" if args.rng == "exact"
                                   else " (Philox4x32 + binary32 erfinv, not the reference's z)"),
                "steps_pipelined": not args.no_pipeline,
                "operand_sets": eng.operand_sets},
        "roofline": {"bound": "tensor", "kernel": "zo2_gemm (tcgen05 cta_group::2, fused epilogues)",
                     "achieved": gemm_tflops, "peak": peak_bf16 / passes,
                     "unit": "TFLOP/s", "frac": (gemm_tflops * passes / peak_bf16
                                                 if gemm_tflops else None),
                     "traffic": traffic,
                     "traffic_note": traffic_note,
                     "peak_source": peak_src + (f", / {passes} tensor passes" if passes > 1 else ""),
                     "algorithmic": "2*M*N*K per GEMM, summed over the step's GEMM launches "
                                    "(CUDA events on the compute stream)",
                     "tensor_passes": passes,
                     "co_running": ("operand_sets=2: K2 of block i+1 shares the SMs with the "
                                    "forward of block i, so GEMM and K2 launch durations "
                                    "include that sharing" if eng.operand_sets >= 2 else None),
                     "gemm_ms_per_step": gemm_ms / args.steps,
                     "k2_ms_per_step": k2_ms / args.steps,
                     "k2_gdraws_per_s": (k2_draws / (k2_ms * 1e-3) / 1e9) if k2_ms else None,
                     "k2": k2_issue_roofline(k2_draws, k2_ms, args.rng, clk.summary(), dev,
                                            cfg["codec"])},
        "step_roofline": {"bound": "pcie" if (t_link or 0) >= t_tensor else "tensor",
                          "link_probe_gbs": {"h2d": probe_up, "d2h": probe_dn,
                                             "note": "1 GiB pinned copies, both directions "
                                                     "at once, best of 3"},
                          "h2d_gbs": h2d_gbs, "d2h_gbs": d2h_gbs, "link_gbs_used": link_gbs,
                          "bytes_per_dir": wire_per_dir, "t_link_ms": (t_link or 0) * 1e3,
                          "t_tensor_ms": t_tensor * 1e3, "frac": t_roof / step_s,
                          "tensor_note": "algorithmic dual-forward FLOPs (scheduler.py:288-295 "
                                         "formula) x tensor passes / sustained bf16 peak"},
        "gpu_idle_pct": idle_pct,
        "e2e": {"value": e2e_value, "unit": "tokens/s",
                "h2d_bytes_per_step": 2 * T * 8 + wire_per_dir,
                "d2h_bytes_per_step": 4 * 8 + wire_per_dir,
                "note": "h2d/d2h include the per-step block weight traffic of the offload"},
        "gpu_launches": int(launches),
        "device_memory": {"max_memory_allocated_bytes": int(torch.cuda.max_memory_allocated(dev)),
                          "max_memory_reserved_bytes": int(torch.cuda.max_memory_reserved(dev)),
                          "cap_bytes": cfg.get("cap"),
                          "pool_peak_bytes": int(rt.pool.peak_used),
                          "under_cap": (torch.cuda.max_memory_reserved(dev) <= cfg["cap"]
                                        if cfg.get("cap") else None),
                          "note": "torch caching-allocator peaks over the whole run (all "
                                  "device tensors: arenas, operands, activations, masters of "
                                  "the resident modules)"},
        "clocks": clk.summary(),
        **({"full_depth_extrapolation": full_depth_estimate(tls, cfg, T * world)}
           if cfg.get("full_blocks") else {}),
        "losses_tail": eng.losses[-2:],
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_reference_step(cfg, 0)  # first call: setup + numpy/BLAS warm-up
        meas, full, _ = cpu_reference_step(cfg, 1)
        line["cpu_baseline"] = {"value": T / full, "unit": "tokens/s", "cores": os.cpu_count(),
                                "kind": "port", "sample": cpu_sample_desc(cfg),
                                "measured_reduced_step_s": meas, "full_step_s": full}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if shm is not None:
        torch.cuda.synchronize()
        dist.barrier()
        shm.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--operand-sets", type=int, default=None,
                    help="1: K2 of block i+1 after the forward of block i; 2: beside it "
                         "(default: 2 when the device capacity admits two sets)")
    ap.add_argument("--replicated-masters", action="store_true",
                    help="data parallel: private host masters per rank and full-block "
                         "transfers (default: one shared copy, sharded transfers)")
    ap.add_argument("--rng", default="exact", choices=["exact", "fast"],
                    help="z generator: the reference's stream (default) or the fast GPU one")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="per-step device barrier instead of cross-step pipelining")
    ap.add_argument("--slots", type=int, default=0,
                    help="device arena slots K (default: the configuration's, 3)")
    ap.add_argument("--gemm-variant", type=int, default=0,
                    help="0 auto (CTA pair for large shapes), 1 single-CTA, 2 pair")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # NCCL over NVLink on a real multi-GPU node; ZO2_DIST_BACKEND=gloo lets
        # several ranks share one GPU for functional tests of the DP path
        backend = os.environ.get("ZO2_DIST_BACKEND", "nccl")
        dev = torch.device("cuda", local_rank % torch.cuda.device_count())
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
