"""Dump the device timelines of a few cfg bench steps as Chrome-trace JSON
(tools only): python tools/timeline_dump.py [cfg2] > gpurun_out/trace.json"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402


def main(name="cfg2", steps=3):
    import torch
    from paper_2503_12668_b200.data import gen_synthetic
    from paper_2503_12668_b200.engine import TransformerWorkload, ZOConfig, Zo2Engine
    from paper_2503_12668_b200.model import ModelSpec
    from paper_2503_12668_b200.numerics import RngState
    from paper_2503_12668_b200.parallel import shard_indices
    from paper_2503_12668_b200.runtime import OffloadRuntime, init_params
    cfg = bench.CONFIGS[name]
    nb, d, H, V, S = cfg["spec"]
    spec = ModelSpec(nb, d, H, V, S)
    dev = torch.device("cuda", 0)
    params = init_params(spec, RngState(1), device=dev, codec=cfg["codec"])
    rt = OffloadRuntime(params, k_slots=cfg["slots"], codec=cfg["codec"],
                        capacity_bytes=cfg.get("cap", float("inf")), device=dev)
    eng = Zo2Engine(TransformerWorkload(params, cfg["arith"]), ZOConfig(1e-3, cfg["lr"], steps, 1), rt)
    ds = gen_synthetic(V, S, 64, RngState(1), "affine", cfg["B"])
    eng.step(ds.batch(shard_indices(1, 0, 64, cfg["B"], 0, 1)), 0)
    for j in range(1, steps + 1):
        eng.step_async(j)
    eng.drain()
    rows = []
    for j, tl in eng.timelines[1:]:
        rows += tl.chrome_trace_rows(j)
    json.dump({"traceEvents": rows}, sys.stdout)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["cfg2"]))
