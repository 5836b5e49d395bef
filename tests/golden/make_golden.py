"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (the reference is importable only here):
    python tests/golden/make_golden.py [--big]
It imports zo2lab from /root/reference/pkg/src (read-only) and writes small
.json/.npz fixtures that travel with the repo; nothing at test time reads
/root/reference.  --big also computes the config-1-shape KAT (OPT-125M
geometry, ~1 min) and the reduced-depth config-2 KAT (~3 min).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF)

from zo2lab import numerics as N  # noqa: E402
from zo2lab.harness.data import gen_synthetic  # noqa: E402
from zo2lab.harness.metrics import params_digest  # noqa: E402
from zo2lab.model import ModelSpec, TransformerWorkload, init_params  # noqa: E402
from zo2lab.runtime import OffloadRuntime  # noqa: E402
from zo2lab.zo2_engine import Zo2Engine  # noqa: E402
from zo2lab.zo_ref import RefEngine, ZOConfig, batch_for_step  # noqa: E402


def rng_fixtures():
    cases = [(7, 0, 0, 9), (123, 5, 3, 6), (2**63 + 5, 1, 2**40 + 1, 7),
             (N.derive_step_seed(1234, 0), 0, 0, 5), (1, 2, 4 * 10**9 + 3, 5),
             (2**64 - 1, 2**64 - 1, 2**64 - 9, 12)]
    raw = []
    for s, st, c, n in cases:
        r, _ = N.raw_uint64(N.RngState(s, st, c), n)
        raw.append({"seed": s, "stream": st, "counter": c, "n": n,
                    "out": [int(x) for x in r]})
    gauss = []
    gcases = cases[:5] + [(20240601, 0, 10**6 + 1, 33), (1, 0, 162_370_560 - 8, 16)]
    for s, st, c, n in gcases:
        z, _ = N.gaussian_fill(N.RngState(s, st, c), n)
        gauss.append({"seed": s, "stream": st, "counter": c, "n": n,
                      "bits": [int(x) for x in z.view(np.uint64)]})
    seeds = [{"base": b, "j": j, "out": N.derive_step_seed(b, j)}
             for b, j in [(1234, 0), (1, 0), (1, 1), (20240601, 99), (2**64 - 1, 2**40)]]
    # a larger bulk sample, stored as a checksum of the f64 bit patterns
    z, _ = N.gaussian_fill(N.RngState(99, 0, 12345), 1_000_000)
    bulk = {"seed": 99, "stream": 0, "counter": 12345, "n": 1_000_000,
            "sum_bits_mod64": int(np.sum(z.view(np.uint64), dtype=np.uint64)),
            "first": float(z[0]), "last": float(z[-1])}
    (OUT / "rng.json").write_text(json.dumps({"raw": raw, "gauss": gauss, "seeds": seeds,
                                              "bulk": bulk}, indent=1))


def codec_fixtures():
    rng = np.random.default_rng(7)
    special = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, -np.nan,
                        3.4028235e38, -3.4028235e38, 65504.0, 65520.0, 65519.99, 1e5, -1e5,
                        448.0, 464.0, 480.0, 500.0, -449.0, 2.0**-9, 2.0**-10, 2.0**-7,
                        1.5 * 2**-7, 2.0**-14, 2.0**-24, 2.0**-25, 1.0000001, 1.00390625,
                        1.01171875, 3.0e-39, -3.0e-39, 0.0625, 0.09375, 17.0, 18.0, 19.0,
                        2.75, 3.25, -3.75], dtype=np.float32)
    rand = np.concatenate([rng.standard_normal(4000).astype(np.float32) * s
                           for s in (1e-6, 1e-3, 0.05, 1.0, 30.0, 300.0, 1e4, 1e6)])
    x = np.concatenate([special, rand]).astype(np.float32)
    out = {"x": x}
    for tag, fmt in (("bf16", N.ElemFormat.BF16), ("f16", N.ElemFormat.F16),
                     ("f8", N.ElemFormat.F8E4M3)):
        summ = N.ConversionSummary()
        enc = N.encode(N.TensorBuf.from_array(x), fmt, summ)
        dec = N.decode(enc, N.ElemFormat.F32)
        bits = enc.data if tag != "f16" else enc.data.view(np.uint16)
        out[f"{tag}_bits"] = bits
        out[f"{tag}_dec"] = dec.data
        out[f"{tag}_counts"] = np.array([summ.nan_count, summ.saturated_count])
    codes = np.arange(256, dtype=np.uint8)
    out["e4m3_table"] = N.decode(N.TensorBuf(codes, (256,), N.ElemFormat.F8E4M3),
                                 N.ElemFormat.F64).data
    np.savez_compressed(OUT / "codecs.npz", **out)


def flat_params(params):
    return {m: b.flat.copy() for m, b in params.buckets()}


def toy_fixtures():
    """Acceptance toy (test_acceptance.py:41-46) in f32: per-step l+/l-/g of
    MeZO, the initial and final buckets, and ZO2 (threaded, deferred) digest."""
    spec = ModelSpec(4, 32, 4, 64, 16)
    seed, T = 20240601, 10
    cfg = ZOConfig(eps=1e-3, lr=1e-3, steps=T, seed=seed)
    ds = gen_synthetic(64, 16, 64, N.RngState(seed), "affine", 2)
    out = {"spec": [4, 32, 4, 64, 16], "seed": seed, "steps": T, "eps": 1e-3, "lr": 1e-3,
           "batch_size": 2, "n_samples": 64}
    res = {}
    for tag, fmt, codec in (("f32", N.ElemFormat.F32, None), ("bf16codec", N.ElemFormat.F32, "bf16"),
                            ("f16codec", N.ElemFormat.F32, "f16"), ("f8codec", N.ElemFormat.F32, "f8")):
        params = init_params(spec, N.RngState(seed), fmt)
        init_flat = flat_params(params)
        if codec is None:
            ref = RefEngine(TransformerWorkload(params), cfg)
            lm = []
            orig = ref.workload.evaluate
            calls = []

            def ev(batch, _o=orig, _c=calls):
                v = _o(batch)
                _c.append(v)
                return v
            ref.workload.evaluate = ev
            batches = []
            for j in range(T):
                idx = batch_for_step(seed, j, ds.n_samples, 2)
                batches.append(idx)
                ref.step(ds.batch(idx), j)
            lp = calls[0::2]
            lm = calls[1::2]
            gs = [(a - b) / (2 * 1e-3) for a, b in zip(lp, lm)]
            res[tag] = {"l_plus": lp, "l_minus": lm, "g": gs,
                        "digest": params_digest(params), "batches": [b.tolist() for b in batches]}
            np.savez_compressed(OUT / f"toy_{tag}.npz",
                                **{f"init::{m}": v for m, v in init_flat.items()},
                                **{f"final::{m}": v for m, v in flat_params(params).items()})
        else:
            rt = OffloadRuntime(params, k_slots=3, codec=codec)
            eng = Zo2Engine(TransformerWorkload(params), cfg, rt)
            for j in range(T):
                idx = batch_for_step(seed, j, ds.n_samples, 2)
                eng.step(ds.batch(idx), j)
            final = eng.finalize()
            res[tag] = {"losses": eng.losses, "g": eng.gs, "digest": params_digest(final),
                        "wire_up": rt.log.wire_bytes("upload"),
                        "conversion": [rt.conversion.nan_count, rt.conversion.saturated_count]}
            np.savez_compressed(OUT / f"toy_{tag}.npz",
                                **{f"final::{m}": v for m, v in flat_params(final).items()})
    out["runs"] = res
    (OUT / "toy.json").write_text(json.dumps(out, indent=1))


def big_fixtures():
    """Step-0 KATs at full width: config-1 shape and config-2 reduced depth."""
    out = {}
    for tag, spec, B, lr in (("cfg1", ModelSpec(12, 768, 12, 50272, 128), 16, 1e-6),
                             ("cfg2_2blk", ModelSpec(2, 2048, 32, 50272, 512), 16, 1e-7)):
        params = init_params(spec, N.RngState(1), N.ElemFormat.F32)
        ds = gen_synthetic(spec.vocab, spec.seq_len, 64, N.RngState(1), "affine", B)
        idx = np.arange(B)
        eng = RefEngine(TransformerWorkload(params), ZOConfig(1e-3, lr, 1, 1))
        calls = []
        orig = eng.workload.evaluate

        def ev(batch, _o=orig, _c=calls):
            v = _o(batch)
            _c.append(v)
            return v
        eng.workload.evaluate = ev
        g = eng.step(ds.batch(idx), 0)
        out[tag] = {"spec": [spec.n_blocks, spec.dim, spec.n_heads, spec.vocab, spec.seq_len],
                    "batch_size": B, "lr": lr, "eps": 1e-3, "seed": 1, "batch_idx": idx.tolist(),
                    "l_plus": calls[0], "l_minus": calls[1], "g": g,
                    "digest_after": params_digest(params)}
        print(tag, out[tag]["l_plus"], out[tag]["l_minus"], g, flush=True)
    (OUT / "big.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    rng_fixtures()
    codec_fixtures()
    toy_fixtures()
    if "--big" in sys.argv:
        big_fixtures()
    print("fixtures written to", OUT)


def dag_fixtures():
    """Task lists and edges of the reference's iteration DAG for several
    (n_blocks, k, overlap, naive) settings (scheduler.py:137-236)."""
    from zo2lab.scheduler import build_iteration_dag
    out = []
    for n, k, ov, nv in [(5, 3, True, False), (7, 4, True, False), (4, 1, False, False),
                         (6, 3, True, True), (3, 2, False, True), (1, 3, True, False)]:
        blocks = [f"block.{i}" for i in range(n)]
        d = build_iteration_dag(blocks, k_slots=k, overlap=ov, naive_update=nv, wire_bytes=7)
        out.append({"n": n, "k": k, "overlap": ov, "naive": nv,
                    "tasks": [[t.key, t.lane.value, t.module, t.kind, t.bytes, t.phase]
                              for t in d.tasks],
                    "edges": [list(e) for e in d.edges]})
    (OUT / "dags.json").write_text(json.dumps(out))


def tied_fixtures():
    """Tied LM head (model.py:145-148, :367-369): 6-step MeZO f32 run."""
    spec = ModelSpec(2, 32, 4, 64, 16, tie_lm_head=True)
    seed, T = 777, 6
    cfg = ZOConfig(eps=1e-3, lr=1e-3, steps=T, seed=seed)
    ds = gen_synthetic(64, 16, 32, N.RngState(seed), "affine", 2)
    params = init_params(spec, N.RngState(seed), N.ElemFormat.F32)
    ref = RefEngine(TransformerWorkload(params), cfg)
    calls = []
    orig = ref.workload.evaluate

    def ev(batch, _o=orig, _c=calls):
        v = _o(batch)
        _c.append(v)
        return v
    ref.workload.evaluate = ev
    for j in range(T):
        ref.step(ds.batch(batch_for_step(seed, j, ds.n_samples, 2)), j)
    lp, lm = calls[0::2], calls[1::2]
    (OUT / "tied.json").write_text(json.dumps(
        {"spec": [2, 32, 4, 64, 16], "seed": seed, "steps": T, "n_samples": 32,
         "batch_size": 2, "eps": 1e-3, "lr": 1e-3, "l_plus": lp, "l_minus": lm,
         "g": [(a - b) / 2e-3 for a, b in zip(lp, lm)], "digest": params_digest(params)}))
    np.savez_compressed(OUT / "tied_final.npz", **{m: v for m, v in flat_params(params).items()})


if __name__ == "__main__" and "--dags" in sys.argv:
    dag_fixtures()
if __name__ == "__main__" and "--tied" in sys.argv:
    tied_fixtures()
