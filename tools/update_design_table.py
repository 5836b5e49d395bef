"""Regenerate DESIGN.md's bench table from profiles/r1_bench_*.json (tools only)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = {"cfg1": "cfg1 OPT-125M MeZO f32, resident (no offload), 16×128",
         "cfg2": "cfg2 OPT-1.3B f32, f32 wire", "cfg3": "cfg3 OPT-6.7B bf16, bf16 wire",
         "cfg4": "cfg4 OPT-30B bf16, 18 GB cap",
         "cfg5": "cfg5 OPT-175B geometry, fp16 wire, 36 of 96 blocks"}


def fmt(x, nd=0):
    return f"{x:,.{nd}f}".replace(",", " ")


def main(tag="r1"):
    rows = []
    for f in ["cfg1", "cfg2", "cfg2_fast", "cfg3", "cfg3_fast", "cfg4", "cfg4_fast", "cfg5",
              "cfg5_fast"]:
        p = os.path.join(ROOT, "profiles", f"{tag}_bench_{f}.json")
        if not os.path.exists(p):
            continue
        d = json.loads(open(p).read())
        base = f.split("_")[0]
        rng = "fast" if f.endswith("fast") else "exact"
        r, sr = d["roofline"], d["step_roofline"]
        val, ms = fmt(d["value"]), fmt(d["ms_per_step"], 1)
        fe = d.get("full_depth_extrapolation")
        if fe:
            val += f" ({fe['blocks_measured']} blocks) → {fmt(fe['tokens_per_s'])} full depth"
            ms += f" → {fmt(fe['step_ms'])}"
        rows.append(f"| {NAMES[base] if rng == 'exact' else base} | {rng} | {val} | {ms} | "
                    f"{r['gemm_ms_per_step']:.1f} | {r['k2_ms_per_step']:.1f} | {r['frac']:.2f} | "
                    f"{sr['frac']:.2f} ({sr['bound']}) | {fmt(d['e2e']['value'])} |")
    ref = json.loads(open(os.path.join(ROOT, "profiles", f"{tag}_bench_reference.json")).read())
    rows.append(f"| reference CPU arm (oracle port, {ref['cpu_baseline']['cores']} host threads) "
                f"| exact | {ref['value']:.0f} | {fmt(ref['ms_per_step'])} | — | — | — | — | — |")
    p = os.path.join(ROOT, "DESIGN.md")
    s = open(p).read()
    a = s.index("| config | rng | tokens/s |")
    b = s.index("\n\n", a)
    header = ("| config | rng | tokens/s | ms/step | GEMM ms | K2 ms | GEMM roofline frac | "
              "step roofline frac | e2e tokens/s |\n|---|---|---|---|---|---|---|---|---|\n")
    open(p, "w").write(s[:a] + header + "\n".join(rows) + s[b:])
    print("\n".join(rows))


if __name__ == "__main__":
    main()
