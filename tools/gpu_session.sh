#!/bin/bash
# One GPU session: full -m gpu suite, cfg4 + cfg3 bench lines, K2 A/B variant.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 ) > gpurun_out/gputests.log
timeout 900 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
for v in "" minb4; do for d in 7168; do if [ -n "$v" ]; then export ZO2_LIB_PATH=build/variants/$v/libzo2b200.so; fi; K2_VARIANT=0 K2_ARENA=bf16 K2_DIM=$d timeout 120 python tools/k2_ab.py; unset ZO2_LIB_PATH; done; done > gpurun_out/k2_variants.log 2>&1
cat gpurun_out/gputests.log gpurun_out/k2_variants.log
python - <<'PY'
import json
for c in ("cfg4","cfg3"):
    try:
        d=json.loads(open(f"gpurun_out/bench_{c}.json").read().strip().splitlines()[-1])
        print(c, "tok/s", round(d["value"]), "ms", round(d["ms_per_step"],1), "step_frac", round(d["step_roofline"]["frac"],3), d["step_roofline"]["bound"], "k2 ms", round(d["roofline"]["k2_ms_per_step"],1), "gemm ms", round(d["roofline"]["gemm_ms_per_step"],1), "link", round(d["step_roofline"]["t_link_ms"],1), "e2e", round(d["e2e"]["value"]), "mem", d.get("device_memory",{}).get("max_memory_reserved_bytes"))
    except Exception as e: print(c, "ERR", e)
PY
