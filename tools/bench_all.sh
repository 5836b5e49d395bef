#!/bin/bash
# all bench lines of a round (run under gpurun); JSON lines into gpurun_out/
R=${R:-r2}
mkdir -p gpurun_out
nproc > gpurun_out/${R}_host.txt; free -g >> gpurun_out/${R}_host.txt
timeout 900 python bench.py > gpurun_out/${R}_bench_default.json 2> gpurun_out/${R}_bench_default.err
timeout 900 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/${R}_bench_cfg2.json 2> gpurun_out/${R}_bench_cfg2.err
timeout 900 python bench.py --config cfg2 --rng fast --no-cpu-baseline > gpurun_out/${R}_bench_cfg2_fast.json 2> gpurun_out/${R}_bench_cfg2_fast.err
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_bench_cfg3.json 2> gpurun_out/${R}_bench_cfg3.err
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --rng fast > gpurun_out/${R}_bench_cfg3_fast.json 2> gpurun_out/${R}_bench_cfg3_fast.err
timeout 1200 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --rng fast > gpurun_out/${R}_bench_cfg4_fast.json 2> gpurun_out/${R}_bench_cfg4_fast.err
timeout 600 python bench.py --config cfg1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_bench_cfg1.json 2> gpurun_out/${R}_bench_cfg1.err
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/${R}_bench_cfg5.json 2> gpurun_out/${R}_bench_cfg5.err
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 2 --no-cpu-baseline --rng fast > gpurun_out/${R}_bench_cfg5_fast.json 2> gpurun_out/${R}_bench_cfg5_fast.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_bench_reference.json 2> gpurun_out/${R}_bench_reference.err
for f in gpurun_out/${R}_bench_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "FAILED", e); sys.exit(0)
r = d.get("roofline", {}); sr = d.get("step_roofline", {})
print(sys.argv[1].split("/")[-1], round(d["value"]), "tok/s", round(d.get("ms_per_step", 0), 1), "ms",
      "gemm", round(r.get("gemm_ms_per_step", 0) or 0, 1), "k2", round(r.get("k2_ms_per_step", 0) or 0, 1),
      "frac", r.get("frac"), "step_frac", sr.get("frac"), "e2e", round(d.get("e2e", {}).get("value", 0)),
      d.get("clocks", {}).get("sm_mhz"), d.get("clocks", {}).get("reasons"))
PY
done
