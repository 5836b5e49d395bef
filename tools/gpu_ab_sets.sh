#!/bin/bash
# cfg4 / cfg3 step A/B: operand sets 1 vs 2, K2 CTAs per SM beside the GEMM
cd "$(dirname "$0")/.."
summ() { python - "$1" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "tok/s", round(d["value"]), "ms", round(d["ms_per_step"],1), "frac", round(d["step_roofline"]["frac"],3), "k2", round(d["roofline"]["k2_ms_per_step"],1), "gemm", round(d["roofline"]["gemm_ms_per_step"],1), "link", round(d["step_roofline"]["t_link_ms"],1), "mhz", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
}
for cfg in cfg4 cfg3; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 2 --no-cpu-baseline --operand-sets 1 > gpurun_out/ab_${cfg}_s1.json 2>/dev/null; summ gpurun_out/ab_${cfg}_s1.json
  for c in 0 2 1; do
    ZO2_K2_CONCURRENT_CTAS=$c timeout 600 python bench.py --config $cfg --steps 5 --warmup 2 --no-cpu-baseline --operand-sets 2 > gpurun_out/ab_${cfg}_s2_c$c.json 2>/dev/null; summ gpurun_out/ab_${cfg}_s2_c$c.json
  done
done
