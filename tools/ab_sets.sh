#!/bin/bash
# A/B of operand sets (tools only): K2 of block i+1 beside the forward of block i
run() { timeout 600 python bench.py --no-cpu-baseline "$@" 2>/tmp/ab.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$*\", round(d[\"value\"]), round(d[\"ms_per_step\"],1), round(d[\"roofline\"][\"gemm_ms_per_step\"],1), round(d[\"roofline\"][\"k2_ms_per_step\"],1), d[\"step_roofline\"][\"frac\"], d[\"clocks\"][\"sm_mhz\"])" || tail -3 /tmp/ab.err; }
for c in ${CONFIGS:-cfg2}; do
  for r in ${RNGS:-exact}; do
    ZO2_K2_CONCURRENT_CTAS=0 run --config $c --steps ${STEPS:-3} --warmup 2 --operand-sets 2 --rng $r
    run --config $c --steps ${STEPS:-3} --warmup 2 --operand-sets 1 --rng $r
  done
done
