#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/sets.log
for cfg in cfg2 cfg3 cfg1; do
  for s in 2 1 2 1; do
    timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --operand-sets $s 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg sets=$s', round(d['value']), round(d['ms_per_step'],1), round(r['gemm_ms_per_step'],1), round(r['k2_ms_per_step'],1), d['step_roofline']['frac'], d['clocks']['sm_mhz'])" >> gpurun_out/sets.log
  done
done
cat gpurun_out/sets.log
