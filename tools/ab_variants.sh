#!/bin/bash
# A/B of built library variants on bench lines (tools only):
# VARIANTS="base build/variants/x/libzo2b200.so ..." ARGS="--config cfg3 ..." bash tools/ab_variants.sh
for v in ${VARIANTS}; do
  lib=$v; [ "$v" = base ] && lib=""
  ZO2_LIB_PATH=$lib timeout 420 python bench.py --no-cpu-baseline ${ARGS} 2>/tmp/abv.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['value']), round(d['ms_per_step'],1), round(r['gemm_ms_per_step'],1), round(r['k2_ms_per_step'],1), d['clocks']['sm_mhz'])" || tail -3 /tmp/abv.err
done
