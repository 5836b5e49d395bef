#!/bin/bash
cd "$(dirname "$0")/.."
for v in 0 1 0 1; do
  timeout 300 python bench.py --config cfg1 --steps 20 --warmup 3 --no-cpu-baseline --gemm-variant $v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg1 variant $v', round(d['value']), round(d['ms_per_step'],2), round(r['gemm_ms_per_step'],2), round(r['k2_ms_per_step'],2), d['clocks'])"
done
for v in 0 1; do
  timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --gemm-variant $v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2 variant $v', round(d['value']), round(d['ms_per_step'],2), round(r['gemm_ms_per_step'],2), round(r['k2_ms_per_step'],2))"
done
