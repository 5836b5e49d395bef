#!/bin/bash
cd "$(dirname "$0")/.."
( timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" 2>&1 | tail -1 )
for v in 0 2 0 2; do
  timeout 300 python bench.py --config cfg1 --steps 20 --warmup 3 --no-cpu-baseline --gemm-variant $v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg1 variant $v', round(d['value']), round(d['ms_per_step'],2), round(r['gemm_ms_per_step'],2))"
done
timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 auto', round(d['value']), round(d['ms_per_step'],2))"
