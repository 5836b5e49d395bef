#!/bin/bash
# host master allocation A/B on one box: torch pinned vs registered mmap (4 KB / THP)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/hostalloc.log
grep -i AnonHugePages /proc/meminfo >> gpurun_out/hostalloc.log; cat /sys/kernel/mm/transparent_hugepage/enabled >> gpurun_out/hostalloc.log 2>&1
for mode in torch register hugepage torch register hugepage; do
  ZO2_HOST_ALLOC=$mode timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); sr=d['step_roofline']; print('$mode', round(d['value']), round(d['ms_per_step'],1), 'live h2d/d2h', round(sr['h2d_gbs'],1), round(sr['d2h_gbs'],1), 'probe', round(sr['link_probe_gbs']['h2d'],1), round(sr['link_probe_gbs']['d2h'],1), 'frac', round(sr['frac'],3), 'idle', round(d.get('gpu_idle_pct',0),1))" >> gpurun_out/hostalloc.log
done
( timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_dp_sharded.py tests/test_gpu_runner.py -q -x 2>&1 | tail -2 ) >> gpurun_out/hostalloc.log
cat gpurun_out/hostalloc.log
