#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/split.log
for cfg in cfg4 cfg3; do
for k in 1 2 1 2; do
  ZO2_UPLOAD_SPLIT=$k timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); sr=d['step_roofline']; print('$cfg split=$k', round(d['value']), round(d['ms_per_step'],1), 'live h2d/d2h', round(sr['h2d_gbs'],1), round(sr['d2h_gbs'],1), 'probe', round(sr['link_probe_gbs']['h2d'],1), round(sr['link_probe_gbs']['d2h'],1), 'frac', round(sr['frac'],3), 'idle', round(d.get('gpu_idle_pct',0),1))" >> gpurun_out/split.log
done
done
( ZO2_UPLOAD_SPLIT=2 timeout 600 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -1 ) >> gpurun_out/split.log
cat gpurun_out/split.log
