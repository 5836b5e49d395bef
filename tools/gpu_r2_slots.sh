#!/bin/bash
cd "$(dirname "$0")/.."
for cfg in cfg3 cfg2; do
  for k in 3 5 3 5; do
    timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --slots $k 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; sr=d['step_roofline']; print('$cfg slots=$k', round(d['value']), round(d['ms_per_step'],1), round(sr['frac'],3), round(sr['link_gbs_used'],1), round(sr['h2d_gbs'],1), round(d.get('gpu_idle_pct',0),1))"
  done
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --slots 4 2>&1 | tail -2 | head -c 600
