#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
free -g > gpurun_out/cfg5deep.log
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_36.json 2> gpurun_out/cfg5deep.err
echo "exit $?" >> gpurun_out/cfg5deep.log
free -g >> gpurun_out/cfg5deep.log
tail -3 gpurun_out/cfg5deep.err >> gpurun_out/cfg5deep.log
python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_cfg5_36.json').read().strip().splitlines()[-1]); sr=d['step_roofline']; print(d['value'], d['ms_per_step'], sr['frac'], d['full_depth_extrapolation'], d['clocks'])" >> gpurun_out/cfg5deep.log 2>&1
cat gpurun_out/cfg5deep.log
