#!/bin/bash
# cfg5 diagnosis: GEMM raster/traffic at d=12288, power/clock under the GEMM alone, sets 1 vs 2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/cfg5_smi.csv & echo $! > /tmp/smi.pid )
RS_DIM=12288 RS_GMS=1,8,16 RS_REPS=6 timeout 600 python tools/raster_sweep.py > gpurun_out/cfg5_raster.log 2>&1
kill $(cat /tmp/smi.pid)
RS_DIM=12288 RS_GMS=1,8 RS_SHAPES=mlp_out,qkv RS_REPS=2 timeout 900 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none --csv \
   -k regex:k_gemm python tools/raster_sweep.py > gpurun_out/cfg5_raster_ncu.csv 2>&1
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 2 --no-cpu-baseline --operand-sets 1 > gpurun_out/r2_bench_cfg5_sets1.json 2> gpurun_out/cfg5_sets1.err
cat gpurun_out/cfg5_raster.log
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2_bench_cfg5_sets1.json').read().strip().splitlines()[-1])
print('sets1', d['value'], d['ms_per_step'], d['step_roofline']['frac'], d['roofline']['gemm_ms_per_step'], d['roofline']['k2_ms_per_step'], d['clocks'])
PY
