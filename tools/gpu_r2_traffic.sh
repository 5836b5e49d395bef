#!/bin/bash
# mlp_out DRAM traffic of the final build at cfg2 (split) and cfg5 shapes; group-height sweep with the dynamic scheduler
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
PK_DIM=2048 timeout 600 $NCU -k regex:k_gemm --launch-skip 3 --launch-count 1 -o gpurun_out/r2f_gemm_mlpout_cfg2 python tools/profile_kernels.py fwd f32 > /dev/null 2>&1
PK_DIM=12288 timeout 600 $NCU -k regex:k_gemm --launch-skip 3 --launch-count 1 -o gpurun_out/r2f_gemm_mlpout_cfg5 python tools/profile_kernels.py fwd bf16 > /dev/null 2>&1
for d in 7168 12288; do
  RS_DIM=$d RS_GMS=4,8,16,32 RS_SHAPES=mlp_out,qkv RS_REPS=2 timeout 900 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none --csv \
      -k regex:k_gemm python tools/raster_sweep.py > gpurun_out/gm_ncu_$d.csv 2>&1
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench_check.json 2> gpurun_out/r2f_bench_check.err
python -c "
import json; d=json.loads(open('gpurun_out/r2f_bench_check.json').read().strip().splitlines()[-1]); print(d['value'], d['step_roofline']['frac'], d['roofline']['traffic'], d['roofline']['traffic_note'], d['roofline']['k2'])"
