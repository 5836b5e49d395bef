#!/bin/bash
# L2 eviction hints (A evict_last, B evict_first) + adaptive raster height
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or attention" 2>&1 | tail -3 ) > gpurun_out/l2h_tests.log
cat gpurun_out/l2h_tests.log
for lib in "" build/variants/nohint/libzo2b200.so; do
  tag=$([ -z "$lib" ] && echo hint || echo nohint)
  for d in 2048 7168 12288; do
    ZO2_LIB_PATH=$lib RS_DIM=$d RS_GMS=0,8 RS_REPS=2 timeout 900 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none --csv \
      -k regex:k_gemm python tools/raster_sweep.py > gpurun_out/l2h_ncu_${d}_$tag.csv 2>&1
  done
done
for cfg in cfg4 cfg5 cfg2; do
  VARIANTS="base build/variants/nohint/libzo2b200.so base" ARGS="--config $cfg --steps 3 --warmup 2" bash tools/ab_variants.sh >> gpurun_out/l2h_ab.log 2>&1
done
cat gpurun_out/l2h_ab.log
