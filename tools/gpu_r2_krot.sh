#!/bin/bash
# K rotation of the GEMM K loop: tests, DRAM traffic A/B, bench A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or attention" 2>&1 | tail -3;
  timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_amp.py -q -x 2>&1 | tail -3 ) > gpurun_out/krot_tests.log
cat gpurun_out/krot_tests.log
for lib in "" build/variants/nokrot/libzo2b200.so; do
  tag=$([ -z "$lib" ] && echo krot || echo nokrot)
  for d in 2048 7168 12288; do
    ZO2_LIB_PATH=$lib RS_DIM=$d RS_GMS=8 RS_REPS=2 timeout 900 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none --csv \
      -k regex:k_gemm python tools/raster_sweep.py > gpurun_out/krot_ncu_${d}_$tag.csv 2>&1
  done
done
for cfg in cfg5 cfg4 cfg2; do
  VARIANTS="base build/variants/nokrot/libzo2b200.so base" ARGS="--config $cfg --steps 3 --warmup 2" bash tools/ab_variants.sh >> gpurun_out/krot_ab.log 2>&1
done
cat gpurun_out/krot_ab.log
