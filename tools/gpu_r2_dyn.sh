#!/bin/bash
# CTA-pair GEMM dynamic tile scheduler: tests (watchdog build first), DRAM traffic, bench A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( ZO2_LIB_PATH=build/variants/gemm2wd/libzo2b200.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" 2>&1 | tail -3 ) > gpurun_out/dyn_tests.log
( timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or attention" 2>&1 | tail -3 ) >> gpurun_out/dyn_tests.log
cat gpurun_out/dyn_tests.log
for lib in "" build/variants/gemm2static/libzo2b200.so; do
  for d in 7168 12288; do
    ZO2_LIB_PATH=$lib RS_DIM=$d RS_GMS=8 RS_SHAPES=mlp_out,qkv RS_REPS=2 timeout 900 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none --csv \
      -k regex:k_gemm python tools/raster_sweep.py > gpurun_out/dyn_ncu_${d}_$(basename "${lib:-dyn}" .so | tr '/' '_').csv 2>&1
    ZO2_LIB_PATH=$lib RS_DIM=$d RS_GMS=8,16 RS_REPS=4 timeout 600 python tools/raster_sweep.py >> gpurun_out/dyn_sweep.log 2>&1
  done
done
cat gpurun_out/dyn_sweep.log
for cfg in cfg5 cfg4; do
  VARIANTS="base build/variants/gemm2static/libzo2b200.so base" ARGS="--config $cfg --steps 3 --warmup 2" bash tools/ab_variants.sh >> gpurun_out/dyn_ab.log 2>&1
done
cat gpurun_out/dyn_ab.log
