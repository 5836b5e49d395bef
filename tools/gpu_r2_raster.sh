#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "raster" 2>&1 | tail -3 ) > gpurun_out/raster_tests.log
timeout 600 python tools/raster_sweep.py > gpurun_out/raster_sweep.log 2>&1
RS_SHAPES=mlp_out,qkv RS_REPS=2 timeout 900 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none --csv \
   -k regex:k_gemm python tools/raster_sweep.py > gpurun_out/raster_ncu.csv 2>&1
timeout 300 python tools/option_b_probe.py > gpurun_out/option_b.json 2>&1
cat gpurun_out/raster_tests.log gpurun_out/raster_sweep.log gpurun_out/option_b.json
