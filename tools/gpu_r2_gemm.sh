#!/bin/bash
# GEMM raster + attention barrier fix: kernel tests, synccheck, cfg4 mlp_out
# traffic, cfg4 bench with 2 and 1 operand sets.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
R=${R:-r2}
( timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or attention" 2>&1 | tail -5 ) > gpurun_out/${R}_gemm_tests.log
SAN_DIM=4096 SAN_BLOCKS=2 SAN_BATCH=2 SAN_VOCAB=8192 timeout 1200 compute-sanitizer --tool synccheck \
    --print-limit 50 python tools/sanitize_step.py > gpurun_out/${R}_sanitizer_synccheck.log 2>&1
echo "exit $?" >> gpurun_out/${R}_sanitizer_synccheck.log
PK_DIM=7168 timeout 600 ncu --set full --import-source on -k regex:k_gemm --launch-skip 3 --launch-count 1 \
    -o gpurun_out/${R}_gemm_mlpout_cfg4_raster python tools/profile_kernels.py fwd bf16 > /dev/null 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${R}_bench_cfg4_raster.json 2> gpurun_out/${R}_bench_err.log
timeout 900 python bench.py --no-cpu-baseline --operand-sets 1 > gpurun_out/${R}_bench_cfg4_raster_sets1.json 2>> gpurun_out/${R}_bench_err.log
cat gpurun_out/${R}_gemm_tests.log; tail -4 gpurun_out/${R}_sanitizer_synccheck.log
python tools/ncu_summary.py gpurun_out/${R}_gemm_mlpout_cfg4_raster.ncu-rep | head -6
for f in gpurun_out/${R}_bench_cfg4_raster*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],1), d['ms_per_step'], d['step_roofline']['frac'], d['roofline']['gemm_ms_per_step'], d['roofline']['k2_ms_per_step'], d['clocks'])"; done
tail -5 gpurun_out/${R}_bench_err.log
