#!/bin/bash
# attention: three S/P buffers at hd 64 with per-buffer P.V barriers
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -2 ) > gpurun_out/attn_tests.log
cat gpurun_out/attn_tests.log
: > gpurun_out/attn_ab.log
for i in 1 2; do
for lib in "" build/variants/attnsb2/libzo2b200.so; do
  echo "lib=${lib:-base(sb3 at hd64)}" >> gpurun_out/attn_ab.log
  ZO2_LIB_PATH=$lib ATTN_SHAPES="16,512,32,64,1;16,512,32,64,0;16,512,32,128,0;16,512,56,128,0;4,2048,32,64,1" timeout 300 python tools/attn_ab.py >> gpurun_out/attn_ab.log 2>&1
done
done
SAN_DIM=2048 SAN_BLOCKS=2 SAN_BATCH=2 SAN_VOCAB=8192 SAN_ARITH=f32 timeout 1500 compute-sanitizer --tool synccheck \
    --print-limit 20 python tools/sanitize_step.py > gpurun_out/r2_sanitizer_synccheck_f32_sb3.log 2>&1
tail -3 gpurun_out/r2_sanitizer_synccheck_f32_sb3.log
VARIANTS="base build/variants/attnsb2/libzo2b200.so base" ARGS="--config cfg2 --steps 5 --warmup 3" bash tools/ab_variants.sh >> gpurun_out/attn_ab.log 2>&1
cat gpurun_out/attn_ab.log
