#!/bin/bash
# compute-sanitizer on the final build (dynamic pair scheduler, cross-CTA tile ring)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in synccheck racecheck memcheck; do
  SAN_DIM=4096 SAN_BLOCKS=2 SAN_BATCH=2 SAN_VOCAB=8192 timeout 1500 compute-sanitizer --tool $tool \
      --print-limit 50 python tools/sanitize_step.py > gpurun_out/r2f_sanitizer_${tool}.log 2>&1
  echo "exit $?" >> gpurun_out/r2f_sanitizer_${tool}.log
done
# the f32 (split) path too: single-CTA + pair kernels, hd-64 attention, queued K2
for tool in synccheck memcheck; do
  SAN_DIM=2048 SAN_BLOCKS=2 SAN_BATCH=2 SAN_VOCAB=8192 SAN_ARITH=f32 timeout 1500 compute-sanitizer --tool $tool \
      --print-limit 50 python tools/sanitize_step.py > gpurun_out/r2f_sanitizer_${tool}_f32.log 2>&1
  echo "exit $?" >> gpurun_out/r2f_sanitizer_${tool}_f32.log
done
tail -4 gpurun_out/r2f_sanitizer_*.log
