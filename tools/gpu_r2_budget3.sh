#!/bin/bash
# staging-budget A/B on one box (after the pair-alloc fix) + the -m gpu suite
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 ) > gpurun_out/budget3_tests.log
: > gpurun_out/budget3.log
for cfg in cfg4 cfg3 cfg2; do
  echo "== $cfg" >> gpurun_out/budget3.log
  VARIANTS="base build/variants/small160/libzo2b200.so build/variants/small136/libzo2b200.so base" ARGS="--config $cfg" bash tools/ab_variants.sh >> gpurun_out/budget3.log 2>&1
done
cat gpurun_out/budget3_tests.log gpurun_out/budget3.log
