#!/bin/bash
# After the relinquish fix: do small staging budgets still hang beside K2?
# Then A/B the budgets on cfg4 / cfg3 bench lines.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/budget.log
for cfg in cfg2 cfg3; do
  ZO2_LIB_PATH=build/variants/small160wd/libzo2b200.so timeout 400 python bench.py --config $cfg --steps 4 --warmup 3 --no-cpu-baseline \
     > gpurun_out/budget_wd_$cfg.json 2> gpurun_out/budget_wd_$cfg.err
  echo "watchdog small160 $cfg exit $?" >> gpurun_out/budget.log
  grep -a watchdog gpurun_out/budget_wd_$cfg.err | head -3 >> gpurun_out/budget.log
done
ZO2_LIB_PATH=build/variants/small136/libzo2b200.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" 2>&1 | tail -2 >> gpurun_out/budget.log
for cfg in cfg4 cfg3; do
  VARIANTS="base build/variants/small160/libzo2b200.so build/variants/small136/libzo2b200.so" ARGS="--config $cfg" bash tools/ab_variants.sh >> gpurun_out/budget.log 2>&1
done
cat gpurun_out/budget.log
