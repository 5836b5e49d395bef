#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/budget2.log
for cfg in cfg2 cfg4; do
  ZO2_LIB_PATH=build/variants/small160sync/libzo2b200.so timeout 300 python bench.py --config $cfg --steps 4 --warmup 3 --no-cpu-baseline \
     > gpurun_out/budget2_$cfg.json 2> gpurun_out/budget2_$cfg.err
  echo "sync-before-alloc small160 $cfg exit $?" >> gpurun_out/budget2.log
  head -c 200 gpurun_out/budget2_$cfg.json >> gpurun_out/budget2.log; echo >> gpurun_out/budget2.log
done
cat gpurun_out/budget2.log
