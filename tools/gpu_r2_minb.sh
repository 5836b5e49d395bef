#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/minb.log
for lib in "" build/variants/k2cminb4/libzo2b200.so build/variants/k2cminb2/libzo2b200.so; do
  for d in 7168 12288; do
    a=$([ $d = 12288 ] && echo f16 || echo bf16)
    echo "lib=${lib:-base}" >> gpurun_out/minb.log
    ZO2_LIB_PATH=$lib K2_ARENA=$a K2_DIM=$d timeout 200 python tools/k2_ab.py >> gpurun_out/minb.log 2>&1
  done
done
VARIANTS="base build/variants/k2cminb4/libzo2b200.so build/variants/k2cminb2/libzo2b200.so base" ARGS="--config cfg5 --steps 3 --warmup 2" bash tools/ab_variants.sh >> gpurun_out/minb.log 2>&1
cat gpurun_out/minb.log
