#!/bin/bash
# f32 arenas: certified update draw (K2 upd_cert) -- parity + A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1500 python -m pytest -q -x tests/test_gpu_kernels.py -k "update_perturb or embed or axpy or init" 2>&1 | tail -3;
  timeout 1500 python -m pytest -q -x tests/test_gpu_engine.py tests/test_gpu_runner.py tests/test_gpu_trace.py tests/test_gpu_f64.py tests/test_gpu_amp.py 2>&1 | tail -3 ) > gpurun_out/k2h_tests.log
: > gpurun_out/k2h_ab.log
for lib in "" build/variants/k2nocert/libzo2b200.so; do
  for d in 2048 768; do
    ZO2_LIB_PATH=$lib K2_ARENA=f32 K2_DIM=$d timeout 120 python tools/k2_ab.py >> gpurun_out/k2h_ab.log 2>&1
  done
done
for cfg in cfg2 cfg1; do
  VARIANTS="base build/variants/k2nocert/libzo2b200.so base" ARGS="--config $cfg" bash tools/ab_variants.sh >> gpurun_out/k2h_ab.log 2>&1
done
cat gpurun_out/k2h_tests.log gpurun_out/k2h_ab.log
