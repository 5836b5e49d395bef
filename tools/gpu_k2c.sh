#!/bin/bash
# K2c bring-up: bound probe, certified-vs-exact parity, K2 codec tests, A/B timing
cd "$(dirname "$0")/.."
timeout 900 python -m pytest -x -q -s tests/test_gpu_kernels.py -k "zapprox or certified or update_perturb or codec" 2>&1 | grep -v "^$" | tail -30 > gpurun_out/k2c_tests.log
for d in 4096 7168; do for v in 1 0; do K2_VARIANT=$v K2_ARENA=bf16 K2_DIM=$d timeout 120 python tools/k2_ab.py; done; done > gpurun_out/k2c_ab.log 2>&1
for v in 1 0; do K2_VARIANT=$v K2_ARENA=f16 K2_DIM=12288 timeout 120 python tools/k2_ab.py; done >> gpurun_out/k2c_ab.log 2>&1
for d in 4096 7168; do ZO2_LIB_PATH=build/variants/prefetch/libzo2b200.so K2_VARIANT=0 K2_ARENA=bf16 K2_DIM=$d timeout 120 python tools/k2_ab.py; done >> gpurun_out/k2c_ab.log 2>&1
K2_VARIANT=0 K2_ARENA=bf16 K2_DIM=4096 timeout 300 ncu --set full --import-source on -k regex:k_update_perturb_cert -s 2 -c 1 -o gpurun_out/k2c_full python tools/k2_ab.py > gpurun_out/k2c_ncu.log 2>&1
cat gpurun_out/k2c_tests.log gpurun_out/k2c_ab.log
