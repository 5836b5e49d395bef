#!/bin/bash
# final bench set on the final code + two more live ncu captures
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
R=r2z bash tools/bench_all.sh > gpurun_out/r2z_bench_all.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
K2_ARENA=f16 K2_DIM=12288 timeout 600 $NCU -k regex:k_update_perturb -s 3 -c 1 -o gpurun_out/r2z_k2_cert_cfg5 python tools/k2_ab.py > /dev/null 2>&1
K2_ARENA=bf16 K2_DIM=7168 timeout 600 $NCU -k regex:k_k2c_fixup -s 3 -c 1 -o gpurun_out/r2z_k2c_fixup_cfg4 python tools/k2_ab.py > /dev/null 2>&1
PK_DIM=7168 timeout 600 $NCU -k regex:k_embed -c 1 -o gpurun_out/r2z_embed_cfg4 python tools/profile_kernels.py embed bf16 > /dev/null 2>&1
cat gpurun_out/r2z_bench_all.log
