#!/bin/bash
# Round profile set (run under gpurun): bench launch list + ncu --set full of
# the dominant GEMM launch (mlp_out, split) and of K2, summaries in gpurun_out/.
set -u
R=${R:-r1}
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches_cfg2.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${R}_launches_cfg2.csv 3 > gpurun_out/${R}_launches_cfg2_summary.txt 2>/dev/null
ncu --set full --import-source on -k regex:k_gemm --launch-skip 3 --launch-count 1 \
    -o gpurun_out/${R}_gemm_mlpout python tools/profile_kernels.py fwd f32 > /dev/null 2>&1
ncu --set full --import-source on -k regex:k_update_perturb -c 1 \
    -o gpurun_out/${R}_k2_exact python tools/profile_kernels.py k2 f32 > /dev/null 2>&1
ZO2_RNG=fast ncu --set full --import-source on -k regex:k_update_perturb -c 1 \
    -o gpurun_out/${R}_k2_fast python tools/profile_kernels.py k2 f32 > /dev/null 2>&1
ncu --set full --import-source on -k regex:k_attn -c 1 \
    -o gpurun_out/${R}_attention python tools/profile_kernels.py fwd f32 > /dev/null 2>&1
ncu --set full --import-source on -k regex:k_layernorm -c 1 \
    -o gpurun_out/${R}_layernorm python tools/profile_kernels.py fwd f32 > /dev/null 2>&1
ncu --set full --import-source on -k regex:k_gemm --launch-skip 1 --launch-count 1 \
    -o gpurun_out/${R}_gemm_head_ce python tools/profile_kernels.py head f32 > /dev/null 2>&1
ncu --set full --import-source on -k regex:k_embed -c 1 \
    -o gpurun_out/${R}_embed python tools/profile_kernels.py embed f32 > /dev/null 2>&1
ls -la gpurun_out | grep $R
