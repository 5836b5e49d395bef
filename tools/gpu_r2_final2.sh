#!/bin/bash
# final round-2 evidence: -m gpu suite + smoke, ncu --set full captures at live
# clocks (--clock-control none), the whole bench set, launch lists
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 ) > gpurun_out/f2_gputests.log
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 ) > gpurun_out/f2_smoke.log
NCU="ncu --set full --clock-control none --import-source on"
K2_ARENA=bf16 K2_DIM=7168 timeout 600 $NCU -k regex:k_update_perturb -s 3 -c 1 -o gpurun_out/r2f_k2_cert_cfg4 python tools/k2_ab.py > /dev/null 2>&1
K2_ARENA=f32 K2_DIM=2048 timeout 600 $NCU -k regex:k_update_perturb -s 3 -c 1 -o gpurun_out/r2f_k2_exact_f32_cfg2 python tools/k2_ab.py > /dev/null 2>&1
PK_DIM=7168 timeout 600 $NCU -k regex:k_gemm --launch-skip 3 --launch-count 1 -o gpurun_out/r2f_gemm_mlpout_cfg4 python tools/profile_kernels.py fwd bf16 > /dev/null 2>&1
PK_DIM=7168 timeout 600 $NCU -k regex:k_attn -c 1 -o gpurun_out/r2f_attention_cfg4 python tools/profile_kernels.py fwd bf16 > /dev/null 2>&1
PK_DIM=2048 timeout 600 $NCU -k regex:k_attn -c 1 -o gpurun_out/r2f_attention_cfg2 python tools/profile_kernels.py fwd f32 > /dev/null 2>&1
PK_DIM=7168 timeout 600 $NCU -k regex:k_layernorm -c 1 -o gpurun_out/r2f_layernorm_cfg4 python tools/profile_kernels.py fwd bf16 > /dev/null 2>&1
PK_DIM=7168 timeout 600 $NCU -k regex:k_gemm --launch-skip 1 --launch-count 1 -o gpurun_out/r2f_gemm_head_ce_cfg4 python tools/profile_kernels.py head bf16 > /dev/null 2>&1
R=r2f bash tools/bench_all.sh > gpurun_out/r2f_bench_all.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2f_launches_cfg4.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2f_launches_cfg4.csv 3 > gpurun_out/r2f_launches_cfg4_summary.txt 2>&1
cat gpurun_out/f2_gputests.log gpurun_out/f2_smoke.log gpurun_out/r2f_bench_all.log gpurun_out/r2f_launches_cfg4_summary.txt | head -60
ls gpurun_out | grep r2f_
