#!/bin/bash
# Round-2 profile set (run under gpurun): new DP tests, cfg4 launch list,
# ncu --set full of K2 (certified binary32 path, OPT-30B bf16 block), the
# cfg4 mlp_out GEMM and hd-128 attention, and compute-sanitizer on a
# co-running step.  Everything lands in gpurun_out/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
R=${R:-r2}
( timeout 900 python -m pytest tests/test_gpu_dp_engine.py -q -x 2>&1 | tail -15 ) > gpurun_out/${R}_dp_tests.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches_cfg4.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${R}_launches_cfg4.out 2>&1
python tools/launch_summary.py gpurun_out/${R}_launches_cfg4.csv 2 > gpurun_out/${R}_launches_cfg4_summary.txt 2>&1
K2_ARENA=bf16 K2_DIM=7168 timeout 600 ncu --set full --import-source on -k regex:k_update_perturb -s 3 -c 1 \
    -o gpurun_out/${R}_k2_cert_cfg4 python tools/k2_ab.py > gpurun_out/${R}_k2_ncu.log 2>&1
PK_DIM=7168 timeout 600 ncu --set full --import-source on -k regex:k_gemm --launch-skip 3 --launch-count 1 \
    -o gpurun_out/${R}_gemm_mlpout_cfg4 python tools/profile_kernels.py fwd bf16 > gpurun_out/${R}_gemm_ncu.log 2>&1
PK_DIM=7168 timeout 600 ncu --set full --import-source on -k regex:k_attn -c 1 \
    -o gpurun_out/${R}_attention_cfg4 python tools/profile_kernels.py fwd bf16 > gpurun_out/${R}_attn_ncu.log 2>&1
PK_DIM=7168 timeout 600 ncu --set full --import-source on -k regex:k_layernorm -c 1 \
    -o gpurun_out/${R}_layernorm_cfg4 python tools/profile_kernels.py fwd bf16 > gpurun_out/${R}_ln_ncu.log 2>&1
for tool in synccheck racecheck memcheck; do
  SAN_DIM=4096 SAN_BLOCKS=2 SAN_BATCH=2 SAN_VOCAB=8192 timeout 1200 compute-sanitizer --tool $tool \
      --print-limit 50 python tools/sanitize_step.py > gpurun_out/${R}_sanitizer_${tool}.log 2>&1
  echo "exit $?" >> gpurun_out/${R}_sanitizer_${tool}.log
done
ls -la gpurun_out
cat gpurun_out/${R}_dp_tests.log; tail -5 gpurun_out/${R}_sanitizer_*.log; cat gpurun_out/${R}_launches_cfg4_summary.txt | head -30
