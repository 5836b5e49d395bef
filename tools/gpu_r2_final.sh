#!/bin/bash
# round-2 bench set + launch lists + a functional 2-rank bench (gloo, one GPU)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
R=r2 bash tools/bench_all.sh > gpurun_out/r2_bench_all.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_launches_cfg4_final.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_launches_cfg4_final.csv 3 > gpurun_out/r2_launches_cfg4_final_summary.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_launches_cfg2.csv \
    python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_launches_cfg2.csv 3 > gpurun_out/r2_launches_cfg2_summary.txt 2>&1
ZO2_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --config cfg2 --steps 2 --warmup 3 > gpurun_out/r2_bench_cfg2_dp2_gloo_shared_gpu.json 2> gpurun_out/r2_dp2.err
tail -3 gpurun_out/r2_dp2.err
cat gpurun_out/r2_bench_all.log gpurun_out/r2_launches_cfg4_final_summary.txt | head -60
