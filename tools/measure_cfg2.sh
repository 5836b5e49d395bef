timeout 600 python bench.py > gpurun_out/r1_bench_cfg2.json 2> gpurun_out/r1_bench_cfg2.err
tail -1 gpurun_out/r1_bench_cfg2.json | cut -c1-600
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches_cfg2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r1_launches_cfg2.csv 3 | head -14
