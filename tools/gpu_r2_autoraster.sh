#!/bin/bash
cd "$(dirname "$0")/.."
( timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" 2>&1 | tail -1 )
for r in 0,0 12,8; do
  PK_DIM=2048 PK_RASTER=$r timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
     -k regex:k_gemm --launch-skip 3 --launch-count 1 python tools/profile_kernels.py fwd f32 2>/dev/null | grep -E "dram__bytes|duration" | awk -F'","' -v g=$r '{print "raster="g, $(NF-2), $NF}'
  PK_DIM=4096 PK_RASTER=$r timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none --csv \
     -k regex:k_gemm python tools/profile_kernels.py fwd bf16 2>/dev/null | grep -E "dram__bytes_read|duration" | awk -F'","' -v g=$r '{print "cfg3 raster="g, $(NF-2), $NF}'
done
for cfg in cfg2 cfg3 cfg4; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value']), round(d['ms_per_step'],1), round(d['step_roofline']['frac'],3), round(d['roofline']['gemm_ms_per_step'],1))"
done
