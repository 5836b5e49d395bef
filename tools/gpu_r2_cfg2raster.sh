#!/bin/bash
cd "$(dirname "$0")/.."
for gm in 1 2 4 8 16; do
  PK_DIM=2048 PK_RASTER=12,$gm timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
     -k regex:k_gemm --launch-skip 3 --launch-count 1 python tools/profile_kernels.py fwd f32 2>/dev/null | grep -E "dram__bytes|duration" | awk -F'","' -v g=$gm '{print "gm="g, $(NF-2), $NF}'
done
