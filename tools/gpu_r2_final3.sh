#!/bin/bash
# final bench set with the final bench.py + gpu suite + smoke
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 ) > gpurun_out/f3_gputests.log
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 ) > gpurun_out/f3_smoke.log
R=r2g bash tools/bench_all.sh > gpurun_out/r2g_bench_all.log 2>&1
cat gpurun_out/f3_gputests.log gpurun_out/f3_smoke.log gpurun_out/r2g_bench_all.log
