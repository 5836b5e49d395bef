#!/bin/bash
# full -m gpu suite + smoke + reference arm (cfg4) + nproc
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
( timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -40 ) > gpurun_out/gputests.log
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5 ) > gpurun_out/smoke.log
s=$(date +%s); timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref wall $(( $(date +%s) - s )) s" >> gpurun_out/bench_ref.err
cat gpurun_out/nproc.txt gpurun_out/gputests.log gpurun_out/smoke.log gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
