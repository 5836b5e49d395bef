#!/bin/bash
# Round-2 check: selected -m gpu tests, smoke(), default bench line (cfg4).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SEL=${SEL:-"tests -m gpu"}
( timeout 2400 python -m pytest $SEL -q -x 2>&1 | tail -40 ) > gpurun_out/gputests.log
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5 ) > gpurun_out/smoke.log
if [ -z "$NOBENCH" ]; then
  s=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench wall $(( $(date +%s) - s )) s" >> gpurun_out/bench_default.err
fi
cat gpurun_out/gputests.log gpurun_out/smoke.log gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
