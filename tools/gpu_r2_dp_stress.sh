#!/bin/bash
# repeated runs of the data-parallel tests (sharded-masters finalize race check)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/r2_dp_stress.log
for i in $(seq 1 15); do
  timeout 300 python -m pytest tests/test_gpu_dp_sharded.py tests/test_gpu_dp_engine.py -q -x 2>&1 | tail -1 | sed "s/^/run $i: /" >> gpurun_out/r2_dp_stress.log
done
cat gpurun_out/r2_dp_stress.log
