#!/bin/bash
# exact-size registered host masters: tests, host RAM of the cfg4 masters, bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 ) > gpurun_out/pinned_tests.log
cat gpurun_out/pinned_tests.log
timeout 600 python - <<'PY' > gpurun_out/pinned_mem.log 2>&1
import subprocess, torch, sys
sys.path.insert(0, ".")
from paper_2503_12668_b200.model import ModelSpec
from paper_2503_12668_b200.numerics import RngState
from paper_2503_12668_b200.runtime import init_params
def used():
    return int(subprocess.run(["free", "-b"], capture_output=True, text=True).stdout.split("\n")[1].split()[2])
u0 = used()
p = init_params(ModelSpec(48, 7168, 56, 50272, 512), RngState(1), codec="bf16")
u1 = used()
print(f"cfg4 masters: host RAM used +{(u1 - u0) / 1e9:.1f} GB for {48 * 616655872 * 2 / 1e9:.1f} GB of bf16 blocks; is_pinned={p.blocks[0].is_pinned()}")
PY
cat gpurun_out/pinned_mem.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/pinned_bench.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/pinned_bench.json').read().strip().splitlines()[-1]); sr=d['step_roofline']; print(d['value'], sr['frac'], sr['h2d_gbs'], sr['link_probe_gbs'], d.get('gpu_idle_pct'))"
