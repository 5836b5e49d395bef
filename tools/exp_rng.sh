for cfg in cfg2 cfg3; do for rng in exact fast; do
timeout 400 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --rng $rng > gpurun_out/rng_${cfg}_$rng.json 2> gpurun_out/rng_${cfg}_$rng.err
python -c "
import json; d=json.loads(open('gpurun_out/rng_${cfg}_$rng.json').read().strip().splitlines()[-1]); r=d['roofline']; sr=d['step_roofline']; print('$cfg $rng', round(d['value']), 'ms', round(d['ms_per_step'],1), 'gemm', round(r['gemm_ms_per_step'],1), 'k2', round(r['k2_ms_per_step'],1), 'link', round(sr['t_link_ms'],1), 'frac', round(sr['frac'],3), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/rng_${cfg}_$rng.err
done; done
