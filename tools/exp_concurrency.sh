B="python bench.py --config ${CFG:-cfg3} --steps 3 --warmup 2 --no-cpu-baseline"
run() { name=$1; shift; env "$@" timeout 300 $B $EXTRA > gpurun_out/exp_$name.json 2>gpurun_out/exp_$name.err; python -c "
import json,sys; d=json.loads(open('gpurun_out/exp_$name.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$name', round(d['value']), 'ms', round(d['ms_per_step'],1), 'gemm', round(r['gemm_ms_per_step'],1), 'k2', round(r['k2_ms_per_step'],1), 'idle', round(d['gpu_idle_pct'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/exp_$name.err; }
EXTRA="" run A_base
EXTRA="--operand-sets 2" run F_160_tiles ZO2_LIB_PATH=build/variants/g160/libzo2b200.so ZO2_K2_CONCURRENT_CTAS=1000
EXTRA="--operand-sets 2" run G_200_tiles ZO2_K2_CONCURRENT_CTAS=1000
EXTRA="--operand-sets 2" run H_128_tiles ZO2_LIB_PATH=build/variants/g128/libzo2b200.so ZO2_K2_CONCURRENT_CTAS=1000
