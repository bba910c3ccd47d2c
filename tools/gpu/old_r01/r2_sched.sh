mkdir -p gpurun_out
run() { timeout 900 env $4 python bench.py --config $1 --no-cpu-baseline --steps $2 --warmup 3 $3 > gpurun_out/bench_$1.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$1.json').read().strip().splitlines()[-1]); print('$1 $4', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['encode_ms_per_image'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'])"; }
run cfg2 20
run cfg2 20 "" "FIC_LEVELS=2 FIC_LANEBEST_MAX=100"
run cfg2 20 "" "FIC_LEVELS=8,2 FIC_LANEBEST_MAX=100"
run cfg2 20 "" "FIC_LEVELS=16,2 FIC_LANEBEST_MAX=100"
run cfg2 20 "" "FIC_LEVELS=4,2 FIC_LANEBEST_MAX=100"
run cfg2 20 "" "FIC_LEVELS=8"
run cfg3 10 "" "FIC_LANEBEST_MAX=200"
run cfg3 10 "" "FIC_LEVELS=16,2 FIC_LANEBEST_MAX=300"
run cfg3 10 "" "FIC_LEVELS=32,4,2 FIC_LANEBEST_MAX=300"
