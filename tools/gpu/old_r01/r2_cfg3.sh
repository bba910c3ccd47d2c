mkdir -p gpurun_out
run() { timeout 900 env $3 python bench.py --config $1 --no-cpu-baseline --steps $2 --warmup 3 > gpurun_out/b.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('$1 $3', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'])"; }
run cfg3 10 ""
run cfg3 10 "FIC_LEVELS=32,8"
run cfg3 10 "FIC_LEVELS=32,8 FIC_LANEBEST_MAX=64"
run cfg3 10 "FIC_LEVELS=64,8"
run cfg3 10 "FIC_LEVELS=16"
run cfg3 10 "FIC_LEVELS=8 FIC_LANEBEST_MAX=64"
run cfg3 10 "FIC_LEVELS=4 FIC_LANEBEST_MAX=200"
run cfg3 10 "FIC_LEVELS=16,4"
run cfg3 10 "FIC_LEVELS=128,16,4"
