# fp16 full level on small pools (cfg3, cfg5): A/B alternated
mkdir -p gpurun_out
run() { timeout 900 env $4 python bench.py --config $1 --no-cpu-baseline --steps $2 --warmup 3 $3 > gpurun_out/bench_$1_$5.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$1_$5.json').read().strip().splitlines()[-1]); print('$1 $4', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'], d['clocks']['sm_mhz'])"; }
for i in 1 2; do run cfg3 10 "" X=1 a$i; run cfg3 10 "" FIC_F16ACC=1 b$i; done
for i in 1 2; do run cfg5 3 "--slices 64" X=1 a$i; run cfg5 3 "--slices 64" FIC_F16ACC=1 b$i; done
