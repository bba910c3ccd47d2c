# cfg4 level schedule A/B with the fp16-accumulator full level
mkdir -p gpurun_out
run() { timeout 900 env $4 python bench.py --config $1 --no-cpu-baseline --steps $2 --warmup 3 $3 > gpurun_out/bench_$1_$5.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$1_$5.json').read().strip().splitlines()[-1]); print('$1 $4', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'], d['clocks']['sm_mhz'])"; }
run cfg4 3 "" X=1 a
run cfg4 3 "" FIC_LEVELS=4096,512,64,16 b
run cfg4 3 "" FIC_LEVELS=4096,512,64 c
run cfg4 3 "" FIC_LEVELS=4096,512,128,32 d
run cfg4 3 "" FIC_LEVELS=2048,256,32 e
run cfg4 3 "" FIC_LEVELS=4096,1024,256,64,16 f
