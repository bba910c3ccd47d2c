mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q > gpurun_out/pytest_enc.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_enc.log
run() { timeout 900 env $4 python bench.py --config $1 --no-cpu-baseline --steps $2 --warmup 3 $3 > gpurun_out/bench_$1.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$1.json').read().strip().splitlines()[-1]); print('$1 $4', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['encode_ms_per_image'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'])"; }
run cfg2 20; run cfg3 10; run cfg5 3 "--slices 64"; run cfg4 3
run cfg3 10 "" FIC_LEVELS=16,4; run cfg3 10 "" FIC_LEVELS=8,1000; run cfg3 10 "" FIC_LEVELS=128,16,4
