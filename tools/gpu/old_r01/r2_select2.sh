mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q > gpurun_out/pytest_enc.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_enc.log
run() { timeout 600 env $1 python bench.py --config $2 --no-cpu-baseline --steps ${3:-10} --warmup 3 > gpurun_out/b.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('$2 $1', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'])"; }
for L in 64,8 16,2 32,4 4 8,2 32,8,2 16,4 64,16,4 128,16,2; do run FIC_LEVELS=$L cfg2; done
for L in 64,8 32,4 16,4 128,16,4; do run FIC_LEVELS=$L cfg3; done
