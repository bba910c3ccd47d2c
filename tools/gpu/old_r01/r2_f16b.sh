# default policy (fp16 accumulator on large-pool full levels) vs FIC_F16ACC=0; full GPU suite
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_f16.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_f16.log
run() { timeout 900 env $4 python bench.py --config $1 --no-cpu-baseline --steps $2 --warmup 3 $3 > gpurun_out/bench_$1_$5.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$1_$5.json').read().strip().splitlines()[-1]); print('$1 $4', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['encode_ms_per_image'],4), 'scan', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3), d['survivors_per_level'], d['clocks'])"; }
run cfg4 3 "" X=1 def; run cfg4 3 "" FIC_F16ACC=0 f32; run cfg4 3 "" X=1 def2
run cfg5 3 "" X=1 def; run cfg5 3 "" FIC_F16ACC=0 f32
run cfg2 20 "" X=1 def
