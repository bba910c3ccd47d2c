run() { c=$1; shift; env "$@" timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v2_sc.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_sc.json').read().strip().splitlines()[-1]); print('$c $*', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'], d['gpu_launches']/d['steps'])"; }
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q 2>&1 | tail -1
for k in 1 2; do run cfg2 FIC_X=0; run cfg2 FIC_EPI_BOUND=0; done
run cfg5 FIC_X=0
run cfg5 FIC_EPI_BOUND=0
timeout 300 python tools/kineto_gaps.py cfg2 2>&1 | grep -v -i warn | tail -12
