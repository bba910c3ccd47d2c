run() { c=$1; shift; env "$@" timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v2_sc.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_sc.json').read().strip().splitlines()[-1]); print('$c $*', round(d['ms_per_step'],4), d['survivors_per_level'], d['gpu_launches']/d['steps'])"; }
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for k in 1 2; do run cfg2 FIC_X=0; run cfg2 FIC_EXPAND=1; done
run cfg3 FIC_X=0; run cfg3 FIC_EXPAND=1
run cfg4 FIC_X=0; run cfg4 FIC_EXPAND=1
