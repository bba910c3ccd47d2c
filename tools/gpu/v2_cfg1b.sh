run() { c=$1; shift; env "$@" timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v2_sc.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_sc.json').read().strip().splitlines()[-1]); print('$c $*', round(d['ms_per_step'],4), d['survivors_per_level'])"; }
run cfg1 FIC_X=0
run cfg1 FIC_SEED=1
run cfg1 FIC_SEED=3
run cfg2 FIC_X=0
