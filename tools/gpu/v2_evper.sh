mkdir -p gpurun_out
run() { c=$1; shift; env "$@" timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v2_sc.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_sc.json').read().strip().splitlines()[-1]); print('$c $*', round(d['ms_per_step'],4), d['survivors_per_level'])"; }
for k in 1 2; do for p in 4 8 16 32; do run cfg2 FIC_EVAL_PER=$p; done; done
for p in 8 16 32; do run cfg3 FIC_EVAL_PER=$p; done
