run() { c=$1; shift; env "$@" timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v2_sc.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_sc.json').read().strip().splitlines()[-1]); print('$c $*', round(d['ms_per_step'],4))"; }
for k in 1 2; do for v in 8 4 2 1; do run cfg2 FIC_ROP_SPLIT=$v; done; done
for v in 8 4 2; do run cfg4 FIC_ROP_SPLIT=$v; done
