run() { c=$1; shift; env "$@" timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v2_sc.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_sc.json').read().strip().splitlines()[-1]); print('$c $*', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'])"; }
for c in cfg2 cfg3; do
run $c FIC_X=0
run $c FIC_COARSE=1
run $c FIC_F16ACC=1
run $c FIC_F16ACC=1 FIC_COARSE=1
run $c FIC_F16ACC=0
done
