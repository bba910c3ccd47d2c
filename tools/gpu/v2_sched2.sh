mkdir -p gpurun_out
run() { c=$1; shift; env "$@" timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v2_sc.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_sc.json').read().strip().splitlines()[-1]); print('$c $*', round(d['ms_per_step'],4), d['survivors_per_level'])"; }
for k in 1 2; do
run cfg3 FIC_X=0
run cfg3 FIC_SELECT=1
run cfg3 FIC_LEVELS=64,4
run cfg3 FIC_LEVELS=16,4
run cfg2 FIC_X=0
done
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q 2>&1 | tail -1
