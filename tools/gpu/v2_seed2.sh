mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q > gpurun_out/v2_seed_t.log 2>&1; tail -2 gpurun_out/v2_seed_t.log
for c in cfg2 cfg3 cfg4; do for v in "FIC_SEED=0" "FIC_SEED=1" "FIC_SEED=3"; do
  st=20; [ $c = cfg4 ] && st=5
  env $v timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/v2_seed_b.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_seed_b.json').read().strip().splitlines()[-1]); print('$c $v', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'], d['gpu_launches']/d['steps'])"
done; done
