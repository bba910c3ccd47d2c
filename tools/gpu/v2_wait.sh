mkdir -p gpurun_out
for v in "FIC_DEBUG=0" "FIC_DEBUG=512"; do for c in cfg2 cfg3 cfg4; do
  st=20; [ $c = cfg4 ] && st=5
  env $v timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/v2_w_b.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_w_b.json').read().strip().splitlines()[-1]); print('$c $v', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'])"
done; done
