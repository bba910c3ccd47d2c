mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v2_of_t.log 2>&1; tail -2 gpurun_out/v2_of_t.log
for c in cfg2 cfg3 cfg4; do
  st=20; [ $c = cfg4 ] && st=5
  timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/v2_of_b.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_of_b.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['encode_ms_per_image'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'])"
done
timeout 300 python tools/kineto_gaps.py cfg2 2>&1 | grep -v Warn | tail -14
