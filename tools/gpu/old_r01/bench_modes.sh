for m in 1cta pair; do
  for c in cfg2 cfg4; do
    FIC_SCAN=$m timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m', '$c', round(d['ms_per_step'],3), 'ms/step', 'scan', round(d['roofline']['kernel_ms'],3), 'frac', round(d['roofline']['frac'],3), d['survivors_per_level'])"
  done
done
