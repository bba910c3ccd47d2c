mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v2_inline_t.log 2>&1; tail -3 gpurun_out/v2_inline_t.log
for v in "FIC_EVAL_SPLIT=0" "FIC_EVAL_SPLIT=1" "FIC_FUSED=1"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/v2_inline_b.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_inline_b.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['encode_ms_per_image'],4), 'scan', round(d['roofline']['kernel_ms'],4), 'matcher', round(d['roofline']['matcher_ms'],4), d['survivors_per_level'], d['gpu_launches'])"
done
for c in cfg3 cfg4; do for v in "FIC_EVAL_SPLIT=0" "FIC_EVAL_SPLIT=1"; do
  env $v timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v2_inline_c.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_inline_c.json').read().strip().splitlines()[-1]); print('$c $v', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'])"
done; done
