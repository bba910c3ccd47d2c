# quick A/B pass: GPU tests of the encoder, cfg2 default / f16, cfg3, cfg4; pool timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encode.py tests/test_gpu_fit.py -x -q > gpurun_out/v2_quick_t.log 2>&1; tail -2 gpurun_out/v2_quick_t.log
for v in "FIC_X=0" "FIC_F16ACC=1"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/v2_quick_b.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_quick_b.json').read().strip().splitlines()[-1]); print('cfg2 $v', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), 'pool', round(d['pool']['ms']*1e3,1), 'us', round(d['pool']['frac'],3), d['survivors_per_level'])"
done
for c in cfg3 cfg4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v2_quick_c.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_quick_c.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), 'pool', round(d['pool']['ms']*1e3,1), 'us', round(d['pool']['frac'],3))"
done
