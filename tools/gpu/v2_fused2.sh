mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_encode.py -x -q -k "fused or noise32 or cfg2_ct" > gpurun_out/v2_fused_t1.log 2>&1; tail -3 gpurun_out/v2_fused_t1.log
for f in 1 0; do
  FIC_FUSED=$f timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/v2_fused_b$f.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_fused_b$f.json').read().strip().splitlines()[-1]); print('fused=$f', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), 'matcher', round(d['roofline']['matcher_ms'],4), d['survivors_per_level'])"
done
