mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v2_e2e_t.log 2>&1; tail -2 gpurun_out/v2_e2e_t.log
timeout 300 python tools/e2e_probe.py
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/v2_e2e_b.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/v2_e2e_b.json').read().strip().splitlines()[-1]); print('cfg2', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['encode_ms_per_image'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'], d['gpu_launches']/d['steps'])"
timeout 300 python tools/kineto_gaps.py cfg2 2>&1 | grep -v Warn | tail -16
