mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_cli.py tests/test_gpu_smoke_api.py -x -q 2>&1 | tail -1
for k in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v2_dec_b.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/v2_dec_b.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['decoder']['ms'], d['decoder']['frac'])"
done
