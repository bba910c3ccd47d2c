timeout 1200 python -m pytest tests -x -q -m gpu -k "batch or cfg5 or volume or slices" 2>&1 | tail -3
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/v2_b5.json 2>&1; tail -1 gpurun_out/v2_b5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['e2e']['encode_ms_per_image'], d['encode_ms_per_image'])"
