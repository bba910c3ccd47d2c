mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_smoke_api.py tests/test_cli.py tests/test_gpu_ref_binding.py -x -q > gpurun_out/v2_dec_t.log 2>&1; tail -3 gpurun_out/v2_dec_t.log
python -c "import __graft_entry__ as g; g.smoke()"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v2_dec_b.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/v2_dec_b.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['decoder'])"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_means --launch-skip 5 --launch-count 1 -o gpurun_out/v2_decode2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
