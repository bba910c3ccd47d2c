FIC_LIB=$PWD/paper_1404_0774_b200/libfic_b200.so timeout 300 python tools/e2e_probe.py cfg2
timeout 300 python tools/e2e_breakdown.py cfg2 2>&1 | tail -28
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v2_b.json 2>&1; tail -1 gpurun_out/v2_b.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e'])"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
