# re-entry check of HEAD: GPU suite, smoke, cfg1/cfg2/cfg3 bench lines
mkdir -p gpurun_out/c
O=gpurun_out/c
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
for c in cfg2 cfg1 cfg3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "import json; d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],4), 'e2e', d['e2e'], 'scan', round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3), 'launches', d.get('gpu_launches'))"
done
