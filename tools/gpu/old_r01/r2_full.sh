# full GPU tests + smoke + bench cfg2/3/4/5 + warm per-kernel timeline of a cfg2 encode
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
run() { timeout 900 python bench.py --config $1 --no-cpu-baseline --steps $2 --warmup 3 $3 > gpurun_out/bench_$1.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$1.json').read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['encode_ms_per_image'],4), 'scan', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3), d['survivors_per_level'])"; }
run cfg2 20; run cfg3 10; run cfg4 3; run cfg5 3 "--slices 64"
timeout 600 python tools/kineto_gaps.py cfg2 > gpurun_out/kineto_cfg2.txt 2>&1; tail -1 gpurun_out/kineto_cfg2.txt
