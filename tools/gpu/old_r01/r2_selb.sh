# batched sparse-level reductions: parity (encode tests) + cfg4/cfg3/cfg2 bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_encode.py -x -q > gpurun_out/pytest_enc.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_enc.log
run() { timeout 900 env $4 python bench.py --config $1 --no-cpu-baseline --steps $2 --warmup 3 $3 > gpurun_out/bench_$1_$5.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$1_$5.json').read().strip().splitlines()[-1]); print('$1 $4', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['encode_ms_per_image'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
run cfg4 3 "" X=1 a; run cfg3 10 "" X=1 a; run cfg2 20 "" X=1 a; run cfg4 3 "" X=1 b
timeout 500 python tools/kineto_gaps.py cfg4 > gpurun_out/kineto_cfg4.txt 2>&1; grep -E "scan_kernel|span" gpurun_out/kineto_cfg4.txt
