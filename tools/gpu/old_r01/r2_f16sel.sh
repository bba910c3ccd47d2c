# fp16 hit-first sparse levels (mode 7) vs fp32 (mode 2): encode parity + cfg4 A/B alternated
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q > gpurun_out/pytest_enc.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_enc.log
run() { timeout 900 env $4 python bench.py --config $1 --no-cpu-baseline --steps $2 --warmup 3 $3 > gpurun_out/bench_$1_$5.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$1_$5.json').read().strip().splitlines()[-1]); print('$1 $4', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
run cfg4 3 "" X=1 new1; run cfg4 3 "" FIC_F16SEL=0 old1
run cfg4 3 "" X=1 new2; run cfg4 3 "" FIC_F16SEL=0 old2
timeout 500 python tools/kineto_gaps.py cfg4 > gpurun_out/kineto_cfg4.txt 2>&1; grep -E "scan_kernel|span" gpurun_out/kineto_cfg4.txt
