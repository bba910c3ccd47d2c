# cfg4 sparse selection modes A/B (FIC_SELECT=1 default hit-first, 2 all-packed, 3 per-lane best)
mkdir -p gpurun_out
run() { timeout 900 env $4 python bench.py --config $1 --no-cpu-baseline --steps $2 --warmup 3 $3 > gpurun_out/bench_$1_$5.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$1_$5.json').read().strip().splitlines()[-1]); print('$1 $4', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
run cfg4 3 "" X=1 a; run cfg4 3 "" FIC_SELECT=2 b; run cfg4 3 "" FIC_SELECT=3 c
timeout 900 env FIC_SELECT=3 FIC_LEVELS=4096,512,64,8 python bench.py --config cfg4 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bench_cfg4_e.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg4_e.json').read().strip().splitlines()[-1]); print('cfg4 sel3 lv..8', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'], d['clocks']['sm_mhz'])"
timeout 900 env FIC_SELECT=3 FIC_LEVELS=4096,512,64,8 python -m pytest tests/test_gpu_encode.py -x -q -k "cfg4 or coarse" > gpurun_out/pytest_sel3.log 2>&1; echo "pytest sel3 rc=$?"; tail -1 gpurun_out/pytest_sel3.log
run cfg4 3 "" X=1 a2
