mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q > gpurun_out/pytest_enc.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_enc.log
for c in cfg2 cfg3; do
timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], 'e2e', d['e2e']['encode_ms_per_image'], 'scan', d['roofline']['kernel_ms'], 'matcher', d['roofline']['matcher_ms'], d['survivors_per_level'], 'decoder ms', d['decoder']['ms'], d['decoder']['frac'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
