# quantisation screen in the scan epilogue: parity + A/B timing (FIC_DEBUG=256 disables it)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encode.py tests/test_gpu_smoke_api.py -x -q > gpurun_out/pytest_enc.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_enc.log
for f in 0 256; do
for c in cfg2 cfg3; do
FIC_DEBUG=$f timeout 600 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/bench_${c}_$f.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_${c}_$f.json').read().strip().splitlines()[-1]); print('$c flags $f', d['ms_per_step'], 'scan', d['roofline']['kernel_ms'], 'matcher', d['roofline']['matcher_ms'], d['survivors_per_level'])"
done
FIC_DEBUG=$f timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_$f.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg4_$f.json').read().strip().splitlines()[-1]); print('cfg4 flags $f', d['ms_per_step'], 'scan', d['roofline']['kernel_ms'], d['roofline']['frac'], d['survivors_per_level'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
