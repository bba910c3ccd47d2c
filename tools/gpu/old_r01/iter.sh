# quick iteration: GPU tests, survivor diagnostics, short benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
FIC_DEBUG=4 timeout 300 python tools/diag.py cfg1 cfg2 cfg3 cfg4 2>&1 | tail -12
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2>&1; cat gpurun_out/bench_cfg2.json | cut -c1-1500
timeout 300 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2>&1; cut -c1-600 gpurun_out/bench_cfg3.json
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2>&1; cut -c1-600 gpurun_out/bench_cfg4.json
for c in cfg2 cfg3 cfg4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$c.csv python tools/encode_once.py $c 2 > /dev/null 2>&1
done
