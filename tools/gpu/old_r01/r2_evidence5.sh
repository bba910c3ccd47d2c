# round evidence v16: smoke, bench lines (cfg2 default with CPU baseline, cfg3, cfg4, cfg5), reference arm,
# launch list of the default bench, ncu --set full of the cfg4 full-level scan (fp16 accumulator, mode 6)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; tail -c 300 gpurun_out/bench_cfg2.json
timeout 600 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2>&1
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2>&1
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --slices 64 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1; echo ncu rc=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 4 --launch-count 1 -o gpurun_out/scan_full_cfg4_v16 -f python tools/encode_once.py cfg4 > gpurun_out/ncu_cfg4.log 2>&1; echo ncu rc=$?
timeout 500 python tools/kineto_gaps.py cfg4 > gpurun_out/kineto_cfg4.txt 2>&1; tail -1 gpurun_out/kineto_cfg4.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
