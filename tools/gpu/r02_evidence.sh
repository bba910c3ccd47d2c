# round-2 evidence set: GPU suite, smoke, bench lines (all configs + reference arm + 2 ranks on one
# GPU), ncu launch list of the default bench, ncu --set full of the dominant kernels, kineto timelines
mkdir -p gpurun_out/ev
O=gpurun_out/ev
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python bench.py --impl reference > $O/bench_reference_cfg2.json 2>&1
timeout 900 python bench.py --config cfg3 > $O/bench_cfg3.json 2>&1
timeout 1200 python bench.py --config cfg4 --steps 5 --warmup 3 > $O/bench_cfg4.json 2>&1
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 3 > $O/bench_cfg5.json 2>&1
timeout 900 python bench.py --config cfg1 > $O/bench_cfg1.json 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg4_2rank.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 python tools/kineto_gaps.py cfg2 > $O/kineto_cfg2.txt 2>&1
timeout 600 python tools/kineto_gaps.py cfg4 > $O/kineto_cfg4.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 3 --launch-count 2 -o $O/scan_cfg2 -f python tools/encode_once.py cfg2 3 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 3 --launch-count 3 -o $O/scan_cfg3 -f python tools/encode_once.py cfg3 2 > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 4 --launch-count 1 -o $O/scan_cfg4 -f python tools/encode_once.py cfg4 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pool_v3 --launch-skip 1 --launch-count 1 -o $O/pool_cfg2 -f python tools/encode_once.py cfg2 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pool_v3 --launch-count 1 -o $O/pool_cfg4 -f python tools/encode_once.py cfg4 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --cache-control none -k regex:eval_kernel --launch-skip 2 --launch-count 2 -o $O/eval_cfg2 -f python tools/encode_once.py cfg2 3 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_means --launch-skip 5 --launch-count 1 -o $O/decode -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for f in $O/bench_*.json; do echo $f; tail -1 $f | cut -c1-300; done
