# round-2 evidence, part A (small outputs): GPU suite, smoke, bench lines, launch list, timelines
mkdir -p gpurun_out/ev
O=${EV_DIR:-gpurun_out/ev}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python bench.py --impl reference > $O/bench_reference_cfg2.json 2>&1
timeout 900 python bench.py --config cfg3 > $O/bench_cfg3.json 2>&1
timeout 1200 python bench.py --config cfg4 --steps 5 --warmup 3 > $O/bench_cfg4.json 2>&1
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 3 > $O/bench_cfg5.json 2>&1
timeout 900 python bench.py --config cfg1 > $O/bench_cfg1.json 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg4_2rank.json 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_cfg5_2rank.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 python tools/kineto_gaps.py cfg2 > $O/kineto_cfg2.txt 2>&1
timeout 600 python tools/kineto_gaps.py cfg3 > $O/kineto_cfg3.txt 2>&1
timeout 600 python tools/kineto_gaps.py cfg4 > $O/kineto_cfg4.txt 2>&1
du -sh $O
