# round-2 evidence pass 1: multi-rank test, benches (cfg2 + reference arm, cfg3, cfg4 at 1 and
# 2 ranks on one GPU, cfg5), ncu of the pool builder (cfg2, cfg4)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -q > gpurun_out/v2_multirank.log 2>&1; tail -2 gpurun_out/v2_multirank.log
timeout 600 python bench.py > gpurun_out/v2_bench_cfg2.json 2> gpurun_out/v2_bench_cfg2.err; tail -c 400 gpurun_out/v2_bench_cfg2.err
timeout 900 python bench.py --impl reference > gpurun_out/v2_bench_ref.json 2>&1
timeout 600 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/v2_bench_cfg3.json 2>&1
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 > gpurun_out/v2_bench_cfg4.json 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/v2_bench_cfg4_2rank.json 2>&1
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/v2_bench_cfg5.json 2>&1
for c in cfg2 cfg4; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:pool_v3 --launch-count 1 -o gpurun_out/v2_pool_$c -f python tools/encode_once.py $c > gpurun_out/v2_ncu_pool_$c.log 2>&1
done
for f in gpurun_out/v2_bench_*.json; do echo $f; cut -c1-400 $f; done
