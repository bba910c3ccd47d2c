# round bench set: default bench (cfg2, with CPU baseline), other configs, reference arm,
# ncu launch list of the bench command, ncu --set full of the full-level scan (traffic)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; tail -c 3000 gpurun_out/bench_cfg2.json
timeout 600 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2>&1
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
for c in cfg2 cfg3; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/scan_full_$c -f python tools/encode_once.py $c > gpurun_out/ncu_$c.log 2>&1
done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 4 --launch-count 1 -o gpurun_out/scan_full_cfg4 -f python tools/encode_once.py cfg4 > gpurun_out/ncu_cfg4.log 2>&1
echo done
