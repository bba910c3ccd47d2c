mkdir -p gpurun_out
timeout 300 python tools/kineto_gaps.py cfg2 > gpurun_out/v2_kineto_cfg2.txt 2>&1
timeout 300 python tools/kineto_gaps.py cfg3 > gpurun_out/v2_kineto_cfg3.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pool_v3 --launch-count 1 -o gpurun_out/v2_pool2_cfg4 -f python tools/encode_once.py cfg4 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_mean --launch-skip 5 --launch-count 1 -o gpurun_out/v2_decode -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/v2_kineto_cfg2.txt | grep -v Warn
