mkdir -p gpurun_out
timeout 800 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/scan_l1_cfg2 -f python tools/encode_once.py cfg2 2 > gpurun_out/ncu_l1.log 2>&1; echo rc=$?
timeout 800 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 5 --launch-count 1 -o gpurun_out/scan_full_cfg3 -f python tools/encode_once.py cfg3 2 > gpurun_out/ncu_c3.log 2>&1; echo rc=$?
timeout 800 ncu --set full --import-source on --clock-control none -k regex:decode_mean --launch-skip 2 --launch-count 1 -o gpurun_out/decode_mean_v3 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_dec3.log 2>&1; echo rc=$?
