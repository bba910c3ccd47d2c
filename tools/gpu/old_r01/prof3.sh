mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/scan4_cfg2_full -f python tools/encode_once.py cfg2 > gpurun_out/ncu_a.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 0 --launch-count 1 -o gpurun_out/scan4_cfg2_l64 -f python tools/encode_once.py cfg2 > gpurun_out/ncu_b.log 2>&1
echo done
