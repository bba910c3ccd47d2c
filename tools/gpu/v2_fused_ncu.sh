mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:scan_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/v2_fused_scan -f python tools/encode_once.py cfg2 3 > gpurun_out/v2_ncu_fused.log 2>&1
tail -2 gpurun_out/v2_ncu_fused.log
