mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --cache-control none -k regex:eval_kernel --launch-skip 6 --launch-count 2 -o gpurun_out/v2_eval -f python tools/encode_once.py cfg2 5 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --cache-control none -k regex:scan_kernel --launch-skip 7 --launch-count 1 -o gpurun_out/v2_scanfull -f python tools/encode_once.py cfg2 5 > /dev/null 2>&1
echo done
