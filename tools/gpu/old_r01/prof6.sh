mkdir -p gpurun_out
FIC_DEBUG=24 timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan2 --launch-skip 3 --launch-count 1 -o gpurun_out/scan2_f24_cfg4 -f python tools/encode_once.py cfg4 > gpurun_out/ncu_a.log 2>&1
echo done
