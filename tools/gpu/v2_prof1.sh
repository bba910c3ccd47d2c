# GPU tests (FIC1 on device, multirank) + ncu --set full of every kernel of one warm cfg2 encode
# (cache-control none: L2 warm as in the timed steps) + the cfg3 full-level scan
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/v2_pytest.log 2>&1; tail -3 gpurun_out/v2_pytest.log
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none --launch-skip 40 --launch-count 20 -o gpurun_out/v2_cfg2_all -f python tools/encode_once.py cfg2 4 > gpurun_out/v2_ncu_cfg2_all.log 2>&1
tail -3 gpurun_out/v2_ncu_cfg2_all.log
