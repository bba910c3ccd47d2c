# diag counters, timing split and ncu captures of the current matcher (round 1 baseline)
mkdir -p gpurun_out
python tools/diag.py cfg2 cfg3 cfg4 > gpurun_out/diag.log 2>&1
FIC_PREPASS=0 python tools/diag.py cfg2 > gpurun_out/diag_noprepass.log 2>&1
python tools/timing_split.py cfg2 cfg3 cfg4 > gpurun_out/split.log 2>&1
python tools/trace.py cfg2 > gpurun_out/trace_cfg2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:matcher_tc --launch-skip 1 --launch-count 1 -o gpurun_out/mtc_cfg2 -f python tools/encode_once.py cfg2 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:seed_kernel --launch-count 1 -o gpurun_out/seed_cfg2 -f python tools/encode_once.py cfg2 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pool_build --launch-count 1 -o gpurun_out/pool_cfg4 -f python tools/encode_once.py cfg4 > gpurun_out/ncu3.log 2>&1
echo done
