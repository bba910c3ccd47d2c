# full GPU test suite + smoke + decoder/scan ncu of the current tree
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 800 ncu --set full --import-source on --clock-control none -k regex:decode_mean --launch-skip 2 --launch-count 1 -o gpurun_out/decode_mean_v1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_dec.log 2>&1; echo ncu rc=$?
timeout 800 ncu --set full --import-source on --clock-control none -k regex:eval_kernel --launch-skip 3 --launch-count 3 -o gpurun_out/eval_cfg2_v1 -f python tools/encode_once.py cfg2 2 > gpurun_out/ncu_eval.log 2>&1; echo ncu rc=$?
