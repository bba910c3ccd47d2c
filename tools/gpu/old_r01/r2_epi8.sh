mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q -k "coarse or cfg4 or cfg2" > gpurun_out/pytest_e8.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_e8.log
for e in 1 0 1 0; do FIC_EPI8=$e timeout 600 python tools/flag_timing.py cfg4 0 2>&1 | grep -v Warn | tail -1 | sed "s/^/EPI8=$e /"; done
