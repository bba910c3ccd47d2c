mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q -k "pair or cfg4 or stacked" > gpurun_out/pytest_pair.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_pair.log
timeout 1000 python tools/flag_timing.py cfg4 0 2>&1 | grep -v Warn
FIC_SCAN=pair timeout 1000 python tools/flag_timing.py cfg4 0 128 2>&1 | grep -v Warn
FIC_SCAN=pair timeout 1000 python tools/flag_timing.py cfg2 0 2>&1 | grep -v Warn
