# batched volume encode: GPU tests + throughput
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for c in 8 16 32 64; do FIC_BATCH_CHUNK=$c timeout 300 python tools/batch_timing.py 64 2>&1 | tail -3; done
