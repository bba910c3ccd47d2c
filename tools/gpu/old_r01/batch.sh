# batched volume encode throughput vs per-slice encodes
mkdir -p gpurun_out
for c in 8 16 32 64; do FIC_BATCH_CHUNK=$c timeout 300 python tools/batch_timing.py 64 2>&1 | tail -3; done
