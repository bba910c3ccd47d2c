# A/B: whole-tile vote on the per-range maxima (FIC_COARSE=1) vs none, cheaper record appends
mkdir -p gpurun_out/v3
k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel\|expand\|span" | cut -c1-60; }
for C in cfg2 cfg3; do k FIC_COARSE=0; k FIC_COARSE=1; done
C=cfg4; k FIC_COARSE=1
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q -m gpu 2>&1 | tail -2
FIC_COARSE=1 timeout 900 python -m pytest tests/test_gpu_encode.py -x -q -m gpu -k "cfg2 or cfg3 or full" 2>&1 | tail -2
