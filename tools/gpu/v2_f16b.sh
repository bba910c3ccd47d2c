k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel\|eval_kernel\|expand\|span" | cut -c1-60; }
for C in cfg2 cfg3 cfg1; do k FIC_F16ACC=0; k FIC_F16ACC=1; done
C=cfg4; k X=0
FIC_F16ACC=1 timeout 600 python -m pytest tests/test_gpu_encode.py -x -q -m gpu 2>&1 | tail -3
