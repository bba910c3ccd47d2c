k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel\|eval_kernel\|expand\|span" | cut -c1-60; }
for C in cfg2 cfg3; do k X=0; k FIC_F16ACC=0; done
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
