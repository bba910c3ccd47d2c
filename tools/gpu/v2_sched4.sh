k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel\|eval_kernel\|span" | cut -c1-60; }
C=cfg2
k X=0; k FIC_LEVELS=3; k FIC_LEVELS=2 FIC_LANEBEST_MAX=64; k FIC_LEVELS=5; k FIC_LEVELS=6; k FIC_LEVELS=16,4; k FIC_LEVELS=32,3; k X=0
