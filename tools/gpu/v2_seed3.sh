k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "seed\|scan_kernel\|eval_kernel\|span" | cut -c1-60; }
C=cfg2; k X=0; k FIC_SEED=1; k FIC_SEED=3; k FIC_SEED=1 FIC_LEVELS=4
C=cfg3; k X=0; k FIC_SEED=1
