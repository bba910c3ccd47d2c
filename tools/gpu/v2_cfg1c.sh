k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "span" | cut -c1-60; }
C=cfg1; k X=0; k FIC_LEVELS=3; k FIC_LEVELS=2; k FIC_LEVELS=3 FIC_SEED=0; k FIC_LEVELS=2 FIC_SEED=0; k X=0
