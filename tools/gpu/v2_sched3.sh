k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel\|eval_kernel\|expand\|span" | cut -c1-60; }
C=cfg3
k X=0; k FIC_LEVELS=16,4; k FIC_LEVELS=32,8; k FIC_LEVELS=16,2; k FIC_LEVELS=128,16,4; k FIC_LANEBEST_MAX=200; k FIC_LANEBEST_MAX=200 FIC_LANE_GROUP=2; k FIC_LEVELS=64,8; k FIC_LEVELS=8
