k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel\|eval_kernel\|span" | cut -c1-60; }
C=cfg3; for a in 0 0.7 0.85 0.95 1.0; do k FIC_SEL_ALPHA=$a; done
C=cfg4; for a in 0 0.85 0.95; do k FIC_SEL_ALPHA=$a; done
