# grouped record reservation per tile + compile-time debug switches: timelines and the encoder's GPU tests
k() { echo "== $C"; timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel\|expand\|span" | cut -c1-62; }
for C in cfg2 cfg3 cfg2 cfg3; do k; done
C=cfg4; k
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
