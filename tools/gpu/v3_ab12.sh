# same-box A/B: base (fa59342) / new (fp32 selection tags in registers), cfg4 sparse levels
D=$PWD/paper_1404_0774_b200
k() { echo "== $C $1"; FIC_LIB=$D/libfic_b200$2.so timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel<2\|span" | cut -c1-62; }
for rep in 1 2; do C=cfg4; k base _base; k new ""; done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
