# same-box A/B: base (1c6abb4) / new (full-level fp16 epilogue tests its tiles in pairs)
D=$PWD/paper_1404_0774_b200
k() { echo "== $C $1"; FIC_LIB=$D/libfic_b200$2.so timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel<[56]\|span" | cut -c1-62; }
for rep in 1 2 3; do for C in cfg2 cfg3; do k base _base; k new ""; done; done
C=cfg4; k base _base; k new ""
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
