# same-box A/B: base (9024c04, 64-thread record blocks) / new (32-thread record blocks)
D=$PWD/paper_1404_0774_b200
k() { echo "== $C $1"; FIC_LIB=$D/libfic_b200$2.so timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "record_kernel\|span" | cut -c1-62; }
for rep in 1 2 3; do for C in cfg2 cfg3; do k base _base; k new ""; done; done
timeout 900 python -m pytest tests/test_gpu_encode.py -m gpu -q -x 2>&1 | tail -2
