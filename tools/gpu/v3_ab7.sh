# same-box A/B of the fp16 hit-first selection (cfg3 sparse levels): v0 branch per range (default),
# v1 no branch, v2 warp max inside the branch; then the GPU suite on the default build
D=$PWD/paper_1404_0774_b200
k() { echo "== $C $1"; FIC_LIB=$D/libfic_b200$2.so timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel<7\|span" | cut -c1-62; }
for rep in 1 2; do C=cfg3; k v0 ""; k v1 _v1; k v2 _v2; done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
