k() { echo "== $L $*"; env FIC_LIB=$PWD/paper_1404_0774_b200/$L "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel" | cut -c1-60; }
for C in cfg2 cfg3; do for L in libfic_b200.so libfic_b200_c2.so; do k FIC_F16ACC=1; k FIC_F16ACC=1 FIC_DEBUG=8; done; done
