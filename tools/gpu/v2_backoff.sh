k() { echo "== $C $L"; FIC_LIB=$PWD/paper_1404_0774_b200/$L timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel\|span" | cut -c1-60; }
for C in cfg2 cfg3; do for L in libfic_b200.so libfic_b200_bo32.so libfic_b200_bo128.so libfic_b200.so; do k; done; done
