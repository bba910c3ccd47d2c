k() { echo "== $C $L"; FIC_LIB=$PWD/paper_1404_0774_b200/$L timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "eval_kernel<[0-9]*, 0>\|span" | cut -c1-60; }
for C in cfg2 cfg3 cfg4; do for L in libfic_b200.so libfic_b200_r4.so libfic_b200_r3.so libfic_b200.so; do k; done; done
FIC_LIB=$PWD/paper_1404_0774_b200/libfic_b200_r4.so timeout 900 python -m pytest tests/test_gpu_encode.py -x -q -m gpu 2>&1 | tail -2
