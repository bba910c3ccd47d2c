k() { echo "== $C $L $*"; env FIC_LIB=$PWD/paper_1404_0774_b200/$L "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel\|eval_kernel\|span" | cut -c1-60; }
for C in cfg2 cfg3; do for L in libfic_b200.so libfic_b200_m2.so; do k X=0; done; L=libfic_b200.so; k FIC_EVAL_NOPRUNE=1; done
C=cfg3; L=libfic_b200.so; k FIC_F16SEL=1
C=cfg4; k X=0; k FIC_F16SEL=1
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q -m gpu 2>&1 | tail -2
FIC_F16SEL=1 timeout 900 python -m pytest tests/test_gpu_encode.py -x -q -m gpu 2>&1 | tail -2
