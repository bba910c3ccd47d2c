for L in libfic_b200.so libfic_pb64.so libfic_pb32.so; do
  echo "== $L"
  FIC_LIB=$PWD/paper_1404_0774_b200/$L timeout 600 python tools/kineto_gaps.py cfg2 2>&1 | grep -E "pool_v3|span"
  FIC_LIB=$PWD/paper_1404_0774_b200/$L timeout 600 python tools/kineto_gaps.py cfg4 2>&1 | grep -E "pool_v3|span"
done
FIC_LIB=$PWD/paper_1404_0774_b200/libfic_pb32.so timeout 900 python -m pytest tests/test_gpu_encode.py -q -x 2>&1 | tail -1
