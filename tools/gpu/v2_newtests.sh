timeout 900 python -m pytest tests/test_gpu_f16acc.py tests/test_gpu_encode.py -x -q -m gpu -k "f16_accumulator_matches or near_threshold" 2>&1 | tail -15
k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "record\|span" | cut -c1-60; }
C=cfg2; k X=0; C=cfg3; k X=0
