k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "range_op\|span" | cut -c1-60; }
for C in cfg2 cfg3 cfg1; do k X=0; done
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/e2e_breakdown.py cfg2 2>&1 | tail -40
