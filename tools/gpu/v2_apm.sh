k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel\|eval_kernel\|span" | cut -c1-60; }
for C in cfg2 cfg3; do k X=0; k X=1; done
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/v2_b.json 2>&1; tail -1 gpurun_out/v2_b.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['e2e']['encode_ms_per_image'],4))"
timeout 900 python -m pytest tests/test_gpu_encode.py -x -q -m gpu 2>&1 | tail -2
