k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "span" | cut -c1-60; }
C=cfg1; k X=0; C=cfg2; k X=0
timeout 600 python bench.py --config cfg1 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/v2_b1.json 2>&1; tail -1 gpurun_out/v2_b1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1', round(d['ms_per_step'],4), round(d['e2e']['encode_ms_per_image'],4))"
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
