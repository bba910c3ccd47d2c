k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep -v Warn | grep -v warn_once | cut -c1-60; }
for C in cfg2 cfg3; do k X=0; done
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v2_b.json 2>&1; tail -1 gpurun_out/v2_b.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['encode_ms_per_image'])"
