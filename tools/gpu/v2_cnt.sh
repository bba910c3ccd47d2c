k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep -v Warn | grep -v warn_once | cut -c1-60 | tail -13; }
C=cfg2; k X=0
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/v2_b.json 2>&1; tail -1 gpurun_out/v2_b.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['e2e']['encode_ms_per_image'],4))"; done
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
