k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "span" | cut -c1-60; }
C=cfg2; for i in 1 2; do k X=0; k FIC_LEVELS=3; done
C=cfg3; k X=0; k FIC_LEVELS=32,3; k FIC_LEVELS=24,4; k FIC_LEVELS=48,4; k X=0
for L in X=0 FIC_LEVELS=3 X=0 FIC_LEVELS=3; do env $L timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/v2_b.json 2>&1; tail -1 gpurun_out/v2_b.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],4), round(d['e2e']['encode_ms_per_image'],4))"; done
