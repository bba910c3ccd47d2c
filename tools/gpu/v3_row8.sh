# A/B on one box: 8-byte range-row loads in the evaluation (default) vs 4-byte (FIC_EVAL_ROW8=0 build)
k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "eval_kernel\|span" | cut -c1-62; }
for rep in 1 2; do for C in cfg2 cfg1; do k FIC_LIB=$PWD/paper_1404_0774_b200/libfic_b200_row4.so; k FIC_LIB=$PWD/paper_1404_0774_b200/libfic_b200.so; done; done
for v in row4 ""; do
  f=$PWD/paper_1404_0774_b200/libfic_b200${v:+_$v}.so
  FIC_LIB=$f timeout 600 python bench.py --no-cpu-baseline --steps 40 --warmup 10 > gpurun_out/v3_b.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v3_b.json').read().strip().splitlines()[-1]); print('cfg2 $v', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['encode_ms_per_image'],4))"
done
