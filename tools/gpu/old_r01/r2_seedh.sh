mkdir -p gpurun_out
for L in libfic_b200.so libfic_b200_s0.so; do
for c in cfg2 cfg3; do
FIC_LIB=$PWD/paper_1404_0774_b200/$L timeout 600 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/b.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('$L $c', round(d['ms_per_step'],4), d['survivors_per_level'])"
done; done
