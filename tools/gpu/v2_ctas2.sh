run() { c=$1; lib=$2; FIC_LIB=$PWD/paper_1404_0774_b200/$lib timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v2_sc.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_sc.json').read().strip().splitlines()[-1]); print('$c $lib', round(d['ms_per_step'],4), 'matcher', round(d['roofline']['matcher_ms'],4))"; }
FIC_LIB=$PWD/paper_1404_0774_b200/libfic_b200_c2.so timeout 600 python -m pytest tests/test_gpu_encode.py -x -q -m gpu 2>&1 | tail -15
for k in 1 2; do for l in libfic_b200.so libfic_b200_c2.so; do run cfg2 $l; done; done
for k in 1 2; do for l in libfic_b200.so libfic_b200_c2.so; do run cfg3 $l; done; done
for l in libfic_b200.so libfic_b200_c2.so; do run cfg4 $l; done
