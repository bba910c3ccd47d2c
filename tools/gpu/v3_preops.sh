# first-level range operands in the pool launch (FIC_PREOPS), 8-byte range-row loads in the
# evaluation, scan-alone roofline timing; full GPU suite
mkdir -p gpurun_out/v3
k() { echo "== $C $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep -v Warn | grep -v warn_once | cut -c1-62; }
for C in cfg2 cfg1; do k FIC_PREOPS=0; k FIC_PREOPS=1; done
C=cfg3; k FIC_PREOPS=1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/v3/pytest_gpu.log 2>&1; tail -2 gpurun_out/v3/pytest_gpu.log
FIC_PREOPS=0 timeout 900 python -m pytest tests/test_gpu_encode.py -x -q -m gpu -k "cfg2" 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/v3/bench_cfg2.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/v3/bench_cfg2.json').read().strip().splitlines()[-1]); r=d['roofline']; print('cfg2', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['encode_ms_per_image'],4), 'scan', round(r['kernel_ms'],4), round(r['frac'],3), 'with expand', round(r['scan_expand_ms'],4), round(r['frac_with_expand'],3), 'pool', d['pool']['frac'], 'launches', d['gpu_launches'])"
