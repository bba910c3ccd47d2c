# pool launch with the range pass on 16 lanes per range (timelines) + GPU suite
for C in cfg2 cfg3 cfg2; do echo "== $C"; timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep -v -i warn | cut -c1-62; done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/v3_pool_b.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/v3_pool_b.json').read().strip().splitlines()[-1]); r=d['roofline']; print('cfg2', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['encode_ms_per_image'],4), 'scan', round(r['kernel_ms'],4), round(r['frac'],3), 'pool', round(d['pool']['ms']*1e3,2), d['pool']['frac'])"
