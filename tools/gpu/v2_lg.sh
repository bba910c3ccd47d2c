mkdir -p gpurun_out
for v in "FIC_LANE_GROUP=1" "FIC_LANE_GROUP=2" "FIC_LANE_GROUP=4"; do
  env $v timeout 600 python -m pytest tests/test_gpu_encode.py -x -q -k "cfg2 or noise32 or selection" 2>&1 | tail -1
  for c in cfg2 cfg3; do
  env $v timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v2_lg_b.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_lg_b.json').read().strip().splitlines()[-1]); print('$c $v', round(d['ms_per_step'],4), 'scan', round(d['roofline']['kernel_ms'],4), d['survivors_per_level'])"
  done
done
