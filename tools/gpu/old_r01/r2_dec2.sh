mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_cli.py -x -q 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/b.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('cfg2 decoder', d['decoder']['ms'], d['decoder']['frac'])"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"decode_mean" -c 2 --csv --log-file gpurun_out/decode_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; grep -E "duration|inst_executed" gpurun_out/decode_launches.csv | cut -d, -f12- | head -4
