mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_cli.py -x -q > gpurun_out/pytest_decode.log 2>&1; echo "decode tests rc=$?"; tail -1 gpurun_out/pytest_decode.log
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_cfg2.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg2.json').read().strip().splitlines()[-1]); print('cfg2', d['ms_per_step'], d['decoder']['ms'], d['decoder']['frac'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"decode_mean" -c 2 --csv --log-file gpurun_out/decode_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
