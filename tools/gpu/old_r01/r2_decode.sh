# tiled decoder parity + bench; pair-mode scan comparison
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/pytest_decode.log 2>&1; echo "decode tests rc=$?"; tail -3 gpurun_out/pytest_decode.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg2.json').read().strip().splitlines()[-1]); print('cfg2', d['ms_per_step'], d['roofline']['kernel_ms'], d['decoder'])"
FIC_DECODE_FLAT=1 timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_cfg2_flat.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg2_flat.json').read().strip().splitlines()[-1]); print('flat decoder', d['decoder'])"
FIC_SCAN=pair timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2_pair.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg2_pair.json').read().strip().splitlines()[-1]); print('cfg2 pair', d['ms_per_step'], d['roofline']['kernel_ms'])"
FIC_SCAN=pair timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_pair.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg4_pair.json').read().strip().splitlines()[-1]); print('cfg4 pair', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:decode -c 20 --csv --log-file gpurun_out/decode_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
