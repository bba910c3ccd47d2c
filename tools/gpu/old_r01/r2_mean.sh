# mean-raster decoder parity + bench; ncu of the current scan (cfg2 full level)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/pytest_decode.log 2>&1; echo "decode tests rc=$?"; tail -3 gpurun_out/pytest_decode.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg2.json').read().strip().splitlines()[-1]); print('cfg2', d['ms_per_step'], d['roofline']['kernel_ms'], d['decoder'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode|mean" -c 6 --csv --log-file gpurun_out/decode_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
timeout 800 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 5 --launch-count 1 -o gpurun_out/scan_full_cfg2_v6 -f python tools/encode_once.py cfg2 2 > gpurun_out/ncu_cfg2_v6.log 2>&1; echo ncu rc=$?
