timeout 300 python tools/e2e_breakdown.py cfg2 2>&1 | tail -13
for v in 1 0 1 0; do if [ $v = 1 ]; then E=FIC_STATUS_COPY=1; else E=X=0; fi; env $E timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/v2_b.json 2>&1; tail -1 gpurun_out/v2_b.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$E', round(d['ms_per_step'],4), round(d['e2e']['encode_ms_per_image'],4))"; done
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
