for L in "64,8" "64,16,4" "64,8,2" "32,8,2" "16,4"; do
  FIC_LEVELS=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],4), d['survivors_per_level'])"
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', round(d['ms_per_step'],4), d['survivors_per_level'])"
for L in "4096,512,64,8" "4096,512,64,16,4"; do
  FIC_LEVELS=$L timeout 600 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline 2>/tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 $L', round(d['ms_per_step'],3), d['survivors_per_level'])"
done
tail -5 /tmp/err.txt
