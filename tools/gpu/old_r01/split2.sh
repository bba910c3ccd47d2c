mkdir -p gpurun_out
for f in 0 8 64; do
  FIC_SCAN=1cta FIC_DEBUG=$f timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/split2_cfg2_$f.csv -k regex:scan python tools/encode_once.py cfg2 1 > /dev/null 2>&1
done
echo done
