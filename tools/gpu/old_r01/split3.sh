mkdir -p gpurun_out
for m in 1cta pair; do
for c in cfg2 cfg4; do
for f in 0 8; do
  FIC_SCAN=$m FIC_DEBUG=$f timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/split3_${m}_${c}_$f.csv -k regex:scan python tools/encode_once.py $c 1 > /dev/null 2>&1
done; done; done
echo done
