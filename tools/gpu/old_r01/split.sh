mkdir -p gpurun_out
for c in cfg2 cfg4; do
for f in 0 8 16 24; do
  FIC_DEBUG=$f timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/split_${c}_$f.csv -k regex:scan python tools/encode_once.py $c 1 > /dev/null 2>&1
done
done
echo done
