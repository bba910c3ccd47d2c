mkdir -p gpurun_out
for f in 0 8 16 24; do
  FIC_DEBUG=$f timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/split_$f.csv -k regex:scan_kernel python tools/encode_once.py ${CFG:-cfg4} 1 > /dev/null 2>&1
done
echo done
