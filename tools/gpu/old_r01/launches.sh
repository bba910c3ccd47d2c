mkdir -p gpurun_out
for c in cfg2 cfg3 cfg4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$c.csv python tools/encode_once.py $c 2 > /dev/null 2>&1
done
echo done
