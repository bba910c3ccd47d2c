mkdir -p gpurun_out/ncu; O=gpurun_out/ncu
for c in cfg2:4:3 cfg3:5:2; do
  IFS=: read cfg skip reps <<< "$c"
  timeout 900 ncu --set full --clock-control none -k regex:scan_kernel --launch-skip $skip --launch-count 1 -o $O/st_$cfg -f python tools/encode_once.py $cfg $reps > /dev/null 2>&1
  echo "=== $cfg"
  python tools/ncu_raw_grep.py $O/st_$cfg.ncu-rep 'smsp__average_warps_issue_stalled_.*_per_issue_active.ratio$' 'sm__inst_executed_pipe_.*pct_of_peak_sustained_active$' 'sm__pipe_.*cycles_active.*pct_of_peak_sustained_active$' 'smsp__issue_active.avg.pct' 'gpu__time_duration.sum'
  rm -f $O/st_$cfg.ncu-rep
done
