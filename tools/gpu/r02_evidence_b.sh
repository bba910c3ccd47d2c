# round-2 evidence, part B: ncu --set full of the dominant kernels, summarised on the box (the
# reports themselves are kept only when small)
mkdir -p gpurun_out/ncu
O=${NCU_DIR:-gpurun_out/ncu}; mkdir -p $O
cap() {  # name, kernel regex, ncu extra args, command...
  n=$1; k=$2; x=$3; shift 3
  timeout 1200 ncu --set full --import-source on --clock-control none $x -k regex:$k -o $O/$n -f "$@" > /dev/null 2>&1
  python tools/ncu_summary.py $O/$n.ncu-rep > $O/$n.txt 2>&1
  python tools/ncu_lines.py $O/$n.ncu-rep > $O/${n}_lines.txt 2>&1
  python tools/ncu_raw_grep.py $O/$n.ncu-rep 'smsp__average_warps_issue_stalled_.*_per_issue_active.ratio$' \
    'sm__inst_executed_pipe_.*avg.pct_of_peak_sustained_active$' >> $O/$n.txt 2>&1
  sz=$(stat -c %s $O/$n.ncu-rep 2>/dev/null || echo 0); [ "$sz" -gt 8000000 ] && rm -f $O/$n.ncu-rep
}
cap scan_full_cfg2 scan_kernel "--launch-skip 3 --launch-count 1" python tools/encode_once.py cfg2 3
cap scan_sparse_cfg2 scan_kernel "--launch-skip 2 --launch-count 1" python tools/encode_once.py cfg2 3
cap scan_full_cfg3 scan_kernel "--launch-skip 5 --launch-count 1" python tools/encode_once.py cfg3 2
cap scan_sparse_cfg3 scan_kernel "--launch-skip 4 --launch-count 1" python tools/encode_once.py cfg3 2
cap scan_full_cfg4 scan_kernel "--launch-skip 4 --launch-count 1" python tools/encode_once.py cfg4
cap pool_cfg2 pool_v3 "--launch-skip 1 --launch-count 1" python tools/encode_once.py cfg2 2
cap pool_cfg4 pool_v3 "--launch-count 1" python tools/encode_once.py cfg4
cap eval_sparse_cfg2 eval_kernel "--cache-control none --launch-skip 2 --launch-count 1" python tools/encode_once.py cfg2 3
cap eval_full_cfg2 eval_kernel "--cache-control none --launch-skip 3 --launch-count 1" python tools/encode_once.py cfg2 3
cap decode_cfg2 decode_means "--launch-skip 5 --launch-count 1" python bench.py --steps 2 --warmup 3 --no-cpu-baseline
du -sh $O; ls -la $O
