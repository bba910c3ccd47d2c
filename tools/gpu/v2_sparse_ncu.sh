mkdir -p gpurun_out/ncu; O=gpurun_out/ncu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 4 --launch-count 1 -o $O/sp3 -f python tools/encode_once.py cfg3 2 > /dev/null 2>&1
python tools/ncu_summary.py $O/sp3.ncu-rep > $O/r02_ncu_scan_sparse_cfg3.txt 2>&1
python tools/ncu_lines.py $O/sp3.ncu-rep > $O/r02_ncu_scan_sparse_cfg3_lines.txt 2>&1
python tools/ncu_raw_grep.py $O/sp3.ncu-rep 'smsp__average_warps_issue_stalled_.*_per_issue_active.ratio$' 'sm__inst_executed_pipe_.*avg.pct_of_peak_sustained_active$' >> $O/r02_ncu_scan_sparse_cfg3.txt
rm -f $O/sp3.ncu-rep
head -30 $O/r02_ncu_scan_sparse_cfg3.txt; head -40 $O/r02_ncu_scan_sparse_cfg3_lines.txt
