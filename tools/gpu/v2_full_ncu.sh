mkdir -p gpurun_out/ncu; O=gpurun_out/ncu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 3 --launch-count 1 -o $O/f2 -f python tools/encode_once.py cfg2 3 > /dev/null 2>&1
python tools/ncu_summary.py $O/f2.ncu-rep > $O/r02_ncu_scan_full_cfg2.txt 2>&1
python tools/ncu_lines.py $O/f2.ncu-rep > $O/r02_ncu_scan_full_cfg2_lines.txt 2>&1
python tools/ncu_raw_grep.py $O/f2.ncu-rep 'smsp__average_warps_issue_stalled_.*_per_issue_active.ratio$' 'sm__inst_executed_pipe_.*avg.pct_of_peak_sustained_active$' >> $O/r02_ncu_scan_full_cfg2.txt
rm -f $O/f2.ncu-rep
head -12 $O/r02_ncu_scan_full_cfg2.txt; grep -E "Grid|Registers|tensor|pipe_alu|pipe_fma|pipe_adu" $O/r02_ncu_scan_full_cfg2.txt; head -45 $O/r02_ncu_scan_full_cfg2_lines.txt
