# Time the curl variants (p=10, C5 size) and collect their stall breakdown. Run from repo root on the GPU box.
cd $GRAFT_REPO_ROOT/tools/curlbench
o=$GRAFT_REPO_ROOT/gpurun_out/${1:-cbv}; mkdir -p $o
for v in cb_*; do [ -x $v ] || continue; timeout 120 ./$v >> $o/times.txt 2>&1; echo "$v done" >> $o/times.txt; done
for v in cb_*; do [ -x $v ] || continue;
timeout 300 ncu --clock-control none -k regex:curl -s 2 -c 1 --metrics gpu__time_duration.sum,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --csv ./$v > $o/ncu_$v.csv 2>&1
done
cat $o/times.txt
