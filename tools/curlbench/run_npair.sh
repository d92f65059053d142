cd $GRAFT_REPO_ROOT/tools/curlbench
o=$GRAFT_REPO_ROOT/gpurun_out/${1:-np}; mkdir -p $o
for v in cb_np1 cb_np2 cb_np4; do timeout 120 ./$v >> $o/times.txt 2>&1; echo "$v" >> $o/times.txt; done
cat $o/times.txt
