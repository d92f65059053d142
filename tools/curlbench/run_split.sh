cd $GRAFT_REPO_ROOT/tools/curlbench
o=$GRAFT_REPO_ROOT/gpurun_out/${1:-split}; mkdir -p $o
for v in cb_s4 cb_s3 cb_s2 cb_s4 cb_s3 cb_s2; do timeout 120 ./$v >> $o/times.txt 2>&1; echo "$v" >> $o/times.txt; done
cat $o/times.txt
