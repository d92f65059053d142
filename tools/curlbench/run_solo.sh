cd $GRAFT_REPO_ROOT/tools/curlbench
o=$GRAFT_REPO_ROOT/gpurun_out/${1:-solo}; mkdir -p $o
for v in cb_pair cb_solo cb_pair cb_solo; do timeout 120 ./$v >> $o/times.txt 2>&1; echo "$v" >> $o/times.txt; done
cat $o/times.txt
