cd $GRAFT_REPO_ROOT/tools/curlbench
ncu --set full --import-source on --clock-control none -k regex:curl -s 2 -c 1 -o prof ./cb_imm > ncu.log 2>&1
ncu -i prof.ncu-rep --page source --csv > source.csv
ncu -i prof.ncu-rep --page raw --csv > raw.csv
mkdir -p $GRAFT_REPO_ROOT/gpurun_out/cb4; cp source.csv raw.csv $GRAFT_REPO_ROOT/gpurun_out/cb4/
