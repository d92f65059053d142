cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lane_stage --launch-skip 4 -c 1 -o gpurun_out/prof_lane_C2 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu38.log 2>&1
tail -1 gpurun_out/ncu38.log
