cd $GRAFT_REPO_ROOT
DGM_HO_K=4 DGM_HO_W=4 timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage3 --launch-skip 2 -c 1 -o gpurun_out/prof_stage3_C4_k4 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu24.log 2>&1
DGM_HO_K=1 DGM_HO_W=4 timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage3 --launch-skip 2 -c 1 -o gpurun_out/prof_stage3_C4_k1 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu24b.log 2>&1
tail -3 gpurun_out/ncu24.log
