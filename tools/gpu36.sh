cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel --launch-skip 1 -c 1 -o gpurun_out/prof_gemmS4_C5 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu36.log 2>&1
tail -1 gpurun_out/ncu36.log
