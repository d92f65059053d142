cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stream_kernel --launch-skip 2 -c 1 -o gpurun_out/prof_stream_C4 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu28.log 2>&1
tail -2 gpurun_out/ncu28.log
