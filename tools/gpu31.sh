cd $GRAFT_REPO_ROOT
DGM_ENGINE=dense timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches_dense_C5.csv python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu31.log 2>&1
DGM_ENGINE=dense timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel --launch-skip 2 -c 1 -o gpurun_out/prof_gemm0_C4 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu31b.log 2>&1
tail -2 gpurun_out/ncu31b.log
