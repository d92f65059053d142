# Per-kernel times of one dense stage (ncu launch list; cold cache per replay)
cd $GRAFT_REPO_ROOT
cfg=${1:-C5}
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm|dense_flux" -c 6 --csv --log-file gpurun_out/launches_dense_$cfg.csv python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_dl.log 2>&1
