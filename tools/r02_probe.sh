# Round-2 probe: smoke, GPU tests, default bench (C5), hybrid C5 bench, ncu of the hybrid curl kernel.
cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-probe}; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $o/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; tail -2 $o/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > $o/pytest_gpu.log 2>&1; tail -2 $o/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $o/bench_default.json 2> $o/bench_default.err; tail -1 $o/bench_default.json | cut -c1-300
DGM_ENGINE=hybrid timeout 900 python bench.py --no-cpu-baseline --no-e2e > $o/bench_C5_hybrid.json 2> $o/bench_C5_hybrid.err; tail -1 $o/bench_C5_hybrid.json | cut -c1-300
DGM_ENGINE=hybrid timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"gemm|dense_flux|curl" -c 8 --csv --log-file $o/launches_stage_C5_hybrid.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_stage.log 2>&1
DGM_ENGINE=hybrid timeout 900 ncu --set full --import-source on --clock-control none -k regex:curl -s 1 -c 1 -o $o/curl_C5 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_curl.log 2>&1
ls $o
