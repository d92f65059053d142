# Round-2 final measurement pass: smoke, GPU tests, bench lines (default C5, C2-C4), reference
# arm, FP64 peaks, launch list of the default bench, per-kernel stage metrics at C5.
cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-final}; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $o/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; tail -5 $o/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > $o/pytest_gpu.log 2>&1; tail -2 $o/pytest_gpu.log
timeout 120 ./tools/peaks/fp64_peaks > $o/fp64_peaks.txt 2>&1
timeout 900 python bench.py > $o/bench_default.json 2> $o/bench_default.err; tail -1 $o/bench_default.json | cut -c1-200
for c in C2 C3 C4; do timeout 600 python bench.py --config $c > $o/bench_$c.json 2> $o/bench_$c.err; tail -1 $o/bench_$c.json | cut -c1-160; done
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $o/bench_reference.json 2> $o/bench_reference.err; tail -1 $o/bench_reference.json | cut -c1-160
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_default.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_launches.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"gemm|dense_flux|curl" -c 8 --csv --log-file $o/launches_stage_C5.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_stage.log 2>&1
ls $o | wc -l
