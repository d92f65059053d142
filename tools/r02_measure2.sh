# Round-2 measurement pass 2: smoke, curved/flat timings, bench lines (default C5 = hybrid,
# C2-C4), reference arm, FP64 peaks, ncu launch list of the default bench, per-kernel
# DRAM/pipe metrics of one C5 stage, and one ncu --set full capture of the C5 stage GEMM.
cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-m2}; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $o/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; tail -4 $o/smoke.log
timeout 900 python tools/curved_bench.py 12 2,4,6,8,10 > $o/curved_bench.txt 2>&1; cat $o/curved_bench.txt
timeout 120 ./tools/peaks/fp64_peaks > $o/fp64_peaks.txt 2>&1
timeout 900 python bench.py > $o/bench_default.json 2> $o/bench_default.err; tail -1 $o/bench_default.json | cut -c1-300
for c in C2 C3 C4; do timeout 600 python bench.py --config $c > $o/bench_$c.json 2> $o/bench_$c.err; tail -1 $o/bench_$c.json | cut -c1-200; done
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $o/bench_reference.json 2> $o/bench_reference.err; tail -1 $o/bench_reference.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_default.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_launches.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"gemm|dense_flux|curl" -c 8 --csv --log-file $o/launches_stage_C5.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_stage.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gemm -s 4 -c 1 -o $o/stage_gemm_C5 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_full.log 2>&1
ls $o
