# Round-2 measurement pass on one B200 (run via gpurun from the repo root):
# smoke, GPU tests, FP64 peaks, bench lines (default = C5, then C2-C4), reference arm,
# the ncu launch list of the default bench command and per-kernel DRAM/DMMA of one C5 stage.
# usage: bash tools/r02_measure.sh [tag] [skip-tests]
cd $GRAFT_REPO_ROOT
tag=${1:-a}
o=gpurun_out/r02$tag
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $o/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $o/smoke.log 2>&1; tail -2 $o/smoke.log
if [ "$2" != "skip-tests" ]; then
  timeout 2700 python -m pytest tests -m gpu -q -x > $o/pytest_gpu.log 2>&1; tail -2 $o/pytest_gpu.log
fi
timeout 120 ./tools/peaks/fp64_peaks > $o/fp64_peaks.txt 2>&1; cat $o/fp64_peaks.txt | head -8
timeout 900 python bench.py > $o/bench_default.json 2> $o/bench_default.err; tail -1 $o/bench_default.json | cut -c1-400
for c in C2 C3 C4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $o/bench_$c.json 2> $o/bench_$c.err; tail -1 $o/bench_$c.json | cut -c1-200; done
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $o/bench_reference.json 2> $o/bench_reference.err; tail -1 $o/bench_reference.json | cut -c1-200
# launch list of the default bench command (recipe: gpu__time_duration, clocks unlocked)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_default.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_launches.log 2>&1
# one C5 stage per kernel: DRAM bytes and DMMA pipe (cold cache per replay)
timeout 1200 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"gemm|dense_flux|stage|stream|sparse|curl|lift|trace" -c 8 --csv --log-file $o/launches_stage_C5.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_stage.log 2>&1
ls -la $o
