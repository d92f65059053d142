cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-c8}; mkdir -p $o
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; tail -4 $o/smoke.log
timeout 2000 python -m pytest tests -m gpu -q -x > $o/pytest.log 2>&1; tail -3 $o/pytest.log
for c in C3 C4 C5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $o/bench_$c.json 2> $o/bench_$c.err; python -c "
import json; d=json.loads(open('$o/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['engine'], d['ms_per_step'], d['roofline']['frac'])"; done
timeout 1200 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"gemm|dense_flux|curl" -c 8 --csv --log-file $o/launches_stage_C5.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_stage.log 2>&1
