cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-lift}; mkdir -p $o
for c in C4 C5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $o/bench_$c.json 2> $o/bench_$c.err; python -c "
import json; d=json.loads(open('$o/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['engine'], d['ms_per_step'], d['roofline']['frac'])"; done
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"gemm_kernel<.int.0" -s 1 -c 1 -o $o/lift_gemm_C5 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_full.log 2>&1; tail -2 $o/ncu_full.log
