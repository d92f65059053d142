cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-lift2}; mkdir -p $o
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stab.py tests/test_gpu_fullsize.py tests/test_gpu_curved.py tests/test_gpu_varmat.py -m gpu -q -x -k "hybrid or curved or varmat" > $o/pytest.log 2>&1; tail -2 $o/pytest.log
for c in C4 C5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $o/bench_$c.json 2> $o/bench_$c.err; python -c "
import json; d=json.loads(open('$o/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['engine'], d['ms_per_step'], d['roofline']['frac'])"; done
