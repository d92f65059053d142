cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-lane}; mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stab.py -m gpu -q -x -k "sparse" > $o/pytest.log 2>&1; tail -2 $o/pytest.log
timeout 600 python bench.py --config C2 --no-cpu-baseline --no-e2e > $o/bench_C2.json 2> $o/bench_C2.err; python -c "
import json; d=json.loads(open('$o/bench_C2.json').read().strip().splitlines()[-1]); print('C2', d['engine'], d['ms_per_step'], d['roofline']['frac'])"
timeout 900 python tools/engine_sweep.py 24 3,4,5 > $o/engine_sweep.txt 2>&1; cat $o/engine_sweep.txt
