cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2; echo TESTS_DONE
for i in 1 2; do for c in C2 C3; do python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_${c}.json 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/b_${c}.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done; done
