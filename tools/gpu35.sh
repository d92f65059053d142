cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for c in C2 C3 C4 C5; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$c.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b_$c.json').read().strip().splitlines()[-1]); print('$c', d['config']['engine'], d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
