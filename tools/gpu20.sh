cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b_e2e.json 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/b_e2e.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"
