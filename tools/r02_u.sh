cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-u}; mkdir -p $o
for c in C3 C4 C5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $o/b_$c.json 2>/dev/null; python -c "
import json; d=json.loads(open('$o/b_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'])"; done
