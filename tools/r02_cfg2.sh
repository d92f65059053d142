cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-cfg2}; mkdir -p $o
for sc in 0 1 2 3; do for c in C4 C5; do DGM_STAGE_CFG=$sc timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $o/b_${c}_$sc.json 2>/dev/null; python -c "
import json; d=json.loads(open('$o/b_${c}_$sc.json').read().strip().splitlines()[-1]); print('stage_cfg=$sc $c', d['ms_per_step'])"; done; done
