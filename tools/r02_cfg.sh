cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-cfg}; mkdir -p $o
for cfg in 0 1 2 3; do for c in C3 C5; do DGM_DENSE_CFG=$cfg timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $o/bench_${c}_$cfg.json 2> $o/bench_${c}_$cfg.err; python -c "
import json; d=json.loads(open('$o/bench_${c}_$cfg.json').read().strip().splitlines()[-1]); print('cfg $cfg $c', d['engine'], d['ms_per_step'])"; done; done
