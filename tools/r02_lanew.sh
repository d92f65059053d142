cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-lw}; mkdir -p $o
for w in 4 5 6 7; do DGM_LANE_WARPS=$w timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e > $o/bench_C2_w$w.json 2>/dev/null; python -c "
import json; d=json.loads(open('$o/bench_C2_w$w.json').read().strip().splitlines()[-1]); print('w=$w', d['ms_per_step'], d['roofline']['frac'])"; done
