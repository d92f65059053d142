cd $GRAFT_REPO_ROOT
for w in 4 5 6 7; do DGM_LANE_WARPS=$w timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_w$w.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b_w$w.json').read().strip().splitlines()[-1]); print('w=$w', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
for w in 2 3 4; do DGM_LANE_WARPS=$w DGM_ENGINE=sparse timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b3_w$w.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b3_w$w.json').read().strip().splitlines()[-1]); print('C3 sparse w=$w', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
