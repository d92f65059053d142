cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-nh}; mkdir -p $o
for v in "1 1" "2 1" "1 2" "2 2"; do set -- $v; DGM_STAGE_NH=$1 DGM_TRACE_NH=$2 timeout 600 python bench.py --no-cpu-baseline --no-e2e > $o/b_$1_$2.json 2>/dev/null; python -c "
import json; d=json.loads(open('$o/b_$1_$2.json').read().strip().splitlines()[-1]); print('stage_nh=$1 trace_nh=$2', d['ms_per_step'])"; done
