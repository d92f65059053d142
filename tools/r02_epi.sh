cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-epi}; mkdir -p $o
timeout 2400 python -m pytest tests -m gpu -q -x > $o/pytest.log 2>&1; tail -2 $o/pytest.log
for epi in reg smem; do for c in C3 C4 C5; do DGM_STAGE_EPI=$epi timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $o/b_${c}_$epi.json 2>/dev/null; python -c "
import json; d=json.loads(open('$o/b_${c}_$epi.json').read().strip().splitlines()[-1]); print('epi=$epi $c', d['ms_per_step'])"; done; done
