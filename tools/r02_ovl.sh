cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-ovl}; mkdir -p $o
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stab.py tests/test_gpu_curved.py tests/test_gpu_fullsize.py -m gpu -q -x -k "hybrid or curved" > $o/pytest.log 2>&1; tail -2 $o/pytest.log
for ov in 0 1; do for c in C4 C5; do DGM_OVERLAP=$ov timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $o/b_${c}_$ov.json 2>/dev/null; python -c "
import json; d=json.loads(open('$o/b_${c}_$ov.json').read().strip().splitlines()[-1]); print('overlap=$ov $c', d['ms_per_step'])"; done; done
