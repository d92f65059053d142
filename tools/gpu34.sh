cd $GRAFT_REPO_ROOT
DGM_ENGINE=dense DGM_DENSE_CFG=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stab.py -q 2>&1 | tail -2
run() { # config cfg
  DGM_ENGINE=dense DGM_DENSE_CFG=$2 timeout 300 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$1_$2.json 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/b_$1_$2.json').read().strip().splitlines()[-1]); print('$1 cfg$2', d['value'], d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1
}
DGM_DEBUG_DENSE=1 DGM_ENGINE=dense python -c "
import dgm_inputs as di
from paper_1104_4208_b200 import Context
for p in (4,6,8,10):
    m = di.kuhn_mesh(2, jitter=0.1, seed=1)
    Context(m.xyz, m.tet, p)
" 2>&1 | tail -4
for c in C2 C3; do run $c 0; done
for k in 0 1 2 3; do run C4 $k; done
for k in 0 1 2 3; do run C5 $k; done
