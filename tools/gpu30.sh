cd $GRAFT_REPO_ROOT
DGM_ENGINE=dense timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stab.py -q 2>&1 | tail -4
run() { # config engine
  DGM_ENGINE=$2 timeout 300 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$1_$2.json 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/b_$1_$2.json').read().strip().splitlines()[-1]); print('$1 $2', d['value'], d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1
}
for c in C2 C3 C4 C5; do run $c dense; done
