cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense and (apply or continue)" 2>&1 | tail -2
run() { # config cfg
  DGM_DENSE_CFG=$2 timeout 300 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$1_$2.json 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/b_$1_$2.json').read().strip().splitlines()[-1]); print('$1 cfg$2', d['config']['engine'], d['value'], d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1
}
run C3 0
for k in 0; do run C4 $k; done
for k in 0; do run C5 $k; done
