# Dense GEMM CTA-shape sweep (DGM_DENSE_CFG: 0 = 64x96/3 stages, 1 = 64x96/4, 2 = 128x96/3, 3 = 32x96/4)
cd $GRAFT_REPO_ROOT
run() { DGM_DENSE_CFG=$2 timeout 300 python bench.py --config $1 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 cfg$2', d['value'], d['ms_per_step'], d['roofline']['frac'])"; }
for c in C3 C4 C5; do for k in 0 1 2 3; do run $c $k; done; done
