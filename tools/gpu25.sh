cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "7 or 8 or 9 or 10" 2>&1 | tail -2
run() { # config K W
  DGM_HO_K=$2 DGM_HO_W=$3 timeout 300 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$1_$2_$3.json 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/b_$1_$2_$3.json').read().strip().splitlines()[-1]); print('$1 K=$2 W=$3', d['value'], d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1
}
for kw in "1 1" "1 2" "1 4" "2 1" "2 2" "2 4" "4 2" "4 4" "4 8"; do run C4 $kw; done
for kw in "1 2" "1 4" "2 2" "2 4" "4 4"; do run C5 $kw; done
