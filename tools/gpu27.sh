cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stab.py -x -q -k "7 or 8 or 9 or 10" 2>&1 | tail -4
run() { # config KW chunk
  DGM_ST_KW=$2 DGM_ST_CHUNK=$3 timeout 300 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$1_$2_$3.json 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/b_$1_$2_$3.json').read().strip().splitlines()[-1]); print('$1 KW=$2 CH=$3', d['value'], d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1
}
for kc in "1 16384" "2 16384" "1 8192" "1 32768"; do run C4 $kc; done
for kc in "1 16384" "2 16384"; do run C5 $kc; done
