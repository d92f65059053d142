cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed.py tests/test_gpu_varmat.py -q -x -k "dense or mixed or varmat" 2>&1 | tail -2
for c in C3 C4 C5; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
