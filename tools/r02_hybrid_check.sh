# Hybrid engine after the constant-table sweeps: parity tests, C4/C5 dense vs hybrid, spectral tests.
cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-hyb}; mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stab.py tests/test_gpu_fullsize.py -q -x -k "hybrid or spectral" > $o/pytest.log 2>&1; tail -2 $o/pytest.log
for c in C4 C5; do for e in dense hybrid; do
DGM_ENGINE=$e timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $o/bench_${c}_$e.json 2> $o/bench_${c}_$e.err
python -c "
import json; d=json.loads(open('$o/bench_${c}_$e.json').read().strip().splitlines()[-1]); print('$c', d['engine'], d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1
done; done
