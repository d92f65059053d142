cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in C3 C4 C5; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_w2.json 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_${c}_w2.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stage2 -s 2 -c 1 -o gpurun_out/prof_w2_C5 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_w2.log 2>&1; echo "ncu rc=$?"
