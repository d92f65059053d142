cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py > gpurun_out/bench_default_r1b.json 2> gpurun_out/bench_default_r1b.err; tail -c 2500 gpurun_out/bench_default_r1b.json
for c in C3 C4 C5; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_r1b.json 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_${c}_r1b.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"; done
