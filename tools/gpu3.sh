cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2_lane.json 2>&1; tail -c 1200 gpurun_out/bench_C2_lane.json
