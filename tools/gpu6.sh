cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2_lane7.json 2>&1; tail -c 900 gpurun_out/bench_C2_lane7.json
python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lane_stage -s 2 -c 1 -o gpurun_out/prof_lane7_C2 python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_lane7.log 2>&1; echo "ncu rc=$?"
