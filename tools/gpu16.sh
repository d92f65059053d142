cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lane_stage -s 2 -c 1 -o gpurun_out/prof_sf_C2 python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_a.log 2>&1; echo "ncu rc=$?"
python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stage2 -s 2 -c 1 -o gpurun_out/prof_sf_C5 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_b.log 2>&1; echo "ncu rc=$?"
