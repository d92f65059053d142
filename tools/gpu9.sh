cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C3.csv python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu0.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:lane_stage -s 2 -c 1 -o gpurun_out/prof_l6_C3 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l6.log 2>&1; echo "ncu rc=$?"
