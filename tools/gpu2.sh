cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
for c in C2 C3 C5; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; tail -c 1500 gpurun_out/bench_$c.json; done
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "default rc=$?"; cat gpurun_out/bench_default.json
python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 4 -c 2 -o gpurun_out/prof_C2 python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
