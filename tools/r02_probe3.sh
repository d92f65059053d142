cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-p3}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stab.py tests/test_gpu_fullsize.py -q -x -k "hybrid" > $o/pytest_hybrid.log 2>&1; tail -2 $o/pytest_hybrid.log
timeout 900 python tools/engine_sweep.py 24 4,5,6,7,8 > $o/engine_sweep.txt 2>&1; cat $o/engine_sweep.txt
DGM_ENGINE=hybrid timeout 600 python bench.py --config C3 --no-cpu-baseline --no-e2e > $o/bench_C3_hybrid.json 2> $o/bench_C3_hybrid.err; tail -1 $o/bench_C3_hybrid.json | cut -c1-250
timeout 900 python tools/curved_bench.py 12 2,4,6,8,10 > $o/curved_bench.txt 2>&1; cat $o/curved_bench.txt
