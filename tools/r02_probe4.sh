cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-p4}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_varmat.py tests/test_gpu_curved.py -q -x > $o/pytest.log 2>&1; tail -3 $o/pytest.log
timeout 900 python tools/curved_bench.py 12 2,4,6,8,10 > $o/curved_bench.txt 2>&1; cat $o/curved_bench.txt
DGM_POINT_GEMM=1 timeout 900 python tools/curved_bench.py 12 4,10 > $o/curved_bench_gemm.txt 2>&1; cat $o/curved_bench_gemm.txt
timeout 600 python tools/varmat_bench.py > $o/varmat_bench.txt 2>&1; cat $o/varmat_bench.txt
