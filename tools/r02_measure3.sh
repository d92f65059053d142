# per-kernel DRAM/pipe metrics of one stage at C2-C4 (traffic for every bench line), the
# full-size stabilised test, and an ncu --set full capture of the C5 lift GEMM
cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-m3}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "stabilized" > $o/pytest_stab.log 2>&1; tail -2 $o/pytest_stab.log
for c in C2 C3 C4; do
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"gemm|dense_flux|curl|lane_stage|stream" -c 12 --csv --log-file $o/launches_stage_$c.csv \
  python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_stage_$c.log 2>&1
done
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"gemm_kernel<.int.0" -s 1 -c 1 -o $o/lift_gemm_C5 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_full.log 2>&1
ls $o
