# Build curl-sweep timing variants (p=10) for a GPU experiment. Run from tools/curlbench.
set -e
I=../../paper_1104_4208_b200/csrc
for coef in imm const; do
  (cd ../.. && SWEEP_COEF=$coef python -c "from paper_1104_4208_b200.gen import sweepgen; sweepgen.emit(10, 'tools/curlbench/sweep_p10_$coef.cuh')")
  for sync in pair cta; do
    def=""; [ $sync = cta ] && def="-DCURL_CTA_SYNC"
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I$I $def -DSWEEP="\"sweep_p10_$coef.cuh\"" -DPP=10 curl_bench.cu -o cb_${coef}_${sync} &
  done
done
wait
ls -la cb_*
