# Build curl-sweep timing variants over warp pairs per CTA (p=10, constant table). Run from tools/curlbench.
set -e
I=../../paper_1104_4208_b200/csrc
(cd ../.. && python -c "from paper_1104_4208_b200.gen import sweepgen; sweepgen.emit(10, 'tools/curlbench/sweep_p10_const.cuh')")
for np in 1 2 4; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I$I -DDGM_CURL_NPAIR=$np -DSWEEP="\"sweep_p10_const.cuh\"" -DPP=10 curl_bench.cu -o cb_np$np &
done
wait
