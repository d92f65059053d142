// Standalone timing of the streamed curl kernel (experiments; not part of the library).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1104_4208_b200/csrc \
//      -DSWEEP='"sweep_p10.cuh"' -DPP=10 curl_bench.cu -o curl_bench
#include <cstdio>
#include <string>
#include "dgm_curl.cuh"
#include SWEEP
DGM_CURL_INSTANTIATE(10)
namespace dgm {
dgm_status set_err(dgm_ctx *, dgm_status s, const std::string &) { return s; }
}
int main(int argc, char **argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 663552;
  using D = dgm::curl::Dims<PP>;
  double *Y, *C, *C2;
  cudaMalloc(&Y, sizeof(double) * 3 * n * D::LD);
  cudaMalloc(&C, sizeof(double) * 3 * n * D::LDC);
  cudaMalloc(&C2, sizeof(double) * 3 * n * D::LDC);
  cudaMemset(Y, 0, sizeof(double) * 3 * n * D::LD);
  dgm_ctx *c = new dgm_ctx();
  c->n_tet = n;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) dgm::launch_curl_p10(c, Y, C, 0);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) dgm::launch_curl_p10(c, Y, C, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%s n=%lld: %.3f ms per launch (%s)\n", SWEEP, (long long)n, ms / 5, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
