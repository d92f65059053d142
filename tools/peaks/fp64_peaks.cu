// FP64 peak microbenchmarks for the roofline denominators.
// DFMA: independent FMA chains per thread, all SMs, timed with CUDA events.
// DMMA: mma.sync.aligned.m8n8k4 f64 (the only FP64 tensor path on sm_100a).
// HBM: read+write copy of 4 GiB (double2 loads/stores), grid = 148*k.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double *out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = t; c[t][1] = -t; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2 *__restrict__ in, double2 *__restrict__ out, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = in[i];
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  int l2 = 0; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  printf("{\"sms\": %d, \"clock_khz\": %d, \"l2_bytes\": %d}\n", nsm, clk, l2);
  double *out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA
  for (int blocks_per_sm = 4; blocks_per_sm <= 8; blocks_per_sm *= 2) {
    int iters = 20000, threads = 256, blocks = nsm * blocks_per_sm;
    dfma_kernel<8><<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * threads * blocks;
    printf("{\"kind\": \"dfma\", \"blocks_per_sm\": %d, \"tflops\": %.3f, \"ms\": %.3f}\n", blocks_per_sm, flops / ms / 1e9, ms);
  }
  // DMMA m8n8k4: 2*8*8*4 = 512 flops per warp instruction
  {
    int iters = 4000, threads = 256, blocks = nsm * 4;
    dmma_kernel<<<blocks, threads>>>(out, 10);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 512.0 * 8 * (double)iters * (threads / 32) * blocks;
    printf("{\"kind\": \"dmma_m8n8k4\", \"tflops\": %.3f, \"ms\": %.3f}\n", flops / ms / 1e9, ms);
  }
  // HBM copy 4 GiB -> 4 GiB
  {
    size_t bytes = (size_t)4 << 30, n = bytes / 16;
    double2 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    CK(cudaMemset(a, 0, bytes)); CK(cudaMemset(b, 0, bytes));
    for (int k = 0; k < 3; ++k) copy_kernel<<<nsm * 8, 512>>>(a, b, n);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int k = 0; k < 10; ++k) {
      cudaEventRecord(e0);
      copy_kernel<<<nsm * 8, 512>>>(a, b, n);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("{\"kind\": \"hbm_copy\", \"gbs\": %.1f, \"ms\": %.3f}\n", 2.0 * bytes / best / 1e6, best);
    cudaFree(a); cudaFree(b);
  }
  return 0;
}
