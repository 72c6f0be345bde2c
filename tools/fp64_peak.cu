// fp64_peak.cu -- measured FP64 (DFMA) throughput of this GPU, the ALU roofline denominator for
// the RAS subdomain solves.  8 independent DFMA chains per thread, full occupancy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o tools/fp64_peak
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

int main(int argc, char** argv) {
  int dev = 0, sms = 0, clk = 0;
  const int reps = argc > 1 ? atoi(argv[1]) : 1;   // timed launches (best and median reported)
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int threads = 256, blocks = sms * 8, iters = 4096;
  double* out;
  cudaMalloc(&out, sizeof(double) * threads * blocks);
  dfma_kernel<<<blocks, threads>>>(out, 16, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::vector<float> t(reps);
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t[r], e0, e1);
  }
  std::sort(t.begin(), t.end());
  const double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
  const float best = t[0], med = t[reps / 2];
  printf("{\"fp64_dfma_tflops\": %.3f, \"fp64_dfma_tflops_median\": %.3f, \"reps\": %d, "
         "\"sms\": %d, \"clock_mhz_attr\": %.0f, \"ms_best\": %.3f, "
         "\"dfma_per_clk_per_sm_at_attr_clock\": %.1f}\n",
         flops / best / 1e9, flops / med / 1e9, reps, sms, clk / 1e3, best,
         flops / 2 / (best * 1e-3) / sms / (clk * 1e3));
  return 0;
}
