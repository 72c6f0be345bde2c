// tma_stream_bench.cu -- microbenchmark: how fast can one CTA per SM stream (TX+8)x(TY+6)x1
// fp64 plane boxes through a TMA ring (the 3D stencil's load pipeline), with no compute?
// Also times a plain coalesced copy for the HBM reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_stream_bench.cu -o tma_bench
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../paper_1703_01202_b200/csrc/pfc_device.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int WX, int WY, int RING, int PF, int NT, int NFIELD>
__global__ void __launch_bounds__(NT, 1) stream_kernel(const __grid_constant__ CUtensorMap ma,
                                                       const __grid_constant__ CUtensorMap mb,
                                                       double* out, int nx, int ny, int nz,
                                                       int zc, int ntx) {
  extern __shared__ __align__(128) double sm[];
  __shared__ uint64_t bars[RING];
  constexpr int WN = WX * WY;
  const int tid = threadIdx.x;
  const int x0 = (blockIdx.x % ntx) * (WX - 8), y0 = (blockIdx.x / ntx) * (WY - 6);
  const int z0 = blockIdx.y * zc;
  const int gx0 = x0 - 4, gy0 = y0 - 3;
  if (tid == 0) {
    for (int i = 0; i < RING; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int T = zc + 6;
  auto issue = [&](int t) {
    const int s = t % RING;
    int zp = (z0 - 3 + t + nz) % nz;
    mbar_expect_tx(&bars[s], NFIELD * WN * 8);
    tma_load_3d(sm + s * WN, &ma, &bars[s], gx0, gy0, zp);
    if (NFIELD == 2) tma_load_3d(sm + (RING + s) * WN, &mb, &bars[s], gx0, gy0, zp);
  };
  if (tid == 0)
    for (int t = 0; t < PF && t < T; ++t) issue(t);
  double acc = 0;
  for (int t = 0; t < T; ++t) {
    if (tid == 0 && t + PF < T) issue(t + PF);
    mbar_wait(&bars[t % RING], (t / RING) & 1);
    for (int q = tid; q < WN; q += NT) acc += sm[(t % RING) * WN + q];
    __syncthreads();
    if (t >= 6) {
      // write the tile interior of plane t-3 (write traffic like the stencil)
      for (int q = tid; q < (WX - 8) * (WY - 6); q += NT) {
        int xx = x0 + q % (WX - 8), yy = y0 + q / (WX - 8);
        out[(size_t)xx + (size_t)nx * yy + (size_t)nx * ny * (z0 + t - 6)] = acc;
      }
    }
  }
}

__global__ void copy_kernel(const double2* a, double2* b, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* fn; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}

template <int WX, int WY, int RING, int PF, int NT, int NFIELD>
void run(const char* name, double* a, double* b, double* o, int n) {
  CUtensorMap ma, mb;
  cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)n};
  cuuint64_t str[2] = {(cuuint64_t)n * 8, (cuuint64_t)n * n * 8};
  cuuint32_t box[3] = {WX, WY, 1}, es[3] = {1, 1, 1};
  auto E = enc();
  E(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  E(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, b, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 2 * RING * WX * WY * 8;
  auto k = stream_kernel<WX, WY, RING, PF, NT, NFIELD>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int ntx = n / (WX - 8), nty = n / (WY - 6);
  const int zc = 64;
  dim3 grid(ntx * nty, n / zc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int r = 0; r < 2; ++r) k<<<grid, NT, smem>>>(ma, mb, o, n, n, n, zc, ntx);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) k<<<grid, NT, smem>>>(ma, mb, o, n, n, n, zc, ntx);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  double bytes = (double)n * n * n * 8 * (NFIELD + 1);
  printf("%-40s box %dx%d ring %d pf %d nt %d: %.3f ms  %.0f GB/s (algorithmic %d-in 1-out)\n",
         name, WX, WY, RING, PF, NT, ms, bytes / ms / 1e6, NFIELD);
}

int main() {
  const int n = 512;
  size_t N = (size_t)n * n * n;
  double *a, *b, *o;
  CK(cudaMalloc(&a, N * 8)); CK(cudaMalloc(&b, N * 8)); CK(cudaMalloc(&o, N * 8));
  CK(cudaMemset(a, 0, N * 8)); CK(cudaMemset(b, 0, N * 8));
  {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    copy_kernel<<<148 * 16, 256>>>((double2*)a, (double2*)o, N / 2);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) copy_kernel<<<148 * 16, 256>>>((double2*)a, (double2*)o, N / 2);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("plain copy: %.3f ms %.0f GB/s\n", ms, 2.0 * N * 8 / ms / 1e6);
  }
  run<40, 22, 8, 4, 448, 2>("tma ring (stencil3d shape)", a, b, o, n);
  run<40, 22, 8, 6, 448, 2>("tma ring prefetch 6", a, b, o, n);
  run<40, 22, 12, 8, 448, 2>("tma ring prefetch 8", a, b, o, n);
  run<40, 38, 6, 4, 448, 2>("tma ring 32x32 tile", a, b, o, n);
  run<72, 22, 6, 4, 448, 2>("tma ring 64x16 tile", a, b, o, n);
  run<40, 22, 8, 4, 1024, 2>("tma ring 1024 thr", a, b, o, n);
  return 0;
}
