// tma_box_test.cu -- diagnostic: does a cp.async.bulk.tensor.3d load of a WX x WY x 1 fp64 box
// land correctly (for the 3D stencil's plane boxes)?  Prints max |error| per box shape.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_box_test.cu -o tma_box_test
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../paper_1703_01202_b200/csrc/pfc_device.cuh"

__device__ CUtensorMap g_map;    // V == 6: descriptor in global memory

template <int V>
__global__ void box_kernel(const __grid_constant__ CUtensorMap m, double* out, int wx, int wy,
                           int x, int y, int z, int off, const double* src) {
  extern __shared__ __align__(1024) double sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    if (V != 5) fence_mbar_init();
  }
  __syncthreads();
  if (V == 4) {   // mbarrier only: plain arrive, then wait for phase 0
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
    mbar_wait(&bar, 0);
    for (int q = threadIdx.x; q < wx * wy; q += blockDim.x) out[q] = -1.0;
    return;
  }
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, wx * wy * 8);
    if (V == 0 || V == 5) tma_load_3d(sm + off, &m, &bar, x, y, z);
    if (V == 1) tma_load_2d(sm + off, &m, &bar, x, y);
    if (V == 2)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                   " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(sm + off)),
                   "l"(reinterpret_cast<uint64_t>(&m)), "r"(smem_u32(&bar)), "r"(x), "r"(y), "r"(z)
                   : "memory");
    if (V == 6) tma_load_3d(sm + off, &g_map, &bar, x, y, z);
    if (V == 7)   // plain bulk copy (no tensor map) of wx*wy doubles starting at element (x,y,z)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(sm + off)), "l"(src + x + 128 * (y + 128 * z)),
                   "r"(wx * wy * 8), "r"(smem_u32(&bar)) : "memory");
    if (V == 3) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&m)) : "memory");
      asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(&m)) : "memory");
      tma_load_3d(sm + off, &m, &bar, x, y, z);
    }
  }
  mbar_wait(&bar, 0);
  for (int q = threadIdx.x; q < wx * wy; q += blockDim.x) out[q] = sm[off + q];
}

int main(int argc, char** argv) {
  const int V = argc > 1 ? atoi(argv[1]) : 0;
  const int n = getenv("TN") ? atoi(getenv("TN")) : 128;
  double* a;
  cudaMalloc(&a, sizeof(double) * (size_t)n * n * (getenv("TN") ? 1 : n));
  const size_t nn = (size_t)n * n * (getenv("TN") ? 1 : n);
  double* h = (double*)malloc(sizeof(double) * nn);
  for (size_t i = 0; i < nn; ++i) h[i] = (double)i;
  cudaMemcpy(a, h, sizeof(double) * nn, cudaMemcpyHostToDevice);
  double* out;
  cudaMalloc(&out, 8 * 256 * 256);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  int shapes[][3] = {{40, 22, 0}, {40, 38, 0}, {64, 32, 0}, {64, 32, 128}, {64, 32, 1152}, {32, 32, 0},
                     {48, 32, 0}, {56, 32, 0}, {64, 8, 0}, {128, 8, 0}};
  for (auto& s : shapes) {
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)n};
    cuuint64_t str[2] = {(cuuint64_t)n * 8, (cuuint64_t)n * n * 8};
    cuuint32_t box[3] = {(cuuint32_t)s[0], (cuuint32_t)s[1], 1}, es[3] = {1, 1, 1};
    const int rank = V == 1 ? 2 : 3;
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, a, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    auto k = V == 0 ? box_kernel<0> : V == 1 ? box_kernel<1> : V == 2 ? box_kernel<2>
           : V == 3 ? box_kernel<3> : V == 4 ? box_kernel<4> : V == 5 ? box_kernel<5>
           : V == 6 ? box_kernel<6> : box_kernel<7>;
    if (V == 6) cudaMemcpyToSymbol(g_map, &m, sizeof(m));
    const int dyn = getenv("DYN_KB") ? atoi(getenv("DYN_KB")) * 1024 : 200 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    const int xs = getenv("TX0") ? atoi(getenv("TX0")) : (V == 7 ? 4 : 5);
    k<<<1, 256, dyn>>>(m, out, s[0], s[1], xs, 7, V == 1 ? 0 : 9, s[2], a);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    double* ho = (double*)malloc(8 * s[0] * s[1]);
    double err = 0;
    if (e == cudaSuccess) {
      cudaMemcpy(ho, out, 8 * s[0] * s[1], cudaMemcpyDeviceToHost);
      for (int yy = 0; yy < s[1]; ++yy)
        for (int xx = 0; xx < s[0]; ++xx) {
          double want = (xs + xx) + n * (7 + yy) + (V == 1 ? 0.0 : (double)n * n * 9);
          if (V == 7) want = xs + (xx + s[0] * yy) + n * 7 + (double)n * n * 9;
          double d = ho[xx + s[0] * yy] - want;
          err = d * d > err ? d * d : err;
        }
    }
    printf("box %3d x %3d smem off %5d: encode %d, kernel %s, max err^2 %g\n", s[0], s[1], s[2],
           (int)r, cudaGetErrorString(e), err);
    free(ho);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
