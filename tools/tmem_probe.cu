// tmem_probe.cu -- is tensor memory usable as extra on-chip storage for the Krylov basis of the
// 3D subdomain kernel?  Measures tcgen05.st / tcgen05.ld (32x32b shape: every thread moves its
// own lane's consecutive 32-bit columns) throughput per SM with 8 warps, next to ld.shared.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem tools/tmem_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int NCOL>   // columns per ld/st instruction (x16 -> 16 registers)
__global__ void __launch_bounds__(256, 1) k_tmem(int iters, double* out, long long* cyc) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s;
  // warp w: lanes 32 (w % 4) .., columns 256 (w / 4) ..
  const uint32_t ta = base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(256 * (warp >> 2));
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 16 + i;
  // store 256 columns (16 x x16)
#pragma unroll
  for (int c = 0; c < 256; c += 16)
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16};" ::"r"(ta + c),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  __syncthreads();
  long long t0 = clock64();
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 256; c += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(ta + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 16; ++i) acc += v[i];
    }
  }
  long long t1 = clock64();
  __syncthreads();
  long long t2 = clock64();
  // stores timed too
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 256; c += 16)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16};" ::"r"(ta + c),
          "r"(r[0] + it), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
          "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),
          "r"(r[14]), "r"(r[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  long long t3 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) {
    cyc[blockIdx.x * 2] = t1 - t0;
    cyc[blockIdx.x * 2 + 1] = t3 - t2;
  }
  out[blockIdx.x * 256 + threadIdx.x] = (double)acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

// the same traffic through ld.shared (8-byte loads, conflict-free)
__global__ void __launch_bounds__(256, 1) k_smem(int iters, double* out, long long* cyc) {
  __shared__ double s[256 * 16];
  for (int i = threadIdx.x; i < 256 * 16; i += 256) s[i] = i;
  __syncthreads();
  long long t0 = clock64();
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 128; ++c) acc += s[(c & 15) * 256 + threadIdx.x];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x * 2] = t1 - t0;
  out[blockIdx.x * 256 + threadIdx.x] = acc;
}

int main() {
  const int nb = 148, iters = 200;
  double* out;
  long long* cyc;
  cudaMalloc(&out, nb * 256 * sizeof(double));
  cudaMalloc(&cyc, nb * 2 * sizeof(long long));
  long long h[2 * 148];
  for (int rep = 0; rep < 2; ++rep) {
    k_tmem<16><<<nb, 256>>>(iters, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("tmem kernel: %s\n", cudaGetErrorString(e)); return 1; }
  }
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  // bytes per SM per timed loop: 256 threads x 256 columns x 4 B x iters
  const double bytes = 256.0 * 256 * 4 * iters;
  printf("tcgen05.ld 32x32b.x16: %.1f B/clk/SM (%lld cycles)\n", bytes / h[0], h[0]);
  printf("tcgen05.st 32x32b.x16: %.1f B/clk/SM (%lld cycles)\n", bytes / h[1], h[1]);
  k_smem<<<nb, 256>>>(iters, out, cyc);
  cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  printf("ld.shared 8 B: %.1f B/clk/SM (%lld cycles)\n", 256.0 * 128 * 8 * iters / h[0], h[0]);
  return 0;
}
