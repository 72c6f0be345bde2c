// tmem.cuh -- tensor memory (TMEM) as per-thread storage for the Krylov basis of the subdomain
// kernels (sm_100a).  tcgen05.st / tcgen05.ld of the 32x32b shape move each thread's own TMEM
// lane row (32-bit columns): warp w reaches lanes 32 (w mod 4) .. + 31, so two warps of the same
// lane quarter split the columns.  A double is two columns.  Measured on this pool
// (tools/tmem_probe.cu, 8 warps): tcgen05.ld 427 B/clk/SM with a wait after every x16,
// tcgen05.st 977 B/clk/SM (shared memory: 128 B/clk).
#pragma once

#include <cstdint>

#include "pfc_device.cuh"

namespace tmem {

template <int NCOL>   // power of two >= 32; one warp allocates (and frees), address into *dst
__device__ __forceinline__ void alloc(uint32_t* dst) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst)), "n"(NCOL)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOL>
__device__ __forceinline__ void dealloc(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(NCOL)
               : "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// the stores' sources are consumed at issue; wait before reading the columns back
__device__ __forceinline__ void wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void st8(uint32_t ta, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
               "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void st4(uint32_t ta, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3])
               : "memory");
}
__device__ __forceinline__ void st2(uint32_t ta, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(ta), "r"(r[0]),
               "r"(r[1])
               : "memory");
}
// loads of 8 / 12 / 4 / 2 columns with their wait in the same statement (registers valid after)
__device__ __forceinline__ void ld8(uint32_t ta, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(ta)
      : "memory");
}
__device__ __forceinline__ void ld12(uint32_t ta, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%12];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8,%9,%10,%11}, [%13];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11])
      : "r"(ta), "r"(ta + 8)
      : "memory");
}
__device__ __forceinline__ void ld4(uint32_t ta, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
      : "r"(ta)
      : "memory");
}
__device__ __forceinline__ void ld2(uint32_t ta, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(v[0]), "=r"(v[1])
      : "r"(ta)
      : "memory");
}

// N doubles of this thread <-> 2N columns at ta (warp-collective: every lane of the warp)
template <int N>
__device__ __forceinline__ void st(uint32_t ta, const double (&d)[N]) {
  uint32_t r[2 * N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    r[2 * k] = (uint32_t)__double2loint(d[k]);
    r[2 * k + 1] = (uint32_t)__double2hiint(d[k]);
  }
  int c = 0;
#pragma unroll
  for (; c + 8 <= 2 * N; c += 8) st8(ta + c, r + c);
  if constexpr ((2 * N) % 8 >= 4) { st4(ta + c, r + c); c += 4; }
  if constexpr ((2 * N) % 4 == 2) st2(ta + c, r + c);
}
template <int N>
__device__ __forceinline__ void ld(uint32_t ta, double (&d)[N]) {
  uint32_t r[2 * N];
  if constexpr (2 * N == 12) {
    ld12(ta, r);
  } else {
    int c = 0;
#pragma unroll
    for (; c + 8 <= 2 * N; c += 8) ld8(ta + c, r + c);
    if constexpr ((2 * N) % 8 >= 4) { ld4(ta + c, r + c); c += 4; }
    if constexpr ((2 * N) % 4 == 2) ld2(ta + c, r + c);
  }
#pragma unroll
  for (int k = 0; k < N; ++k) d[k] = __hiloint2double((int)r[2 * k + 1], (int)r[2 * k]);
}

}  // namespace tmem
