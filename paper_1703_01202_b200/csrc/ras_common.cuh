// ras_common.cuh -- warp/block reduction helpers shared by the subdomain-solve kernels
// (ras2d.cu, ras3d_col.cu): fixed shuffle trees, deterministic.
#pragma once

#include <cuda_runtime.h>

namespace {

constexpr int pow2_at_least(int x) { return x <= 1 ? 1 : 2 * pow2_at_least((x + 1) / 2); }

// One reduce-scatter step: lanes exchange the half they do not keep across lane offset `off`
// (HALF is a template parameter so every array index is compile-time: registers only).
template <int NVP, int HALF>
__device__ __forceinline__ void rs_step(double (&a)[NVP], int lane, int off) {
  const bool upper = (lane & off) != 0;
#pragma unroll
  for (int i = 0; i < HALF; ++i) {
    const double lo = a[i], hi = a[i + HALF];      // compile-time indices: registers
    const double send = upper ? lo : hi, keep = upper ? hi : lo;
    a[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
  }
  if constexpr (HALF > 1) rs_step<NVP, HALF / 2>(a, lane, off >> 1);
}

// Warp reduce-scatter of NVP (power of two, <= 32) values: afterwards lane l holds the warp
// sum of value (l >> (5 - log2 NVP)).  Fixed shuffle tree, deterministic.
template <int NVP>
__device__ __forceinline__ double warp_reduce_scatter(double (&a)[NVP]) {
  const int lane = threadIdx.x & 31;
  int off = 16;
  if constexpr (NVP > 1) {
    rs_step<NVP, NVP / 2>(a, lane, 16);
    off = 16 / (NVP / 2) / 2;
  }
  double s = a[0];
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1)
    if (o <= off) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}


// Block all-reduce of NV values per thread (NV <= 16), one barrier: warp reduce-scatter sized
// to the value count, per-warp partials in red[warp][16], then every warp sums the partials of
// all NWMAX (absent warps add 0) in a fixed pairwise tree; totals in hw[0..NV) of this warp.
template <int NV, int NWMAX>
__device__ __forceinline__ void sized_allreduce(const double (&acc)[NV], double* red, double* hw,
                                                int nwt) {
  constexpr int NVP = pow2_at_least(NV);
  constexpr int SH = 5 - (NVP == 1 ? 0 : NVP == 2 ? 1 : NVP == 4 ? 2 : NVP == 8 ? 3 : 4);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double a[NVP];
#pragma unroll
  for (int i = 0; i < NVP; ++i) a[i] = i < NV ? acc[i] : 0.0;
  const double s = warp_reduce_scatter<NVP>(a);
  const int vi = lane >> SH;
  if ((lane & ((1 << SH) - 1)) == 0 && vi < NV) red[wid * 16 + vi] = s;
  __syncthreads();
  if (lane < NV) {
    double t[NWMAX];
#pragma unroll
    for (int w = 0; w < NWMAX; ++w) t[w] = w < nwt ? red[w * 16 + lane] : 0.0;
#pragma unroll
    for (int st = 1; st < NWMAX; st *= 2)
#pragma unroll
      for (int w = 0; w + st < NWMAX; w += 2 * st) t[w] += t[w + st];
    hw[lane] = t[0];
  }
  __syncwarp();
}

}  // namespace

// Arnoldi steps actually taken by the subdomain solves of a launch (bench roofline): one thread
// per box adds jm, jm^2 and 1 (boxes that exit at beta = 0 or break down early do less than
// k steps, so the algorithmic flops are counted from these sums, not from k).  Null unless the
// library is profiling.
__device__ __forceinline__ void ras_count(unsigned long long* cnt, int jm) {
  if (cnt) {
    atomicAdd(cnt, (unsigned long long)jm);
    atomicAdd(cnt + 1, (unsigned long long)jm * (unsigned long long)jm);
    atomicAdd(cnt + 2, 1ull);
  }
}
