// ras2d.cu -- left restricted additive Schwarz apply (K4), 2D, sm_100a.
//
//   z = sum_k (R_k^0)^T inv(A_k) R_k^delta v          Eq. (eq:ras) P:398-409
//
// One CTA per subdomain box Omega_k (b_x x b_y owned nodes).  The CTA gathers v and the
// Jacobian coefficient c on the extended box Omega_k^delta (E = b + 2o nodes per axis,
// periodic wrap = restriction R_k^delta), then runs exactly K steps of GMRES on
// A_k y = R_k^delta v entirely on chip (reading R9: fixed-work local solve, zero initial guess,
// CGS2, Givens, early exit only on exact breakdown), and writes only the owned nodes
// (R_k^0)^T -- disjoint writes, no atomics.
//
// A_k is the local Jacobian with phi = 0 on the 3-layer ring around the extended box
// (modified subdomain BC): the Krylov vector lives in the interior of a zero-padded
// (E+6)^2 shared-memory plane whose ring is never written, and the local J v is the composed
// stencil of K2 in three stages (halo 2 -> 1 -> 0):
//   L1 = Delta v,  B = ((1-gamma)/2 + c) v + L1 + Delta L1 / 2,  w = v/dt - Delta B.
//
// Latency design (one box per SM at E = 36..40: the K basis vectors take 104-128 KB):
//  * the Arnoldi vector w of the thread's own nodes stays in registers;
//  * each CGS2 pass is ONE block reduction: warp reduce-scatter (16 values in 16 shuffles
//    instead of 80), one barrier, lane-parallel cross-warp sums, shuffle broadcast;
//  * pass 2 also reduces |w'|^2 and the new norm is |w''|^2 = |w'|^2 - |h2|^2 (exact for an
//    orthonormal basis; pass 2 only removes rounding-size components), with an explicit extra
//    reduction when |h2|^2 > 1e-8 |w'|^2;
//  * normalisation writes V_{j+1} and the padded plane in one pass; the Givens QR of the small
//    Hessenberg matrix is deferred to one thread after the K steps (nothing inside the fixed-work
//    loop depends on it).  Five barriers per Arnoldi step.
#include "pfc_device.cuh"
#include "pfc_internal.h"

#include <stdlib.h>

namespace {

constexpr int NT = 512;
constexpr int NW = NT / 32;
constexpr int MAXN = 1600;                 // largest ext box (E = 40)
constexpr int SLOTS = (MAXN + NT - 1) / NT;

struct RasArgs {
  const double* v;
  const double* c;
  double* z;
  int nx, ny;
  int bx, by, o;
  double idt, gamma, ih2;
};

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

// Block sum of nv (runtime, <= NVP) values held by every thread in acc[]: the sums are left in
// this warp's private copy hw[0..nv) (valid after return for every lane of the warp).  One
// barrier; `red` alternates between two buffers so consecutive reductions never race.
// Value NVP-1 is also reduced when `with_last` (the norm slot).
template <int NVP, int NWB = NW>
__device__ __forceinline__ void block_allreduce(double (&acc)[NVP], int nv, double* red,
                                                double* hw, bool with_last = false) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int SH = 5 - (NVP == 1 ? 0 : NVP == 2 ? 1 : NVP == 4 ? 2 : NVP == 8 ? 3 : NVP == 16 ? 4 : 5);
  double s = warp_reduce_scatter<NVP>(acc);
  const int vi = lane >> SH;
  if ((lane & ((1 << SH) - 1)) == 0 && (vi < nv || (with_last && vi == NVP - 1)))
    red[wid * NVP + vi] = s;
  __syncthreads();
  if (lane < nv || (with_last && lane == NVP - 1)) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NWB; ++w) t += red[w * NVP + lane];
    hw[lane] = t;
  }
  __syncwarp();
}

template <int K>
__global__ void __launch_bounds__(NT, 1) ras2d_kernel(RasArgs p) {
  constexpr int NVP = pow2_at_least(K + 2);   // values 0..K-1 plus the norm slot NVP-1
  // declared as a shared array (not re-derived through an integer) so that every access
  // compiles to LDS/STS with 32-bit shared addressing; 128-B aligned for TMA destinations
  extern __shared__ __align__(128) double smem_dyn[];
  double* sm = smem_dyn;
  const int Ex = p.bx + 2 * p.o, Ey = p.by + 2 * p.o;
  const int n = Ex * Ey;
  const int Px = Ex + 6, Py = Ey + 6;
  const int np = Px * Py;
  double* V = sm;                        // K n
  double* cl = V + (size_t)K * n;        // n
  double* pv = cl + n;                   // np (zero ring)
  double* pl = pv + np;                  // np
  double* pb = pl + np;                  // np
  double* red = pb + np;                 // 2 x NW x NVP
  double* hwall = red + 2 * NW * NVP;    // NW x 3 NVP: per-warp copies of h1 | h2 | misc
  __shared__ double H[(K + 1) * K];
  __shared__ double gv[K + 1], cs[K], sn[K], yv[K];

  const int tid = threadIdx.x;
  double* h1 = hwall + (tid >> 5) * 3 * NVP;
  double* h2 = h1 + NVP;
  double* hx = h2 + NVP;
  const int nbx = p.nx / p.bx;
  const int ibx = blockIdx.x % nbx, iby = blockIdx.x / nbx;
  const int gx0 = ibx * p.bx - p.o, gy0 = iby * p.by - p.o;
  const double ih2 = p.ih2, idt = p.idt, alpha = 0.5 * (1.0 - p.gamma);

  // own box nodes: l = tid + s*NT; padded index of node l
  int pidx[SLOTS];
  bool own[SLOTS];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    int l = tid + s * NT;
    own[s] = l < n;
    pidx[s] = own[s] ? ((l / Ex) + 3) * Px + (l % Ex) + 3 : 0;
  }

  // zero the padded planes (ring stays zero), gather R_k^delta v and c with periodic wrap
  for (int q = tid; q < 3 * np; q += NT) pv[q] = 0.0;
  double w[SLOTS];
  double acc[NVP];
#pragma unroll
  for (int i = 0; i < NVP; ++i) acc[i] = 0.0;
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    w[s] = 0.0;
    if (own[s]) {
      int l = tid + s * NT;
      size_t g = (size_t)wrapi(gx0 + l % Ex, p.nx) + (size_t)p.nx * wrapi(gy0 + l / Ex, p.ny);
      w[s] = p.v[g];
      cl[l] = p.c[g];
      acc[0] += w[s] * w[s];
    }
  }
  int rb = 0;
  block_allreduce<NVP>(acc, 1, red + rb * NW * NVP, hx);
  rb ^= 1;
  const double beta = sqrt(hx[0]);
  if (beta == 0.0) {
    for (int l = tid; l < p.bx * p.by; l += NT)
      p.z[(size_t)(ibx * p.bx + l % p.bx) + (size_t)p.nx * (iby * p.by + l / p.bx)] = 0.0;
    return;
  }
  {
    const double ib = 1.0 / beta;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s)
      if (own[s]) {
        double v0 = w[s] * ib;
        V[tid + s * NT] = v0;
        pv[pidx[s]] = v0;
      }
  }
  if (tid == 0) gv[0] = beta;

  // stage iteration geometry, hoisted out of the Arnoldi loop (no integer division inside it)
  const int wxL = Px - 2, cntL = wxL * (Py - 2), r0L = tid / wxL, c0L = tid % wxL;
  const int wxB = Px - 4, cntB = wxB * (Py - 4), r0B = tid / wxB, c0B = tid % wxB;
  const int drL = NT / wxL, dcL = NT % wxL, drB = NT / wxB, dcB = NT % wxB;

  int jm = 0;
#pragma unroll 1
  for (int j = 0; j < K; ++j) {
    __syncthreads();                                   // pv holds V_j
    {   // L1 = Delta v on padded [1, P-1)
      int r = r0L, c = c0L;
      for (int q = tid; q < cntL; q += NT) {
        const int f = (1 + r) * Px + 1 + c;
        pl[f] = ih2 * ((pv[f - 1] + pv[f + 1]) + (pv[f - Px] + pv[f + Px]) - 4.0 * pv[f]);
        r += drL; c += dcL;
        if (c >= wxL) { c -= wxL; ++r; }
      }
    }
    __syncthreads();
    {   // B on padded [2, P-2); c v = 0 outside the extended box
      int r = r0B, c = c0B;
      for (int q = tid; q < cntB; q += NT) {
        const int pi = 2 + c, pj = 2 + r;
        r += drB; c += dcB;
        if (c >= wxB) { c -= wxB; ++r; }
        int f = pj * Px + pi;
        double vv = pv[f];
        int li = pi - 3, lj = pj - 3;
        double cv = (li >= 0 && li < Ex && lj >= 0 && lj < Ey) ? cl[lj * Ex + li] * vv : 0.0;
        double lapl = ih2 * ((pl[f - 1] + pl[f + 1]) + (pl[f - Px] + pl[f + Px]) - 4.0 * pl[f]);
        pb[f] = alpha * vv + cv + pl[f] + 0.5 * lapl;
      }
    }
    __syncthreads();
    // w = v/dt - Delta B on own nodes (registers); CGS2 pass 1: h1 = V^T w
#pragma unroll
    for (int i = 0; i < NVP; ++i) acc[i] = 0.0;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      if (own[s]) {
        const int f = pidx[s], l = tid + s * NT;
        double lapb = ih2 * ((pb[f - 1] + pb[f + 1]) + (pb[f - Px] + pb[f + Px]) - 4.0 * pb[f]);
        double ww = pv[f] * idt - lapb;
        w[s] = ww;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i > j) break;
          acc[i] += V[(size_t)i * n + l] * ww;
        }
      }
    }
    block_allreduce<NVP>(acc, j + 1, red + rb * NW * NVP, h1);
    rb ^= 1;
    // w' = w - V h1 ; pass 2: h2 = V^T w', and |w'|^2 (slot K of the reduction)
#pragma unroll
    for (int i = 0; i < NVP; ++i) acc[i] = 0.0;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      if (own[s]) {
        const int l = tid + s * NT;
        double vv[K];
        double ww = w[s];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i > j) break;
          vv[i] = V[(size_t)i * n + l];
          ww -= h1[i] * vv[i];
        }
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i > j) break;
          acc[i] += vv[i] * ww;
        }
        acc[NVP - 1] += ww * ww;
        w[s] = ww;
      }
    }
    block_allreduce<NVP>(acc, j + 1, red + rb * NW * NVP, h2, true);
    rb ^= 1;
    const double wn2 = h2[NVP - 1];
    double h2n = 0.0;
    for (int i = 0; i <= j; ++i) h2n += h2[i] * h2[i];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      if (own[s]) {
        const int l = tid + s * NT;
        double ww = w[s];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i > j) break;
          ww -= h2[i] * V[(size_t)i * n + l];
        }
        w[s] = ww;
      }
    }
    double hn2;
    if (h2n <= 1e-8 * wn2) {
      hn2 = wn2 - h2n;                                  // |w''|^2 = |w'|^2 - |h2|^2
    } else {                                            // rare: explicit |w''|^2
#pragma unroll
      for (int i = 0; i < NVP; ++i) acc[i] = 0.0;
#pragma unroll
      for (int s = 0; s < SLOTS; ++s)
        if (own[s]) acc[0] += w[s] * w[s];
      block_allreduce<NVP>(acc, 1, red + rb * NW * NVP, hx);
      rb ^= 1;
      hn2 = hx[0];
    }
    const double hn = sqrt(hn2 > 0.0 ? hn2 : 0.0);
    if (tid == 0) {   // Hessenberg column j (the Givens QR runs once, after the loop)
      const int ld = K + 1;
      for (int i = 0; i <= j; ++i) H[i + ld * j] = h1[i] + h2[i];
      H[j + 1 + ld * j] = hn;
    }
    jm = j + 1;
    if (hn <= 1e-14 * beta) break;                     // exact breakdown (uniform)
    if (j + 1 < K) {
      const double ihn = 1.0 / hn;
#pragma unroll
      for (int s = 0; s < SLOTS; ++s)
        if (own[s]) {
          double vn = w[s] * ihn;
          V[(size_t)(j + 1) * n + tid + s * NT] = vn;
          pv[pidx[s]] = vn;
        }
    }
  }
  __syncthreads();
  if (tid == 0) {
    // Givens QR of the (jm+1) x jm Hessenberg matrix, column by column in Arnoldi order (the
    // same operations an incremental update performs), then back substitution R y = g
    const int ld = K + 1;
    for (int j = 0; j < jm; ++j) {
      for (int i = 0; i < j; ++i) {
        double a = H[i + ld * j], b = H[i + 1 + ld * j];
        H[i + ld * j] = cs[i] * a + sn[i] * b;
        H[i + 1 + ld * j] = -sn[i] * a + cs[i] * b;
      }
      double a = H[j + ld * j], b = H[j + 1 + ld * j];
      double r = sqrt(a * a + b * b);
      double cc = 1.0, ss = 0.0;
      if (r != 0.0) { cc = a / r; ss = b / r; }
      cs[j] = cc; sn[j] = ss;
      H[j + ld * j] = cc * a + ss * b;
      H[j + 1 + ld * j] = 0.0;
      gv[j + 1] = -ss * gv[j];
      gv[j] = cc * gv[j];
    }
    for (int i = jm - 1; i >= 0; --i) {
      double s = gv[i];
      for (int l = i + 1; l < jm; ++l) s -= H[i + ld * l] * yv[l];
      yv[i] = s / H[i + ld * i];
    }
  }
  __syncthreads();
  // (R_k^0)^T: owned nodes only, y = V yv
  for (int l = tid; l < p.bx * p.by; l += NT) {
    int li = l % p.bx, lj = l / p.bx;
    int ll = (lj + p.o) * Ex + li + p.o;
    double s = 0.0;
    for (int i = 0; i < jm; ++i) s += yv[i] * V[(size_t)i * n + ll];
    p.z[(size_t)(ibx * p.bx + li) + (size_t)p.nx * (iby * p.by + lj)] = s;
  }
}

// ---------------------------------------------------------------------------------------
// Register-basis variant (extended boxes of up to SLOTS*NTT nodes, e.g. 36^2 on 384 threads x 4
// slots; 12 warps = 3 per SM sub-partition leaves up to 168 registers per thread):
// every thread keeps the K basis vectors of its own nodes in registers, so CGS2 touches no
// shared memory at all; shared memory holds only c and the three zero-padded stencil planes.
// Same arithmetic and order as ras2d_kernel (parity with the oracle).
#ifdef PFC_RAS_PROFILE
// diagnostic build only: thread 0 of block 0 records clock64() at phase boundaries and writes
// the deltas over z[0..] at exit (the output is garbage in this build)
#define RPROF(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) prof_t[i] += clock64() - prof_last; \
                      prof_last = clock64(); } while (0)
#else
#define RPROF(i) do {} while (0)
#endif

template <int K, int SLOTS, int NTT>
__global__ void __launch_bounds__(NTT, 1) ras2d_reg_kernel(RasArgs p) {
#ifdef PFC_RAS_PROFILE
  long long prof_t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long prof_last = clock64();
#endif
  constexpr int NVP = pow2_at_least(K + 2);
  constexpr int NWT = NTT / 32;
  extern __shared__ __align__(128) double smem_dyn[];
  const int Ex = p.bx + 2 * p.o, Ey = p.by + 2 * p.o;
  const int n = Ex * Ey;
  const int Px = Ex + 6, Py = Ey + 6;
  const int np = Px * Py;
  double* cl = smem_dyn;                 // n
  double* pv = cl + n;                   // np (zero ring)
  double* pl = pv + np;                  // np
  double* pb = pl + np;                  // np
  double* red = pb + np;                 // 2 x NWT x NVP
  double* hwall = red + 2 * NWT * NVP;   // NWT x 3 NVP
  __shared__ double H[(K + 1) * K];
  __shared__ double gv[K + 1], cs[K], sn[K], yv[K];

  const int tid = threadIdx.x;
  double* h1 = hwall + (tid >> 5) * 3 * NVP;
  double* h2 = h1 + NVP;
  double* hx = h2 + NVP;
  const int nbx = p.nx / p.bx;
  const int ibx = blockIdx.x % nbx, iby = blockIdx.x / nbx;
  const int gx0 = ibx * p.bx - p.o, gy0 = iby * p.by - p.o;
  const double ih2 = p.ih2, idt = p.idt, alpha = 0.5 * (1.0 - p.gamma);

  int pidx[SLOTS];
  bool own[SLOTS];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    const int l = tid + s * NTT;
    own[s] = l < n;
    pidx[s] = own[s] ? ((l / Ex) + 3) * Px + (l % Ex) + 3 : 0;
  }
  for (int q = tid; q < 3 * np; q += NTT) pv[q] = 0.0;
  double Vr[K][SLOTS];                    // basis, own nodes
  double w[SLOTS];
  double acc[NVP];
#pragma unroll
  for (int i = 0; i < NVP; ++i) acc[i] = 0.0;
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    w[s] = 0.0;
    if (own[s]) {
      const int l = tid + s * NTT;
      const size_t g = (size_t)wrapi(gx0 + l % Ex, p.nx) + (size_t)p.nx * wrapi(gy0 + l / Ex, p.ny);
      w[s] = p.v[g];
      cl[l] = p.c[g];
      acc[0] += w[s] * w[s];
    }
  }
  int rb = 0;
  block_allreduce<NVP, NWT>(acc, 1, red + rb * NWT * NVP, hx);
  rb ^= 1;
  const double beta = sqrt(hx[0]);
  if (beta == 0.0) {
    for (int l = tid; l < p.bx * p.by; l += NTT)
      p.z[(size_t)(ibx * p.bx + l % p.bx) + (size_t)p.nx * (iby * p.by + l / p.bx)] = 0.0;
    return;
  }
  {
    const double ib = 1.0 / beta;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const double v0 = w[s] * ib;
      Vr[0][s] = v0;
      if (own[s]) pv[pidx[s]] = v0;
    }
  }
  if (tid == 0) gv[0] = beta;

  const int wxL = Px - 2, cntL = wxL * (Py - 2), r0L = tid / wxL, c0L = tid % wxL;
  const int wxB = Px - 4, cntB = wxB * (Py - 4), r0B = tid / wxB, c0B = tid % wxB;
  const int drL = NTT / wxL, dcL = NTT % wxL, drB = NTT / wxB, dcB = NTT % wxB;

  int jm = 0;
  RPROF(0);
#pragma unroll 1
  for (int j = 0; j < K; ++j) {
    __syncthreads();                                   // pv holds V_j
    RPROF(1);
    {   // L1 = Delta v on padded [1, P-1)
      int r = r0L, c = c0L;
      for (int q = tid; q < cntL; q += NTT) {
        const int f = (1 + r) * Px + 1 + c;
        pl[f] = ih2 * ((pv[f - 1] + pv[f + 1]) + (pv[f - Px] + pv[f + Px]) - 4.0 * pv[f]);
        r += drL; c += dcL;
        if (c >= wxL) { c -= wxL; ++r; }
      }
    }
    __syncthreads();
    {   // B on padded [2, P-2); c v = 0 outside the extended box
      int r = r0B, c = c0B;
      for (int q = tid; q < cntB; q += NTT) {
        const int pi = 2 + c, pj = 2 + r;
        r += drB; c += dcB;
        if (c >= wxB) { c -= wxB; ++r; }
        const int f = pj * Px + pi;
        const double vv = pv[f];
        const int li = pi - 3, lj = pj - 3;
        const double cv = (li >= 0 && li < Ex && lj >= 0 && lj < Ey) ? cl[lj * Ex + li] * vv : 0.0;
        const double lapl = ih2 * ((pl[f - 1] + pl[f + 1]) + (pl[f - Px] + pl[f + Px]) - 4.0 * pl[f]);
        pb[f] = alpha * vv + cv + pl[f] + 0.5 * lapl;
      }
    }
    __syncthreads();
    RPROF(2);
    // w = v/dt - Delta B (registers); CGS2 pass 1: h1 = V^T w
#pragma unroll
    for (int i = 0; i < NVP; ++i) acc[i] = 0.0;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      if (own[s]) {
        const int f = pidx[s];
        const double lapb = ih2 * ((pb[f - 1] + pb[f + 1]) + (pb[f - Px] + pb[f + Px]) - 4.0 * pb[f]);
        w[s] = pv[f] * idt - lapb;
      } else {
        w[s] = 0.0;
      }
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (i > j) break;
        acc[i] += Vr[i][s] * w[s];
      }
    }
    RPROF(3);
    block_allreduce<NVP, NWT>(acc, j + 1, red + rb * NWT * NVP, h1);
    rb ^= 1;
    RPROF(4);
    // w' = w - V h1 ; pass 2: h2 = V^T w' and |w'|^2 (norm slot NVP-1)
#pragma unroll
    for (int i = 0; i < NVP; ++i) acc[i] = 0.0;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      double ww = w[s];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (i > j) break;
        ww -= h1[i] * Vr[i][s];
      }
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (i > j) break;
        acc[i] += Vr[i][s] * ww;
      }
      acc[NVP - 1] += ww * ww;
      w[s] = ww;
    }
    RPROF(5);
    block_allreduce<NVP, NWT>(acc, j + 1, red + rb * NWT * NVP, h2, true);
    rb ^= 1;
    RPROF(6);
    const double wn2 = h2[NVP - 1];
    double h2n = 0.0;
    for (int i = 0; i <= j; ++i) h2n += h2[i] * h2[i];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      double ww = w[s];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (i > j) break;
        ww -= h2[i] * Vr[i][s];
      }
      w[s] = ww;
    }
    double hn2;
    if (h2n <= 1e-8 * wn2) {
      hn2 = wn2 - h2n;                                  // |w''|^2 = |w'|^2 - |h2|^2
    } else {                                            // rare: explicit |w''|^2
#pragma unroll
      for (int i = 0; i < NVP; ++i) acc[i] = 0.0;
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) acc[0] += w[s] * w[s];
      block_allreduce<NVP, NWT>(acc, 1, red + rb * NWT * NVP, hx);
      rb ^= 1;
      hn2 = hx[0];
    }
    const double hn = sqrt(hn2 > 0.0 ? hn2 : 0.0);
    if (tid == 0) {
      const int ld = K + 1;
      for (int i = 0; i <= j; ++i) H[i + ld * j] = h1[i] + h2[i];
      H[j + 1 + ld * j] = hn;
    }
    jm = j + 1;
    if (hn <= 1e-14 * beta) break;                     // exact breakdown (uniform)
    if (j + 1 < K) {
      const double ihn = 1.0 / hn;
#pragma unroll
      for (int s = 0; s < SLOTS; ++s) {
        const double vn = w[s] * ihn;
#pragma unroll
        for (int i = 1; i < K; ++i)
          if (i == j + 1) Vr[i][s] = vn;               // compile-time register index
        if (own[s]) pv[pidx[s]] = vn;
      }
    }
    RPROF(7);
  }
  __syncthreads();
#ifdef PFC_RAS_PROFILE
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) p.z[i] = (double)prof_t[i];
  }
  return;
#endif
  if (tid == 0) {
    const int ld = K + 1;
    for (int j = 0; j < jm; ++j) {
      for (int i = 0; i < j; ++i) {
        const double a = H[i + ld * j], b = H[i + 1 + ld * j];
        H[i + ld * j] = cs[i] * a + sn[i] * b;
        H[i + 1 + ld * j] = -sn[i] * a + cs[i] * b;
      }
      const double a = H[j + ld * j], b = H[j + 1 + ld * j];
      const double r = sqrt(a * a + b * b);
      double cc = 1.0, ss = 0.0;
      if (r != 0.0) { cc = a / r; ss = b / r; }
      cs[j] = cc; sn[j] = ss;
      H[j + ld * j] = cc * a + ss * b;
      H[j + 1 + ld * j] = 0.0;
      gv[j + 1] = -ss * gv[j];
      gv[j] = cc * gv[j];
    }
    for (int i = jm - 1; i >= 0; --i) {
      double s2 = gv[i];
      for (int l = i + 1; l < jm; ++l) s2 -= H[i + ld * l] * yv[l];
      yv[i] = s2 / H[i + ld * i];
    }
  }
  __syncthreads();
  // (R_k^0)^T: the owner thread of each owned node writes y = V yv
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    if (!own[s]) continue;
    const int l = tid + s * NTT;
    const int li = l % Ex - p.o, lj = l / Ex - p.o;
    if (li < 0 || li >= p.bx || lj < 0 || lj >= p.by) continue;
    double acc2 = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i >= jm) break;
      acc2 += yv[i] * Vr[i][s];
    }
    p.z[(size_t)(ibx * p.bx + li) + (size_t)p.nx * (iby * p.by + lj)] = acc2;
  }
}

size_t ras2d_reg_smem_bytes(int bx, int by, int o, int ntt) {
  const size_t Ex = bx + 2 * o, Ey = by + 2 * o, n = Ex * Ey, np = (Ex + 6) * (Ey + 6);
  const size_t nw = ntt / 32;
  return (n + 3 * np + 2 * nw * 16 + nw * 3 * 16) * sizeof(double);
}

typedef void (*ras2d_fn)(RasArgs);
size_t ras2d_smem_bytes(int bx, int by, int o, int k) {
  const size_t Ex = bx + 2 * o, Ey = by + 2 * o, n = Ex * Ey, np = (Ex + 6) * (Ey + 6);
  size_t d = (size_t)k * n + n + 3 * np + 2 * NW * 16 + NW * 3 * 16;
  return d * sizeof(double) + 128;
}

ras2d_fn pick(int k) {
  switch (k) {
#define X(K) case K: return ras2d_kernel<K>;
    X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15)
#undef X
  }
  return nullptr;
}

// register-basis instantiations: (SLOTS, threads) covering extended boxes up to SLOTS*threads
ras2d_fn pick_reg(int k, int n, int* ntt) {
#define RK(K)                                                                       \
  case K:                                                                           \
    if (n <= 256 * 2) { *ntt = 256; return ras2d_reg_kernel<K, 2, 256>; }         \
    if (n <= 384 * 4) { *ntt = 384; return ras2d_reg_kernel<K, 4, 384>; }         \
    return nullptr;
  switch (k) {
    RK(1) RK(2) RK(3) RK(4) RK(5) RK(6) RK(7) RK(8) RK(9) RK(10) RK(11) RK(12)
  }
#undef RK
  return nullptr;
}

}  // namespace

int ras2d_plan(pfc_ctx* ctx) {
  const pfc_config& c = ctx->cfg;
  const int Ex = c.ras_box[0] + 2 * c.ras_overlap, Ey = c.ras_box[1] + 2 * c.ras_overlap;
  if (Ex * Ey > MAXN) return 0;
  int ntt = 0;
  if (getenv("PFC_RAS_SMEM_BASIS") == nullptr && pick_reg(c.ras_local_k, Ex * Ey, &ntt)) {
    ctx->ras_smem = (int)ras2d_reg_smem_bytes(c.ras_box[0], c.ras_box[1], c.ras_overlap, ntt);
    ctx->ras_threads = ntt;     // register-basis kernel
    ctx->ras_cluster = 0;
    return 1;
  }
  size_t sm = ras2d_smem_bytes(c.ras_box[0], c.ras_box[1], c.ras_overlap, c.ras_local_k);
  if (sm + 2048 > 227 * 1024) return 0;   // + static shared memory (H, Givens, reductions)
  ctx->ras_smem = (int)sm;
  ctx->ras_threads = NT;        // shared-memory-basis kernel
  ctx->ras_cluster = 1;
  return 1;
}

cudaError_t launch_ras_2d(pfc_ctx* ctx, const double* v, const double* c, double dt, double* z) {
  const pfc_config& cf = ctx->cfg;
  const int Ex = cf.ras_box[0] + 2 * cf.ras_overlap, Ey = cf.ras_box[1] + 2 * cf.ras_overlap;
  int ntt = NT;
  ras2d_fn fn = ctx->ras_cluster == 0 ? pick_reg(cf.ras_local_k, Ex * Ey, &ntt)
                                      : pick(cf.ras_local_k);
  if (!fn) return cudaErrorInvalidValue;
  // opt in to the dynamic shared memory once per kernel
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       ctx->ras_smem);
  if (e != cudaSuccess) return e;
  RasArgs p{v, c, z, cf.n[0], cf.n[1], cf.ras_box[0], cf.ras_box[1], cf.ras_overlap,
            1.0 / dt, cf.gamma, ctx->ih2};
  const int nb = (cf.n[0] / cf.ras_box[0]) * (cf.n[1] / cf.ras_box[1]);
  fn<<<nb, ntt, ctx->ras_smem, ctx->stream>>>(p);
  ctx->launches++;
  {  // algorithmic: v, c gathered on the extended boxes, z written on owned nodes; flops of
     // k local J v (25/pt) + CGS2 vector work 4k(k+1) + 3k + 3 per ext node + V y
    const double k = cf.ras_local_k;
    const double next = (double)nb * (cf.ras_box[0] + 2 * cf.ras_overlap) *
                        (cf.ras_box[1] + 2 * cf.ras_overlap);
    pfc_account(ctx, PFC_K_RAS, 8.0 * (2.0 * next + ctx->N),
                next * (25.0 * k + 4.0 * k * (k + 1) + 3.0 * k + 3.0) + 2.0 * k * ctx->N);
  }
  return cudaGetLastError();
}
