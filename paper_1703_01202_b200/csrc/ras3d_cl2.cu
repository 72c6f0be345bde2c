// ras3d_cl2.cu -- 3D Schwarz subdomain solves on a 2-CTA cluster with the WHOLE Krylov basis
// on chip (K4, sm_100a).
//
// Same algorithm as the oracle and the other subdomain kernels: Eq. (eq:ras) P:398-409 (and
// the AS / right-RAS variants P:387-419), the modified subdomain BC phi = 0 on the 3-layer ring
// outside the extended box as zero padding, and exactly K steps of GMRES with a
// zero initial guess, CGS2 and Givens (reading R9), exit only on exact breakdown.
//
// Why a cluster: one extended box of E^3 = 20^3 nodes has a K = 10 basis of 640 KB, more than
// one SM holds (228 KB shared + 256 KB registers); the single-CTA column kernel keeps it in an
// L2 scratch whose three passes per Arnoldi step are bound by the ~12 TB/s L2 (and spill to
// HBM).  Two CTAs of a cluster (two SMs) split the box into z-halves of ZL = E/2 planes:
//  * thread (x, y) owns the ZL nodes of its z-column in its half;
//  * basis vectors 0..NR-1 live in registers (NR = 3: 30 doubles per thread; 13 warps on 4 SM
//    sub-partitions cap a thread at 128 registers), NR..NR+NS-1 in shared memory (NS = 4),
//    the last NG = 2 in a small per-CTA global scratch (64 KB per CTA, 9.5 MB in all: L2-
//    resident, read only by Arnoldi steps >= 8), and v_{K-1} in the stencil planes;
//  * the current vector v_j sits in ZL + 3 unpadded 20x20 planes (the own ZL planes plus the 3
//    halo planes on the partner's side, written by the partner through DSMEM; beyond the box
//    the planes are zero by the modified BC and are never read); the x/y zero ring is a
//    bounds mask on the 24 neighbour columns;
//  * c' = -c/h^2 on the own planes plus the one plane on the partner's side (static per box);
//  * w = A_k v_j is the direct 63-point stencil of the linear part plus -Delta(c v) (class
//    weights of h^2 Delta = L, L^2, L^3 summed on the host), evaluated column by column with
//    the symmetric neighbour columns summed first (4 / 4+4 / 4+8 columns per ring R = 1, 2, 3
//    share one z-weight profile), about 48 FP64 operations per node instead of 71;
//  * the halo exchange is split-phase: arrive (release) after writing v_j, accumulate the own
//    planes' contributions, wait (acquire), then the halo planes';
//  * every inner product is a cluster all-reduce: a fixed xor-butterfly per warp, the warp
//    partials stored into both CTAs' shared memory, one cluster barrier, then a fixed-order
//    sum of the 2 x NW partials -- both CTAs obtain bitwise identical values and therefore take
//    identical decisions (breakdown, Givens, back substitution run redundantly on both);
//  * persistent: cluster c walks the boxes c, c + #clusters, ...
#include "pfc_device.cuh"
#include "pfc_internal.h"
#include "ras_common.cuh"

namespace {

constexpr int RS = 12;   // reduction slot stride (>= K + 1 values)

struct Ras3Cl2Args {
  const double* v;
  const double* c;
  double* z;
  double* gscr;          // per-CTA basis scratch: NG x ZL x PL doubles per CTA
  int nx, ny, nz, bx, by, bz, o;
  int restrict_owned;    // right-RAS: R_k^0
  double* y_ext;         // AS / right-RAS: ext-box solutions [box][ext node]
  const int* gate;       // device-resident FGMRES: skip when *gate != 0
  double W[7];           // classes (0,0,0) (0,0,1) (0,0,2) (0,1,1) (0,0,3) (0,1,2) (1,1,1)
  double ih2;
  unsigned long long* jcnt;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void cl_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_sync() {
  cl_arrive();
  cl_wait();
}

template <int E>
struct Cl2 {
  static constexpr int ZL = E / 2;                 // own z-planes per CTA
  static constexpr int PL = E * E;                 // plane size (unpadded)
  static constexpr int NT = (PL + 31) / 32 * 32;   // threads
  static constexpr int NW = NT / 32;
  static constexpr int NVB = ZL + 3;   // v_j planes: own + 3 on the partner's side
  static constexpr int NCB = ZL + 1;   // c' planes: own + 1 on the partner's side
};

template <int K>
struct Cl2K {
  static constexpr int NR = (K - 1) < 3 ? (K - 1) : 3;                     // registers
  static constexpr int NS = (K - 1 - NR) < 4 ? (K - 1 - NR) : 4;          // shared memory
  static constexpr int NG = K - 1 - NR - NS;                               // global scratch
};

template <int K, int E>
constexpr size_t cl2_smem_doubles() {
  return (size_t)Cl2<E>::NVB * Cl2<E>::PL + (size_t)Cl2<E>::NCB * Cl2<E>::PL +
         (size_t)Cl2K<K>::NS * Cl2<E>::ZL * Cl2<E>::PL + 2 * 2 * Cl2<E>::NW * RS +
         Cl2<E>::NW * 3 * RS;
}

// Warp partial of one inner-product value: fixed xor butterfly, lane 0 stores it into slot
// [rank][warp][i] of the reduction buffer in BOTH CTAs (local store + DSMEM store).
template <int NW>
__device__ __forceinline__ void cl2_put(double s, int i, double* redb, uint32_t redb_rem,
                                        int rank, int wid, int lane) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const int off = (rank * NW + wid) * RS + i;
    redb[off] = s;
    st_cluster(redb_rem + off * 8u, s);
  }
}

// After the cluster barrier: lanes < nv sum the 2 x NW warp partials of value `lane` in a fixed
// order (rank 0's warps, then rank 1's) into this warp's copy hwv[lane].
template <int NW>
__device__ __forceinline__ void cl2_get(int nv, const double* redb, double* hwv, int lane) {
  if (lane < nv) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 2 * NW; ++q) t += redb[q * RS + lane];
    hwv[lane] = t;
  }
  __syncwarp();
}

// Contributions of the v_j planes zz in [LO, HI) to the thread's ZL outputs (all bounds
// compile-time: out[] stays in registers).  pv -> own column at zl = 0 of the v_j planes,
// pc -> own column at zl = 0 of the c' planes.  Neighbour columns outside the extended box
// are zero (the modified BC), hence the x/y masks.
template <int E, int LO, int HI>
__device__ __forceinline__ void cl2_stencil(const Ras3Cl2Args& p, const double* pv,
                                            const double* pc, int x, int y, double (&out)[E / 2]) {
  constexpr int ZL = E / 2, PL = E * E;
  const double W0 = p.W[0], W1 = p.W[1], W2 = p.W[2], W3 = p.W[3], W4 = p.W[4], W5 = p.W[5],
               W6 = p.W[6];
  auto ok = [&](int dx, int dy) {
    return (unsigned)(x + dx) < (unsigned)E && (unsigned)(y + dy) < (unsigned)E;
  };
  auto ld = [&](int dx, int dy, int zz) -> double {
    return ok(dx, dy) ? pv[zz * PL + dx + E * dy] : 0.0;
  };
  // R = 0: own column, z-reach 3; with the z-neighbour and centre terms of -Delta(c v)
#pragma unroll
  for (int zz = (LO > -3 ? LO : -3); zz < (HI < ZL + 3 ? HI : ZL + 3); ++zz) {
    const double val = pv[zz * PL];
#pragma unroll
    for (int z = (zz - 3 > 0 ? zz - 3 : 0); z <= (zz + 3 < ZL - 1 ? zz + 3 : ZL - 1); ++z) {
      const int dz = zz > z ? zz - z : z - zz;
      const double wgt = dz == 0 ? W0 : dz == 1 ? W1 : dz == 2 ? W2 : W4;
      out[z] = fma(wgt, val, out[z]);
    }
    if (zz >= -1 && zz <= ZL) {
      const double cv = pc[zz * PL] * val;            // c' v, c' = -c / h^2
      if (zz - 1 >= 0 && zz - 1 < ZL) out[zz - 1] += cv;
      if (zz + 1 >= 0 && zz + 1 < ZL) out[zz + 1] += cv;
      if (zz >= 0 && zz < ZL) out[zz] = fma(-6.0, cv, out[zz]);
    }
  }
  // R = 1: (+-1, 0), (0, +-1), z-reach 2 (weights W1, W3, W5); -Delta(c v) xy-neighbours
#pragma unroll
  for (int zz = (LO > -2 ? LO : -2); zz < (HI < ZL + 2 ? HI : ZL + 2); ++zz) {
    const double a = ld(-1, 0, zz), b = ld(1, 0, zz), cc = ld(0, -1, zz), d = ld(0, 1, zz);
    const double s = (a + b) + (cc + d);
#pragma unroll
    for (int z = (zz - 2 > 0 ? zz - 2 : 0); z <= (zz + 2 < ZL - 1 ? zz + 2 : ZL - 1); ++z) {
      const int dz = zz > z ? zz - z : z - zz;
      out[z] = fma(dz == 0 ? W1 : dz == 1 ? W3 : W5, s, out[z]);
    }
    if (zz >= 0 && zz < ZL) {
      double t = out[zz];
      if (ok(-1, 0)) t = fma(pc[zz * PL - 1], a, t);
      if (ok(1, 0)) t = fma(pc[zz * PL + 1], b, t);
      if (ok(0, -1)) t = fma(pc[zz * PL - E], cc, t);
      if (ok(0, 1)) t = fma(pc[zz * PL + E], d, t);
      out[zz] = t;
    }
  }
  // R = 2: axis (+-2, 0), (0, +-2) [W2, W5] and diagonal (+-1, +-1) [W3, W6], z-reach 1
#pragma unroll
  for (int zz = (LO > -1 ? LO : -1); zz < (HI < ZL + 1 ? HI : ZL + 1); ++zz) {
    const double sa = (ld(-2, 0, zz) + ld(2, 0, zz)) + (ld(0, -2, zz) + ld(0, 2, zz));
    const double sb = (ld(-1, -1, zz) + ld(1, -1, zz)) + (ld(-1, 1, zz) + ld(1, 1, zz));
#pragma unroll
    for (int z = (zz - 1 > 0 ? zz - 1 : 0); z <= (zz + 1 < ZL - 1 ? zz + 1 : ZL - 1); ++z) {
      const bool d0 = z == zz;
      out[z] = fma(d0 ? W2 : W5, sa, out[z]);
      out[z] = fma(d0 ? W3 : W6, sb, out[z]);
    }
  }
  // R = 3: axis (+-3, 0), (0, +-3) [W4] and (+-1, +-2), (+-2, +-1) [W5], same plane only
#pragma unroll
  for (int zz = (LO > 0 ? LO : 0); zz < (HI < ZL ? HI : ZL); ++zz) {
    const double sa = (ld(-3, 0, zz) + ld(3, 0, zz)) + (ld(0, -3, zz) + ld(0, 3, zz));
    const double sb = ((ld(-1, -2, zz) + ld(1, -2, zz)) + (ld(-2, -1, zz) + ld(2, -1, zz))) +
                      ((ld(-2, 1, zz) + ld(2, 1, zz)) + (ld(-1, 2, zz) + ld(1, 2, zz)));
    out[zz] = fma(W4, sa, out[zz]);
    out[zz] = fma(W5, sb, out[zz]);
  }
}

template <int K, int E>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cl2<E>::NT, 1)
    ras3d_cl2_kernel(const __grid_constant__ Ras3Cl2Args p) {
  if (p.gate && *p.gate) return;     // uniform over the cluster: both CTAs leave at once
  constexpr int ZL = Cl2<E>::ZL, PL = Cl2<E>::PL, NW = Cl2<E>::NW;
  constexpr int NVB = Cl2<E>::NVB, NCB = Cl2<E>::NCB;
  constexpr int NR = Cl2K<K>::NR, NS = Cl2K<K>::NS, NG = Cl2K<K>::NG;
  constexpr int NE = E * E * E;
  extern __shared__ __align__(128) double smem_dyn[];
  double* vb = smem_dyn;                 // NVB planes: v_j (rank 0: zl in [0, ZL+3), rank 1: [-3, ZL))
  double* cb = vb + NVB * PL;            // NCB planes: c' = -c/h^2 (rank 0: [0, ZL], rank 1: [-1, ZL))
  double* vs = cb + NCB * PL;            // NS x ZL x PL: basis vectors NR..K-2
  double* red = vs + NS * ZL * PL;       // 2 buffers x [rank][warp][RS]
  double* hw = red + 2 * 2 * NW * RS;    // per warp: h1, h2, scratch
  __shared__ double H[(K + 1) * K];
  __shared__ double gv[K + 1], cs[K], sn[K], yv[K];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int rank = (int)cluster_rank(), partner = rank ^ 1;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const bool act = tid < PL;
  const int x = act ? tid % E : 0, y = act ? tid / E : 0;
  const int pv0 = rank == 0 ? 0 : 3, pc0 = rank == 0 ? 0 : 1;   // plane of zl = 0
  const double* pv = vb + pv0 * PL + tid;          // own column, zl = 0
  const double* pc = cb + pc0 * PL + tid;
  double* gs = p.gscr + (size_t)blockIdx.x * (NG > 0 ? NG : 1) * ZL * PL + tid;
  double* h1 = hw + wid * 3 * RS;
  double* h2 = h1 + RS;
  double* hx = h2 + RS;
  const uint32_t red_rem = mapa_rank(smem_u32(red), (uint32_t)partner);
  const uint32_t vb_rem = mapa_rank(smem_u32(vb), (uint32_t)partner);
  const int nbx = p.nx / p.bx, nby = p.ny / p.by, nbz = p.nz / p.bz;
  const int nboxes = nbx * nby * nbz;
  const size_t NX = p.nx, NXY = (size_t)p.nx * p.ny;

  cl_sync();   // the partner is running before any DSMEM store

  double vr[NR > 0 ? NR : 1][ZL];
  int rb = 0;
  for (int box = cid; box < nboxes; box += ncl) {
    const int ibx = box % nbx, iby = (box / nbx) % nby, ibz = box / (nbx * nby);
    const int gx0 = ibx * p.bx - p.o, gy0 = iby * p.by - p.o, gz0 = ibz * p.bz - p.o;
    const int ez0 = rank * ZL;                     // ext-box z of own plane zl = 0
    double w[ZL];
    double acc = 0.0;
    if (act) {
      const size_t gxy = (size_t)wrapi(gx0 + x, p.nx) + NX * wrapi(gy0 + y, p.ny);
      const bool oxy = x >= p.o && x < p.o + p.bx && y >= p.o && y < p.o + p.by;
#pragma unroll
      for (int zl = 0; zl < ZL; ++zl) {
        const size_t g = gxy + NXY * wrapi(gz0 + ez0 + zl, p.nz);
        const int ez = ez0 + zl;
        const bool owned = oxy && ez >= p.o && ez < p.o + p.bz;
        w[zl] = (p.restrict_owned && !owned) ? 0.0 : p.v[g];
        cb[(zl + pc0) * PL + tid] = -p.ih2 * p.c[g];
        acc = fma(w[zl], w[zl], acc);
      }
      // the c' plane on the partner's side (inside the box): zl = ZL (rank 0) / -1 (rank 1)
      const int zh = rank == 0 ? ZL : -1;
      cb[(zh + pc0) * PL + tid] = -p.ih2 * p.c[gxy + NXY * wrapi(gz0 + ez0 + zh, p.nz)];
    } else {
#pragma unroll
      for (int zl = 0; zl < ZL; ++zl) w[zl] = 0.0;
    }
    double* redb = red + rb * 2 * NW * RS;
    uint32_t redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
    cl2_put<NW>(acc, 0, redb, redr, rank, wid, lane);
    cl_sync();
    cl2_get<NW>(1, redb, hx, lane);
    rb ^= 1;
    const double beta = sqrt(hx[0]);
    if (beta == 0.0) {
      if (act) {
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) {
          const int ez = ez0 + zl, li = x - p.o, lj = y - p.o, lk = ez - p.o;
          if (p.y_ext) p.y_ext[(size_t)box * NE + (ez * E + y) * E + x] = 0.0;
          else if (li >= 0 && li < p.bx && lj >= 0 && lj < p.by && lk >= 0 && lk < p.bz)
            p.z[(size_t)(ibx * p.bx + li) + NX * (iby * p.by + lj) + NXY * (ibz * p.bz + lk)] = 0.0;
        }
      }
      if (tid == 0 && rank == 0) ras_count(p.jcnt, 0);
      continue;   // uniform over the cluster
    }
    // v_j into basis slot `slot`, the own v_j planes and the partner's halo planes
    auto put_v = [&](int slot) {
      if (!act) return;
#pragma unroll
      for (int s = 0; s < NR; ++s)
        if (s == slot) {
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) vr[s][zl] = w[zl];
        }
      if (slot >= NR && slot < NR + NS) {
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) vs[((slot - NR) * ZL + zl) * PL + tid] = w[zl];
      } else if (slot >= NR + NS && slot < K - 1) {
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) gs[((slot - NR - NS) * ZL + zl) * PL] = w[zl];
      }
#pragma unroll
      for (int zl = 0; zl < ZL; ++zl) vb[(zl + pv0) * PL + tid] = w[zl];
      if (rank == 0) {   // own planes ZL-3..ZL-1 -> partner's zl' = -3..-1 (its planes 0..2)
#pragma unroll
        for (int q = 0; q < 3; ++q)
          st_cluster(vb_rem + (uint32_t)(q * PL + tid) * 8u, w[ZL - 3 + q]);
      } else {           // own planes 0..2 -> partner's zl' = ZL..ZL+2 (its planes ZL..ZL+2)
#pragma unroll
        for (int q = 0; q < 3; ++q)
          st_cluster(vb_rem + (uint32_t)((ZL + q) * PL + tid) * 8u, w[q]);
      }
    };
    // basis value i of the thread's node zl (i compile-time after unrolling)
    auto V = [&](int i, int zl) -> double {
      if (i < NR) return vr[i < NR ? i : 0][zl];
      if (i < NR + NS) return vs[((i - NR) * ZL + zl) * PL + tid];
      if (i < K - 1) return gs[((i - NR - NS) * ZL + zl) * PL];
      return pv[zl * PL];                            // v_{K-1}: only in the v_j planes
    };
    {
      const double ib = 1.0 / beta;
#pragma unroll
      for (int zl = 0; zl < ZL; ++zl) w[zl] *= ib;
      put_v(0);
    }
    if (tid == 0) gv[0] = beta;
    int jm = 0;
#pragma unroll 1
    for (int j = 0; j < K; ++j) {
      // ---- w = A_k v_j: own planes while the partner's halo planes are in flight
      cl_arrive();
      __syncthreads();
#pragma unroll
      for (int zl = 0; zl < ZL; ++zl) w[zl] = 0.0;
      if (act) cl2_stencil<E, 0, ZL>(p, pv, pc, x, y, w);
      cl_wait();
      if (act) {
        if (rank == 0) cl2_stencil<E, ZL, ZL + 3>(p, pv, pc, x, y, w);
        else cl2_stencil<E, -3, 0>(p, pv, pc, x, y, w);
      }
      // ---- CGS2 pass 1: h1 = V^T w
      redb = red + rb * 2 * NW * RS;
      redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
#pragma unroll
      for (int i = 0; i < K; ++i)
        if (i <= j) {
          double s = 0.0;
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) s = fma(V(i, zl), w[zl], s);
          cl2_put<NW>(s, i, redb, redr, rank, wid, lane);
        }
      cl_sync();
      cl2_get<NW>(j + 1, redb, h1, lane);
      rb ^= 1;
      // ---- pass 2: w' = w - V h1, h2 = V^T w', |w'|^2
#pragma unroll
      for (int i = 0; i < K; ++i)
        if (i <= j) {
          const double hi = h1[i];
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) w[zl] = fma(-hi, V(i, zl), w[zl]);
        }
      redb = red + rb * 2 * NW * RS;
      redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
#pragma unroll
      for (int i = 0; i < K; ++i)
        if (i <= j) {
          double s = 0.0;
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) s = fma(V(i, zl), w[zl], s);
          cl2_put<NW>(s, i, redb, redr, rank, wid, lane);
        }
      {
        double s = 0.0;
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) s = fma(w[zl], w[zl], s);
        cl2_put<NW>(s, j + 1, redb, redr, rank, wid, lane);
      }
      cl_sync();
      cl2_get<NW>(j + 2, redb, h2, lane);
      rb ^= 1;
      double h2n = 0.0;
      for (int i = 0; i <= j; ++i) h2n += h2[i] * h2[i];
      const double wn2 = h2[j + 1];
      // ---- pass 3: w'' = w' - V h2
#pragma unroll
      for (int i = 0; i < K; ++i)
        if (i <= j) {
          const double hi = h2[i];
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) w[zl] = fma(-hi, V(i, zl), w[zl]);
        }
      double hn2;
      if (h2n <= 1e-8 * wn2) {
        hn2 = wn2 - h2n;                             // |w''|^2 = |w'|^2 - |h2|^2
      } else {
        redb = red + rb * 2 * NW * RS;
        redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
        double s = 0.0;
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) s = fma(w[zl], w[zl], s);
        cl2_put<NW>(s, 0, redb, redr, rank, wid, lane);
        cl_sync();
        cl2_get<NW>(1, redb, hx, lane);
        rb ^= 1;
        hn2 = hx[0];
      }
      const double hn = sqrt(hn2 > 0.0 ? hn2 : 0.0);
      if (tid == 0) {   // Hessenberg column j: previous rotations, a new one (oracle order)
        double col[K + 1];
#pragma unroll
        for (int i = 0; i <= K; ++i) col[i] = 0.0;
        for (int i = 0; i <= j; ++i) col[i] = h1[i] + h2[i];
        col[j + 1] = hn;
        for (int i = 0; i < j; ++i) {
          const double a = col[i], b = col[i + 1];
          col[i] = cs[i] * a + sn[i] * b;
          col[i + 1] = -sn[i] * a + cs[i] * b;
        }
        const double a = col[j], b = col[j + 1];
        const double rr = sqrt(a * a + b * b);
        double cc = 1.0, ss = 0.0;
        if (rr != 0.0) { cc = a / rr; ss = b / rr; }
        cs[j] = cc; sn[j] = ss;
        col[j] = cc * a + ss * b;
        const double g = gv[j];
        gv[j + 1] = -ss * g;
        gv[j] = cc * g;
        for (int i = 0; i <= j; ++i) H[i + (K + 1) * j] = col[i];
      }
      jm = j + 1;
      if (hn <= 1e-14 * beta) break;                 // exact breakdown (identical on both CTAs)
      if (j + 1 < K) {
        const double ihn = 1.0 / hn;
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) w[zl] *= ihn;
        put_v(j + 1);
      }
    }
    __syncthreads();
    if (tid == 0) {   // back substitution R yv = g (R reduced column by column)
      const int ld = K + 1;
      for (int i = jm - 1; i >= 0; --i) {
        double s = gv[i];
        for (int l = i + 1; l < jm; ++l) s -= H[i + ld * l] * yv[l];
        yv[i] = s / H[i + ld * i];
      }
      if (rank == 0) ras_count(p.jcnt, jm);
    }
    __syncthreads();
    if (act) {
      double yl[ZL];
#pragma unroll
      for (int zl = 0; zl < ZL; ++zl) yl[zl] = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i)
        if (i < jm) {
          const double yi = yv[i];
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) yl[zl] = fma(yi, V(i, zl), yl[zl]);
        }
#pragma unroll
      for (int zl = 0; zl < ZL; ++zl) {
        const int ez = ez0 + zl, li = x - p.o, lj = y - p.o, lk = ez - p.o;
        if (p.y_ext) {
          p.y_ext[(size_t)box * NE + (ez * E + y) * E + x] = yl[zl];
        } else if (li >= 0 && li < p.bx && lj >= 0 && lj < p.by && lk >= 0 && lk < p.bz) {
          p.z[(size_t)(ibx * p.bx + li) + NX * (iby * p.by + lj) + NXY * (ibz * p.bz + lk)] =
              yl[zl];
        }
      }
    }
  }
  cl_sync();   // no CTA leaves while its partner may still address its shared memory
}

typedef void (*ras3cl2_fn)(const Ras3Cl2Args);

ras3cl2_fn pick_cl2(int k, int e, size_t* smem, int* threads) {
#define C2(K, E)                                                \
  if (k == K && e == E) {                                       \
    *smem = cl2_smem_doubles<K, E>() * sizeof(double);          \
    *threads = Cl2<E>::NT;                                      \
    return ras3d_cl2_kernel<K, E>;                              \
  }
  C2(10, 20) C2(4, 20) C2(10, 12) C2(4, 12)
#undef C2
  return nullptr;
}

}  // namespace

// 1 if the 2-CTA cluster kernel handles this configuration (cubic extended box with an even
// edge, instantiated K and E, periodic, M = 1); *clusters = concurrent clusters to launch
int ras3d_cl2_plan(pfc_ctx* ctx, int* clusters, size_t* scratch_doubles) {
  const pfc_config& c = ctx->cfg;
  const int e = c.ras_box[0] + 2 * c.ras_overlap;
  if (c.ras_box[1] != c.ras_box[0] || c.ras_box[2] != c.ras_box[0] || (e & 1)) return 0;
  size_t smem = 0;
  int threads = 0;
  if (!pick_cl2(c.ras_local_k, e, &smem, &threads)) return 0;
  if (smem + 2048 > 227 * 1024) return 0;
  const int nboxes = (c.n[0] / c.ras_box[0]) * (c.n[1] / c.ras_box[1]) * (c.n[2] / c.ras_box[2]);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  *clusters = nboxes < sms / 2 ? nboxes : sms / 2;
  const int ng = c.ras_local_k - 1 - 3 - 4;   // Cl2K<K>::NG
  *scratch_doubles = (size_t)2 * (*clusters) * (ng > 0 ? ng : 1) * (e / 2) * e * e;
  return 1;
}

cudaError_t launch_ras_3d_cl2(pfc_ctx* ctx, const double* v, const double* c, double dt,
                              double* z, double* scratch) {
  const pfc_config& cf = ctx->cfg;
  const int e = cf.ras_box[0] + 2 * cf.ras_overlap;
  size_t smem = 0;
  int threads = 0;
  ras3cl2_fn fn = pick_cl2(cf.ras_local_k, e, &smem, &threads);
  if (!fn) return cudaErrorInvalidValue;
  cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
  if (err != cudaSuccess) return err;
  int clusters = 0;
  size_t sd = 0;
  ras3d_cl2_plan(ctx, &clusters, &sd);
  Ras3Cl2Args p{};
  p.v = v; p.c = c; p.z = z; p.gscr = scratch;
  p.nx = cf.n[0]; p.ny = cf.n[1]; p.nz = cf.n[2];
  p.bx = cf.ras_box[0]; p.by = cf.ras_box[1]; p.bz = cf.ras_box[2]; p.o = cf.ras_overlap;
  p.restrict_owned = cf.ras_variant == PFC_RAS_RIGHT;
  p.y_ext = cf.ras_variant == PFC_RAS_LEFT ? nullptr : ctx->ras_y;
  p.gate = ctx->gate;
  p.jcnt = ctx->prof ? ctx->d_jcnt : nullptr;
  // class weights of v/dt - alpha Delta v - Delta^2 v - Delta^3 v / 2 with h^2 Delta = L:
  // L (000) -6, (001) 1;  L^2 (000) 42, (001) -12, (002) 1, (011) 2;
  // L^3 (000) -324, (001) 123, (002) -18, (011) -36, (003) 1, (012) 3, (111) 6
  const double ih2 = ctx->ih2, ih4 = ih2 * ih2, ih6 = ih4 * ih2;
  const double al = 0.5 * (1.0 - cf.gamma);
  p.W[0] = 1.0 / dt + 6.0 * al * ih2 - 42.0 * ih4 + 162.0 * ih6;
  p.W[1] = -al * ih2 + 12.0 * ih4 - 61.5 * ih6;
  p.W[2] = -ih4 + 9.0 * ih6;
  p.W[3] = -2.0 * ih4 + 18.0 * ih6;
  p.W[4] = -0.5 * ih6;
  p.W[5] = -1.5 * ih6;
  p.W[6] = -3.0 * ih6;
  p.ih2 = ih2;
  fn<<<2 * clusters, threads, smem, ctx->stream>>>(p);
  ctx->launches++;
  {
    const double nb = (double)(cf.n[0] / cf.ras_box[0]) * (cf.n[1] / cf.ras_box[1]) *
                      (cf.n[2] / cf.ras_box[2]);
    const double next = nb * e * e * e;
    const double nout = cf.ras_variant == PFC_RAS_LEFT ? (double)ctx->N : next;
    pfc_account(ctx, PFC_K_RAS, 8.0 * (2.0 * next + nout), 0.0);
    ras_flop_model(ctx, (double)e * e * e, 31.0, nout / nb);   // flops from the step counters
  }
  cudaError_t e2 = cudaGetLastError();
  if (e2 != cudaSuccess || cf.ras_variant == PFC_RAS_LEFT) return e2;
  return launch_ras_extend(ctx, z);
}
