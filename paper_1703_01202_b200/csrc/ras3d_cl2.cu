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
//  * the current vector v_j sits in ZL + 3 planes (the own ZL planes plus the 3 halo planes on
//    the partner's side, written by the partner through DSMEM; beyond the box the planes are
//    zero by the modified BC and are never read), padded by the 3-node zero ring in x and y
//    (row pitch 28 = 12 mod 16): a half-warp owns a 4x4 tile of columns, so every 8-byte
//    neighbour load of a half-warp hits 16 distinct bank pairs, with no bounds masks;
//  * c' = -c/h^2 on the own planes plus the one plane on the partner's side (static per box),
//    unpadded (pitch E, also conflict-free for 4x4 tiles): an xy-neighbour c' outside the box
//    is read from a finite neighbouring cell or guard row and multiplies a zero v;
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

#include <type_traits>

// diagnostic builds only (tools: PFC_EXTRA_NVCC_FLAGS=-DCL2_DIAG=n, results WRONG): bit 0 skips
// the stencil, bit 1 skips the CGS2 vector arithmetic (the reductions still run)
#ifndef CL2_DIAG
#define CL2_DIAG 0
#endif
// phase timing of CTA 0's thread 0 (diagnostic builds with -DCL2_PROF; tools/ras3_probe.py)
#ifdef CL2_PROF
// thread 0 of CTA 0 accumulates in registers-backed locals (no global traffic inside the timed
// region), flushed to cl2_prof at the end of the kernel
__device__ long long cl2_prof[16];
__device__ long long cl2_prof_last;
#define C2P(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { long long t_ = clock64(); \
    c2p_acc[i] += t_ - c2p_last; c2p_last = t_; } } while (0)
#else
#define C2P(i) do {} while (0)
#endif

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
  double idt;            // 1 / dt (host value; the graph path reads dtp[1])
  double HW[9];          // Horner-in-T form (CL2T_HORNER): z-weights of q0 (|dz| = 0..3, [0] without
                         // the 1/dt term), q1 (|dz| = 0..2), q2 (|dz| = 0..1)
  double GW[7];          // two-stage form (CL2T_HORNER = 2), U1 = [q1(Z) + T q2(Z) + a3 T^2] v: own
                         // column |dz| = 0..2, R1 columns |dz| = 0..1, R2 axis, R2 diagonal
  unsigned long long* jcnt;
  const double* dtp;     // graph path (f1): dt-dependent scalars on the device
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
// asynchronous 8-byte store into the partner CTA's shared memory that completes 8 bytes of
// transaction count on the partner's mbarrier (no cluster barrier, no memory fence)
__device__ __forceinline__ void st_async(uint32_t addr, double v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr),
               "l"(__double_as_longlong(v)), "r"(mbar)
               : "memory");
}
// wait for phase `parity` of a local mbarrier, acquiring at cluster scope (the data came from
// the partner CTA through st.async)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int E>
struct Cl2 {
  static constexpr int ZL = E / 2;                 // own z-planes per CTA
  static constexpr int PL = E * E;                 // nodes per plane (= columns)
  static constexpr int NWN = (PL + 31) / 32;      // node warps (E % 4 == 0: 4x4 column tiles)
  static constexpr int NW = NWN + 1;               // + the Givens warp
  static constexpr int NT = NW * 32;
  static constexpr int PX = E + 6 + ((12 - (E + 6)) % 16 + 16) % 16;   // >= E+6, = 12 mod 16
  static constexpr int PP = PX * (E + 6);          // padded v plane
  static constexpr int NVB = ZL + 3;   // v_j planes: own + 3 on the partner's side
  static constexpr int NCB = ZL + 1;   // c' planes: own + 1 on the partner's side
  static constexpr int CG = 2 * E;     // c' guard before and after the planes
};

template <int K, int NRX>
struct Cl2K {
  static constexpr int NR = (K - 1) < NRX ? (K - 1) : NRX;                 // registers
  static constexpr int NS = (K - 1 - NR) < 3 ? (K - 1 - NR) : 3;          // shared memory
  static constexpr int NG = K - 1 - NR - NS;                               // global scratch
};

template <int K, int E, int NRX>
constexpr size_t cl2_smem_doubles() {
  return (size_t)Cl2<E>::NVB * Cl2<E>::PP + (size_t)Cl2<E>::NCB * Cl2<E>::PL + 2 * Cl2<E>::CG +
         (size_t)Cl2K<K, NRX>::NS * Cl2<E>::ZL * Cl2<E>::PL + 2 * 2 * Cl2<E>::NW * RS +
         Cl2<E>::NW * 3 * RS;
}

// Warp partial of one inner-product value: fixed xor butterfly, lane 0 stores it into slot
// [rank][warp][i] of the reduction buffer in BOTH CTAs (local store + DSMEM store).
template <int NW>
__device__ __forceinline__ void cl2_put(double s, int i, double* redb, uint32_t redb_rem,
                                        uint32_t mbar_rem, int rank, int wid, int lane) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const int off = (rank * NW + wid) * RS + i;
    redb[off] = s;
    if (!(CL2_DIAG & 4)) st_async(redb_rem + off * 8u, s, mbar_rem);
  }
}

// Warp partials of nv values at once (acc[0..nv), nv <= 16): a sized reduce-scatter over the
// lanes (fewer shuffles than nv butterflies); the lane holding value i stores it in both CTAs.
template <int NW, int NVP>
__device__ __forceinline__ void cl2_rs_put(const double (&acc)[16], int nv, double* redb,
                                           uint32_t redb_rem, uint32_t mbar_rem, int rank,
                                           int wid, int lane) {
  constexpr int SH = 5 - (NVP == 1 ? 0 : NVP == 2 ? 1 : NVP == 4 ? 2 : NVP == 8 ? 3 : 4);
  double a[NVP];
#pragma unroll
  for (int i = 0; i < NVP; ++i) a[i] = acc[i];
  const double s = warp_reduce_scatter<NVP>(a);
  const int vi = lane >> SH;
  if ((lane & ((1 << SH) - 1)) == 0 && vi < nv) {
    const int off = (rank * NW + wid) * RS + vi;
    redb[off] = s;
    if (!(CL2_DIAG & 4)) st_async(redb_rem + off * 8u, s, mbar_rem);
  }
}
template <int NW>
__device__ __forceinline__ void cl2_put_multi(const double (&acc)[16], int nv, double* redb,
                                              uint32_t redb_rem, uint32_t mbar_rem, int rank,
                                              int wid, int lane) {
  if (nv <= 2) cl2_rs_put<NW, 2>(acc, nv, redb, redb_rem, mbar_rem, rank, wid, lane);
  else if (nv <= 4) cl2_rs_put<NW, 4>(acc, nv, redb, redb_rem, mbar_rem, rank, wid, lane);
  else if (nv <= 8) cl2_rs_put<NW, 8>(acc, nv, redb, redb_rem, mbar_rem, rank, wid, lane);
  else cl2_rs_put<NW, 16>(acc, nv, redb, redb_rem, mbar_rem, rank, wid, lane);
}

// call f(std::integral_constant<int, j>) for the runtime j in [0, K)
template <int K, int J = 0, typename F>
__device__ __forceinline__ void dispatch_j(int j, F& f) {
  if constexpr (J < K) {
    if (j == J) f(std::integral_constant<int, J>{});
    else dispatch_j<K, J + 1>(j, f);
  }
}

// Givens update of Hessenberg column j (previous rotations, then a new one) in the oracle's
// order, on shared-memory arrays (runtime indices): run by one lane of the Givens warp
__device__ __forceinline__ void givens_col(int j, const double* h1, const double* h2, double hn,
                                           double* H, double* cs, double* sn, double* gv, int ld) {
  for (int i = 0; i <= j; ++i) H[i + ld * j] = h1[i] + h2[i];
  H[j + 1 + ld * j] = hn;
  for (int i = 0; i < j; ++i) {
    const double a = H[i + ld * j], b = H[i + 1 + ld * j];
    H[i + ld * j] = cs[i] * a + sn[i] * b;
    H[i + 1 + ld * j] = -sn[i] * a + cs[i] * b;
  }
  const double a = H[j + ld * j], b = H[j + 1 + ld * j];
  const double rr = sqrt(a * a + b * b);
  double cc = 1.0, ss = 0.0;
  if (rr != 0.0) { cc = a / rr; ss = b / rr; }
  cs[j] = cc; sn[j] = ss;
  H[j + ld * j] = cc * a + ss * b;
  H[j + 1 + ld * j] = 0.0;
  gv[j + 1] = -ss * gv[j];
  gv[j] = cc * gv[j];
}

// After the cluster barrier: lanes < nv sum the 2 x NW warp partials of value `lane` in a fixed
// order (rank 0's warps, then rank 1's) into this warp's copy hwv[lane].
template <int NW>
__device__ __forceinline__ void cl2_get(int nv, const double* redb, double* hwv, int lane) {
  if (lane < nv) {   // two independent chains (rank 0's warps, rank 1's), then their sum
    double t0 = 0.0, t1 = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      t0 += redb[q * RS + lane];
      t1 += redb[(NW + q) * RS + lane];
    }
    hwv[lane] = t0 + t1;
  }
  __syncwarp();
}

// Contributions of the v_j planes zz in [LO, HI) to the thread's ZL outputs (all bounds
// compile-time: out[] stays in registers).  pv -> own column at zl = 0 of the padded v_j planes
// (the zero ring outside the extended box is the modified BC), pc -> own column at zl = 0 of
// the unpadded c' planes.
template <int E, int LO, int HI>
__device__ __forceinline__ void cl2_stencil(const Ras3Cl2Args& p, const double* pv,
                                            const double* pc, double (&out)[E / 2]) {
  constexpr int ZL = E / 2, PL = E * E, PX = Cl2<E>::PX, PP = Cl2<E>::PP;
  const double W0 = dt_w0<3>(p.dtp, p.W[0]), W1 = p.W[1], W2 = p.W[2], W3 = p.W[3], W4 = p.W[4], W5 = p.W[5],
               W6 = p.W[6];
  auto ld = [&](int dx, int dy, int zz) -> double { return pv[zz * PP + dx + PX * dy]; };
  // R = 0: own column, z-reach 3; with the z-neighbour and centre terms of -Delta(c v)
#pragma unroll
  for (int zz = (LO > -3 ? LO : -3); zz < (HI < ZL + 3 ? HI : ZL + 3); ++zz) {
    const double val = pv[zz * PP];
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
    if (zz >= 0 && zz < ZL) {   // v = 0 outside the box: the c' read there is inert
      double t = out[zz];
      t = fma(pc[zz * PL - 1], a, t);
      t = fma(pc[zz * PL + 1], b, t);
      t = fma(pc[zz * PL - E], cc, t);
      t = fma(pc[zz * PL + E], d, t);
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

template <int K, int E, int NRX>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cl2<E>::NT, 1)
    ras3d_cl2_kernel(const __grid_constant__ Ras3Cl2Args p) {
  if (p.gate && *p.gate) return;     // uniform over the cluster: both CTAs leave at once
  constexpr int ZL = Cl2<E>::ZL, PL = Cl2<E>::PL, NW = Cl2<E>::NW;
  constexpr int NVB = Cl2<E>::NVB, NCB = Cl2<E>::NCB, PX = Cl2<E>::PX, PP = Cl2<E>::PP;
  constexpr int CG = Cl2<E>::CG;
  constexpr int NR = Cl2K<K, NRX>::NR, NS = Cl2K<K, NRX>::NS, NG = Cl2K<K, NRX>::NG;
  constexpr int NE = E * E * E;
  extern __shared__ __align__(128) double smem_dyn[];
  double* vb = smem_dyn;                 // NVB padded planes: v_j (rank 0: zl in [0, ZL+3),
                                         // rank 1: [-3, ZL))
  double* cb = vb + NVB * PP + CG;       // NCB planes: c' = -c/h^2 (rank 0: [0, ZL], rank 1:
                                         // [-1, ZL)), guard rows before and after
  double* vs = cb + NCB * PL + CG;       // NS x ZL x PL: basis vectors NR..K-2
  double* red = vs + NS * ZL * PL;       // 2 buffers x [rank][warp][RS]
  double* hw = red + 2 * 2 * NW * RS;    // per warp: h1, h2, scratch
  __shared__ double H[(K + 1) * K];
  __shared__ double gv[K + 1], cs[K], sn[K], yv[K];
  // mbarriers: [0], [1] the two reduction buffers, [2] the halo planes; each completes when the
  // local thread 0 has armed it (arrive + expected bytes) and the partner's bytes have landed
  __shared__ __align__(8) uint64_t mbar[3];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool g0 = wid == NW - 1 && lane == 0;   // Givens lane: Hessenberg columns, back-subst.
  const int rank = (int)cluster_rank(), partner = rank ^ 1;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  // half-warp h owns the 4x4 column tile h of the E/4 x E/4 tiling of the xy plane
  const int tile = tid >> 4, l16 = tid & 15;
  const bool act = tile < (E / 4) * (E / 4);
  const int x = act ? 4 * (tile % (E / 4)) + (l16 & 3) : 0;
  const int y = act ? 4 * (tile / (E / 4)) + (l16 >> 2) : 0;
  const int col = y * E + x;                       // unpadded column index
  const int colp = (y + 3) * PX + (x + 3);         // padded column index
  const int pv0 = rank == 0 ? 0 : 3, pc0 = rank == 0 ? 0 : 1;   // plane of zl = 0
  const double* pv = vb + pv0 * PP + colp;         // own column, zl = 0
  const double* pc = cb + pc0 * PL + col;
  double* gs = p.gscr + (size_t)blockIdx.x * (NG > 0 ? NG : 1) * ZL * PL + tid;
  double* h1 = hw + wid * 3 * RS;
  double* h2 = h1 + RS;
  double* hx = h2 + RS;
  const uint32_t red_rem = mapa_rank(smem_u32(red), (uint32_t)partner);
  const uint32_t vb_rem = mapa_rank(smem_u32(vb), (uint32_t)partner);
  const int nbx = p.nx / p.bx, nby = p.ny / p.by, nbz = p.nz / p.bz;
  const int nboxes = nbx * nby * nbz;
  const size_t NX = p.nx, NXY = (size_t)p.nx * p.ny;

  int rb = 0;
  const uint32_t mbar_rem0 = mapa_rank(smem_u32(&mbar[0]), (uint32_t)partner);
  // zero v planes (the ring stays zero: only interior columns are ever written) and finite c'
  for (int q = tid; q < NVB * PP + NCB * PL + 2 * CG; q += blockDim.x) vb[q] = 0.0;
  if (tid == 0) {
    for (int q = 0; q < 3; ++q) mbar_init(&mbar[q], 1);
    fence_mbar_init();
  }
  cl_sync();   // the partner is running, zeroed and its mbarriers initialised before any DSMEM store
#ifdef CL2_PROF
  long long c2p_acc[16] = {0}, c2p_last = clock64();
#endif
  uint32_t ph = 0;   // phase parity bits: bit q for mbar[q]
  constexpr uint32_t HALO_BYTES = (uint32_t)PL * 3u * 8u;
  // one cluster reduction: warp partials are in both CTAs (cl2_put); arm, sync, wait, sum
  auto reduce = [&](int nsent, int nget, double* hwv) {
    if (!(CL2_DIAG & 4) && tid == 0) mbar_expect_tx(&mbar[rb], (uint32_t)(NW * nsent * 8));
    __syncthreads();
    if (!(CL2_DIAG & 4)) mbar_wait_cluster(&mbar[rb], (ph >> rb) & 1u);
    ph ^= 1u << rb;
    cl2_get<NW>(nget, red + rb * 2 * NW * RS, hwv, lane);
    rb ^= 1;
  };

  double vr[NR > 0 ? NR : 1][ZL];
#pragma unroll
  for (int s = 0; s < (NR > 0 ? NR : 1); ++s)
#pragma unroll
    for (int zl = 0; zl < ZL; ++zl) vr[s][zl] = 0.0;
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
        cb[(zl + pc0) * PL + col] = -p.ih2 * p.c[g];
        acc = fma(w[zl], w[zl], acc);
      }
      // the c' plane on the partner's side (inside the box): zl = ZL (rank 0) / -1 (rank 1)
      const int zh = rank == 0 ? ZL : -1;
      cb[(zh + pc0) * PL + col] = -p.ih2 * p.c[gxy + NXY * wrapi(gz0 + ez0 + zh, p.nz)];
    } else {
#pragma unroll
      for (int zl = 0; zl < ZL; ++zl) w[zl] = 0.0;
    }
    double* redb = red + rb * 2 * NW * RS;
    uint32_t redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
    uint32_t mbr = mbar_rem0 + 8u * rb;
    C2P(0);   // gather v, c of the box
    cl2_put<NW>(acc, 0, redb, redr, mbr, rank, wid, lane);
    reduce(1, 1, hx);
    C2P(1);   // beta reduction
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
      for (int zl = 0; zl < ZL; ++zl) vb[(zl + pv0) * PP + colp] = w[zl];
      const uint32_t hm = mbar_rem0 + 16u;   // the partner's halo mbarrier
      if (rank == 0) {   // own planes ZL-3..ZL-1 -> partner's zl' = -3..-1 (its planes 0..2)
#pragma unroll
        for (int q = 0; q < 3; ++q)
          st_async(vb_rem + (uint32_t)(q * PP + colp) * 8u, w[ZL - 3 + q], hm);
      } else {           // own planes 0..2 -> partner's zl' = ZL..ZL+2 (its planes ZL..ZL+2)
#pragma unroll
        for (int q = 0; q < 3; ++q)
          st_async(vb_rem + (uint32_t)((ZL + q) * PP + colp) * 8u, w[q], hm);
      }
    };
    // basis value i of the thread's node zl (i compile-time after unrolling)
    auto V = [&](int i, int zl) -> double {
      if (i < NR) return vr[i < NR ? i : 0][zl];
      if (i < NR + NS) return vs[((i - NR) * ZL + zl) * PL + tid];
      if (i < K - 1) return gs[((i - NR - NS) * ZL + zl) * PL];
      return pv[zl * PP];                            // v_{K-1}: only in the v_j planes
    };
    {
      const double ib = 1.0 / beta;
#pragma unroll
      for (int zl = 0; zl < ZL; ++zl) w[zl] *= ib;
      put_v(0);
    }
    if (g0) gv[0] = beta;
    int jm = 0;
    double hn_prev = 0.0;
#pragma unroll 1
    for (int j = 0; j < K; ++j) {
      // ---- w = A_k v_j: own planes while the partner's halo planes are in flight
      C2P(10);  // put_v / loop top
      if (tid == 0) mbar_expect_tx(&mbar[2], HALO_BYTES);
      __syncthreads();
      C2P(2);   // step barrier
      // the Givens lane turns column j-1 while the node warps run the stencil (its h1, h2
      // copies of step j-1 are overwritten only by this step's reductions)
      if (g0 && j > 0) givens_col(j - 1, h1, h2, hn_prev, H, cs, sn, gv, K + 1);
#pragma unroll
      for (int zl = 0; zl < ZL; ++zl) w[zl] = 0.0;
      if (act && !(CL2_DIAG & 1)) cl2_stencil<E, 0, ZL>(p, pv, pc, w);
      if (CL2_DIAG & 1) {
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) w[zl] = pv[zl * PP] * (1.0 + 0.01 * zl);
      }
      C2P(3);   // stencil, own planes
      mbar_wait_cluster(&mbar[2], (ph >> 2) & 1u);
      ph ^= 4u;
      C2P(4);   // halo wait
      if (act) {
        if (CL2_DIAG & 1) {
        } else if (rank == 0) cl2_stencil<E, ZL, ZL + 3>(p, pv, pc, w);
        else cl2_stencil<E, -3, 0>(p, pv, pc, w);
      }
      C2P(5);   // stencil, halo planes
      // ---- CGS2 on w (Arnoldi step j dispatched to code specialised for J = j: every basis
      // index compile-time, no per-node guards)
      double hn2 = 0.0;
      auto cgs2 = [&](auto Jc) {
        constexpr int J = decltype(Jc)::value;
        // pass 1: h1 = V^T w (node-outer loops: J+1 independent accumulation chains)
        redb = red + rb * 2 * NW * RS;
        redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
        mbr = mbar_rem0 + 8u * rb;
        {
          double acc[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] = 0.0;
          if (act) {   // threads without a node contribute exactly 0
#pragma unroll
            for (int zl = 0; zl < ZL; ++zl) {
              const double wz = w[zl];
#pragma unroll
              for (int i = 0; i <= J; ++i)
                acc[i] = (CL2_DIAG & 2) ? wz : fma(V(i, zl), wz, acc[i]);
            }
          }
          cl2_put_multi<NW>(acc, J + 1, redb, redr, mbr, rank, wid, lane);
        }
        reduce(J + 1, J + 1, h1);
        // pass 2: w' = w - V h1, h2 = V^T w', |w'|^2
        redb = red + rb * 2 * NW * RS;
        redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
        mbr = mbar_rem0 + 8u * rb;
        {
          double hv[J + 1], acc[16], nrm = 0.0;
#pragma unroll
          for (int i = 0; i <= J; ++i) hv[i] = h1[i];
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] = 0.0;
          if (act) {
#pragma unroll
            for (int zl = 0; zl < ZL; ++zl) {
              double ww = w[zl];
#pragma unroll
              for (int i = 0; i <= J; ++i)
                ww = (CL2_DIAG & 2) ? ww : fma(-hv[i], V(i, zl), ww);
#pragma unroll
              for (int i = 0; i <= J; ++i)
                acc[i] = (CL2_DIAG & 2) ? ww : fma(V(i, zl), ww, acc[i]);
              nrm = fma(ww, ww, nrm);
              w[zl] = ww;
            }
          }
          cl2_put_multi<NW>(acc, J + 1, redb, redr, mbr, rank, wid, lane);
          cl2_put<NW>(nrm, J + 1, redb, redr, mbr, rank, wid, lane);   // |w'|^2 in slot j+1
        }
        reduce(J + 2, J + 2, h2);
        double h2n = 0.0;
        for (int i = 0; i <= J; ++i) h2n += h2[i] * h2[i];
        const double wn2 = h2[J + 1];
        // pass 3: w'' = w' - V h2
        if (act) {
          double hv[J + 1];
#pragma unroll
          for (int i = 0; i <= J; ++i) hv[i] = h2[i];
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) {
            double ww = w[zl];
#pragma unroll
            for (int i = 0; i <= J; ++i)
              ww = (CL2_DIAG & 2) ? ww : fma(-hv[i], V(i, zl), ww);
            w[zl] = ww;
          }
        }
        if (h2n <= 1e-8 * wn2) {
          hn2 = wn2 - h2n;                             // |w''|^2 = |w'|^2 - |h2|^2
        } else {
          redb = red + rb * 2 * NW * RS;
          redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
          mbr = mbar_rem0 + 8u * rb;
          double s = 0.0;
          if (act) {
#pragma unroll
            for (int zl = 0; zl < ZL; ++zl) s = fma(w[zl], w[zl], s);
          }
          cl2_put<NW>(s, 0, redb, redr, mbr, rank, wid, lane);
          reduce(1, 1, hx);
          hn2 = hx[0];
        }
        return hn2;
      };
      dispatch_j<K>(j, cgs2);
      C2P(6);   // CGS2 (three passes, two or three reductions)
      const double hn = CL2_DIAG ? 1.0 : sqrt(hn2 > 0.0 ? hn2 : 0.0);
      hn_prev = hn;
      jm = j + 1;
      if (hn <= 1e-14 * beta) break;                 // exact breakdown (identical on both CTAs)
      if (j + 1 < K) {
        const double ihn = 1.0 / hn;
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) w[zl] *= ihn;
        put_v(j + 1);
      }
    }
    C2P(10);
    if (g0) {   // last Hessenberg column, then back substitution R yv = g
      const int ld = K + 1;
      givens_col(jm - 1, h1, h2, hn_prev, H, cs, sn, gv, ld);
      for (int i = jm - 1; i >= 0; --i) {
        double s = gv[i];
        for (int l = i + 1; l < jm; ++l) s -= H[i + ld * l] * yv[l];
        yv[i] = s / H[i + ld * i];
      }
      if (rank == 0) ras_count(p.jcnt, jm);
    }
    __syncthreads();
    C2P(7);   // Givens / back substitution (waiting for the Givens warp)
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
    C2P(9);   // final V y and the output stores
  }
  C2P(8);
#ifdef CL2_PROF
  if (blockIdx.x == 0 && tid == 0)
    for (int i = 0; i < 16; ++i) cl2_prof[i] += c2p_acc[i];
#endif
  cl_sync();   // no CTA leaves while its partner may still address its shared memory
}

// ============================================================================================
// Two columns per thread (CP = 2): thread t < E^2/2 owns the z-columns (x, y0) and (x, y0+1),
// x = t % E, y0 = 2 (t / E), of its CTA's z-half.  The 63-point stencils of the two columns
// read the union of their radius-3 diamonds, 32 neighbour columns instead of 2 x 25, so the
// shared-memory traffic of the stencil (the bound of the one-column kernel: ~90% of the
// shared-memory bandwidth while the stencil runs) falls by ~35%; 7 node warps + the Givens
// warp, up to 255 registers per thread, which holds NR basis vectors of both columns.
// Layouts (linear thread order, conflict-free because a half-warp spans at most two row pairs
// and 2 PX = E (mod 16)): v_j planes padded to PX x (E+6), c' planes padded to CX x (E+2).
template <int E>
struct Cl2p {
  static constexpr int ZL = E / 2, PL = E * E;
  static constexpr int NTN = PL / 2;                 // node threads
  static constexpr int NWN = (NTN + 31) / 32;        // node warps
  static constexpr int NW = NWN + 1;                 // + the Givens warp
  static constexpr int NT = NW * 32;
  // smallest pitch >= w with 2 pitch = E (mod 16)
  static constexpr int pitch(int w) {
    int q = w;
    while (((2 * q - E) % 16 + 16) % 16 != 0) ++q;
    return q;
  }
  static constexpr int PX = pitch(E + 6), PP = PX * (E + 6);   // v_j plane
  static constexpr int CX = pitch(E + 2), CP = CX * (E + 2);   // c' plane
  static constexpr int NVB = ZL + 3, NCB = ZL + 1;
};

template <int K, int NRX>
struct Cl2pK {
  static constexpr int NR = (K - 1) < NRX ? (K - 1) : NRX;
  static constexpr int NS = (K - 1 - NR) < 3 ? (K - 1 - NR) : 3;
  static constexpr int NG = K - 1 - NR - NS;
};

template <int K, int E, int NRX>
constexpr size_t cl2p_smem_doubles() {
  using C = Cl2p<E>;
  return (size_t)C::NVB * C::PP + (size_t)C::NCB * C::CP +
         (size_t)Cl2pK<K, NRX>::NS * 2 * C::ZL * C::NTN + 2 * 2 * C::NW * RS + C::NW * 3 * RS;
}

// group of union column (dx, du) for output o (dy = du - o): 0 own, 1 R1, 2 R2 axis,
// 3 R2 diagonal, 4 R3 axis, 5 R3 off-axis, -1 none
__host__ __device__ constexpr int cl2p_group(int o, int dx, int du) {
  const int dy = du - o;
  const int ax = dx < 0 ? -dx : dx, ay = dy < 0 ? -dy : dy, r = ax + ay;
  return r == 0 ? 0 : r == 1 ? 1 : r == 2 ? ((ax == 0 || ay == 0) ? 2 : 3)
         : r == 3 ? ((ax == 0 || ay == 0) ? 4 : 5) : -1;
}
__host__ __device__ constexpr int cl2p_reach(int g) {
  return g == 0 ? 3 : g == 1 ? 2 : (g == 2 || g == 3) ? 1 : 0;
}

template <int E, int LO, int HI>
__device__ __forceinline__ void cl2p_stencil(const Ras3Cl2Args& p, const double* pv,
                                             const double* pc, double (&out)[2][E / 2]) {
  using C = Cl2p<E>;
  constexpr int ZL = C::ZL, PX = C::PX, PP = C::PP, CX = C::CX, CP = C::CP;
  const double W0 = dt_w0<3>(p.dtp, p.W[0]), W1 = p.W[1], W2 = p.W[2], W3 = p.W[3], W4 = p.W[4], W5 = p.W[5],
               W6 = p.W[6];
#pragma unroll
  for (int zz = (LO > -3 ? LO : -3); zz < (HI < ZL + 3 ? HI : ZL + 3); ++zz) {
    double g[2][6], cvn[2], cvo[2];
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      cvn[o] = 0.0;
      cvo[o] = 0.0;
#pragma unroll
      for (int k = 0; k < 6; ++k) g[o][k] = 0.0;
    }
#pragma unroll
    for (int dx = -3; dx <= 3; ++dx) {
#pragma unroll
      for (int du = -3; du <= 4; ++du) {
        bool need = false;
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          const int k = cl2p_group(o, dx, du);
          if (k >= 0 && zz >= -cl2p_reach(k) && zz < ZL + cl2p_reach(k)) need = true;
        }
        if (!need) continue;
        const double val = pv[zz * PP + dx + PX * du];
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          const int k = cl2p_group(o, dx, du);
          if (k < 0 || zz < -cl2p_reach(k) || zz >= ZL + cl2p_reach(k)) continue;
          g[o][k] += val;
          // -Delta(c v): the xy neighbours at dz = 0 and the own column (c' = -c/h^2; v = 0
          // outside the box, so the finite c' read there is inert)
          if (k == 1 && zz >= 0 && zz < ZL) cvn[o] = fma(pc[zz * CP + dx + CX * du], val, cvn[o]);
          if (k == 0 && zz >= -1 && zz <= ZL) cvo[o] = pc[zz * CP + CX * o] * val;
        }
      }
    }
#pragma unroll
    for (int o = 0; o < 2; ++o) {
#pragma unroll
      for (int z = (zz - 3 > 0 ? zz - 3 : 0); z <= (zz + 3 < ZL - 1 ? zz + 3 : ZL - 1); ++z) {
        const int dz = zz > z ? zz - z : z - zz;
        out[o][z] = fma(dz == 0 ? W0 : dz == 1 ? W1 : dz == 2 ? W2 : W4, g[o][0], out[o][z]);
        if (dz <= 2) out[o][z] = fma(dz == 0 ? W1 : dz == 1 ? W3 : W5, g[o][1], out[o][z]);
        if (dz <= 1) {
          out[o][z] = fma(dz == 0 ? W2 : W5, g[o][2], out[o][z]);
          out[o][z] = fma(dz == 0 ? W3 : W6, g[o][3], out[o][z]);
        }
        if (dz == 0) {
          out[o][z] = fma(W4, g[o][4], out[o][z]);
          out[o][z] = fma(W5, g[o][5], out[o][z]);
        }
      }
      if (zz >= 0 && zz < ZL) out[o][zz] += cvn[o];
      if (zz >= -1 && zz <= ZL) {
        if (zz - 1 >= 0 && zz - 1 < ZL) out[o][zz - 1] += cvo[o];
        if (zz + 1 >= 0 && zz + 1 < ZL) out[o][zz + 1] += cvo[o];
        if (zz >= 0 && zz < ZL) out[o][zz] = fma(-6.0, cvo[o], out[o][zz]);
      }
    }
  }
}

template <int K, int E, int NRX>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cl2p<E>::NT, 1)
    ras3d_cl2p_kernel(const __grid_constant__ Ras3Cl2Args p) {
  if (p.gate && *p.gate) return;     // uniform over the cluster: both CTAs leave at once
  using C = Cl2p<E>;
  constexpr int ZL = C::ZL, PL = C::PL, NW = C::NW, NTN = C::NTN;
  constexpr int PX = C::PX, PP = C::PP, CX = C::CX, CP = C::CP, NVB = C::NVB, NCB = C::NCB;
  constexpr int NR = Cl2pK<K, NRX>::NR, NS = Cl2pK<K, NRX>::NS, NG = Cl2pK<K, NRX>::NG;
  constexpr int NE = E * E * E;
  extern __shared__ __align__(128) double smem_dyn[];
  double* vb = smem_dyn;                 // NVB padded planes of v_j (rank 0: zl in [0, ZL+3),
                                         // rank 1: [-3, ZL))
  double* cb = vb + NVB * PP;            // NCB padded planes of c' (rank 0: [0, ZL], rank 1:
                                         // [-1, ZL))
  double* vs = cb + NCB * CP;            // NS x [col][zl][thread]: basis vectors NR..NR+NS-1
  double* red = vs + NS * 2 * ZL * NTN;  // 2 buffers x [rank][warp][RS]
  double* hw = red + 2 * 2 * NW * RS;    // per warp: h1, h2, scratch
  __shared__ double H[(K + 1) * K];
  __shared__ double gv[K + 1], cs[K], sn[K], yv[K];
  __shared__ __align__(8) uint64_t mbar[3];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool g0 = wid == NW - 1 && lane == 0;
  const int rank = (int)cluster_rank(), partner = rank ^ 1;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const bool act = tid < NTN;
  const int x = act ? tid % E : 0, y0 = act ? 2 * (tid / E) : 0;
  const int colp = (y0 + 3) * PX + (x + 3);        // padded v column of (x, y0)
  const int colc = (y0 + 1) * CX + (x + 1);        // padded c' column of (x, y0)
  const int pv0 = rank == 0 ? 0 : 3, pc0 = rank == 0 ? 0 : 1;   // plane of zl = 0
  const double* pv = vb + pv0 * PP + colp;
  const double* pc = cb + pc0 * CP + colc;
  double* gs = p.gscr + (size_t)blockIdx.x * (NG > 0 ? NG : 1) * 2 * ZL * NTN + tid;
  double* h1 = hw + wid * 3 * RS;
  double* h2 = h1 + RS;
  double* hx = h2 + RS;
  const uint32_t red_rem = mapa_rank(smem_u32(red), (uint32_t)partner);
  const uint32_t vb_rem = mapa_rank(smem_u32(vb), (uint32_t)partner);
  const int nbx = p.nx / p.bx, nby = p.ny / p.by, nbz = p.nz / p.bz;
  const int nboxes = nbx * nby * nbz;
  const size_t NX = p.nx, NXY = (size_t)p.nx * p.ny;

  int rb = 0;
  const uint32_t mbar_rem0 = mapa_rank(smem_u32(&mbar[0]), (uint32_t)partner);
  // zero v planes (ring stays zero), finite c' and finite basis slots (the final V y reads
  // every slot with a zero coefficient beyond the steps taken; the L2 scratch is zeroed at
  // context creation)
  for (int q = tid; q < NVB * PP + NCB * CP + NS * 2 * ZL * NTN; q += blockDim.x) vb[q] = 0.0;
  if (tid == 0) {
    for (int q = 0; q < 3; ++q) mbar_init(&mbar[q], 1);
    fence_mbar_init();
  }
  cl_sync();   // the partner is running, zeroed and its mbarriers initialised before any DSMEM store
#ifdef CL2_PROF
  long long c2p_acc[16] = {0}, c2p_last = clock64();
#endif
  uint32_t ph = 0;
  constexpr uint32_t HALO_BYTES = (uint32_t)PL * 3u * 8u;
  auto reduce = [&](int nsent, int nget, double* hwv) {
    if (tid == 0) mbar_expect_tx(&mbar[rb], (uint32_t)(NW * nsent * 8));
    __syncthreads();
    mbar_wait_cluster(&mbar[rb], (ph >> rb) & 1u);
    ph ^= 1u << rb;
    cl2_get<NW>(nget, red + rb * 2 * NW * RS, hwv, lane);
    rb ^= 1;
  };

  double vr[NR > 0 ? NR : 1][2][ZL];
#pragma unroll
  for (int s = 0; s < (NR > 0 ? NR : 1); ++s)
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int zl = 0; zl < ZL; ++zl) vr[s][c][zl] = 0.0;
  for (int box = cid; box < nboxes; box += ncl) {
    const int ibx = box % nbx, iby = (box / nbx) % nby, ibz = box / (nbx * nby);
    const int gx0 = ibx * p.bx - p.o, gy0 = iby * p.by - p.o, gz0 = ibz * p.bz - p.o;
    const int ez0 = rank * ZL;
    double w[2][ZL];
    double acc = 0.0;
    if (act) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int y = y0 + c;
        const size_t gxy = (size_t)wrapi(gx0 + x, p.nx) + NX * wrapi(gy0 + y, p.ny);
        const bool oxy = x >= p.o && x < p.o + p.bx && y >= p.o && y < p.o + p.by;
        int gz = wrapi(gz0 + ez0, p.nz);   // wrapped z of own plane 0, advanced without '%'
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl, gz = gz + 1 == p.nz ? 0 : gz + 1) {
          const size_t g = gxy + NXY * (size_t)gz;
          const int ez = ez0 + zl;
          const bool owned = oxy && ez >= p.o && ez < p.o + p.bz;
          w[c][zl] = (p.restrict_owned && !owned) ? 0.0 : p.v[g];
          cb[(zl + pc0) * CP + colc + c * CX] = -p.ih2 * p.c[g];
          acc = fma(w[c][zl], w[c][zl], acc);
        }
        const int zh = rank == 0 ? ZL : -1;
        cb[(zh + pc0) * CP + colc + c * CX] =
            -p.ih2 * p.c[gxy + NXY * wrapi(gz0 + ez0 + zh, p.nz)];
      }
    } else {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) w[c][zl] = 0.0;
    }
    double* redb = red + rb * 2 * NW * RS;
    uint32_t redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
    uint32_t mbr = mbar_rem0 + 8u * rb;
    C2P(0);
    cl2_put<NW>(acc, 0, redb, redr, mbr, rank, wid, lane);
    reduce(1, 1, hx);
    C2P(1);
    const double beta = sqrt(hx[0]);
    if (beta == 0.0) {
      if (act) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) {
            const int y = y0 + c;
            const int ez = ez0 + zl, li = x - p.o, lj = y - p.o, lk = ez - p.o;
            if (p.y_ext) p.y_ext[(size_t)box * NE + (ez * E + y) * E + x] = 0.0;
            else if (li >= 0 && li < p.bx && lj >= 0 && lj < p.by && lk >= 0 && lk < p.bz)
              p.z[(size_t)(ibx * p.bx + li) + NX * (iby * p.by + lj) + NXY * (ibz * p.bz + lk)] = 0.0;
          }
      }
      if (tid == 0 && rank == 0) ras_count(p.jcnt, 0);
      continue;
    }
    auto put_v = [&](int slot) {
      if (!act) return;
#pragma unroll
      for (int s = 0; s < NR; ++s)
        if (s == slot) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int zl = 0; zl < ZL; ++zl) vr[s][c][zl] = w[c][zl];
        }
      if (slot >= NR && slot < NR + NS) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl)
            vs[(((slot - NR) * 2 + c) * ZL + zl) * NTN + tid] = w[c][zl];
      } else if (slot >= NR + NS && slot < K - 1) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl)
            gs[(((slot - NR - NS) * 2 + c) * ZL + zl) * NTN] = w[c][zl];
      }
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) vb[(zl + pv0) * PP + colp + c * PX] = w[c][zl];
      const uint32_t hm = mbar_rem0 + 16u;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (rank == 0) {
#pragma unroll
          for (int q = 0; q < 3; ++q)
            st_async(vb_rem + (uint32_t)(q * PP + colp + c * PX) * 8u, w[c][ZL - 3 + q], hm);
        } else {
#pragma unroll
          for (int q = 0; q < 3; ++q)
            st_async(vb_rem + (uint32_t)((ZL + q) * PP + colp + c * PX) * 8u, w[c][q], hm);
        }
      }
    };
    auto V = [&](int i, int c, int zl) -> double {
      if (i < NR) return vr[i < NR ? i : 0][c][zl];
      if (i < NR + NS) return vs[(((i - NR) * 2 + c) * ZL + zl) * NTN + tid];
      if (i < K - 1) return gs[(((i - NR - NS) * 2 + c) * ZL + zl) * NTN];
      return pv[zl * PP + c * PX];
    };
    {
      const double ib = 1.0 / beta;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) w[c][zl] *= ib;
      put_v(0);
    }
    if (g0) gv[0] = beta;
    int jm = 0;
    double hn_prev = 0.0;
#pragma unroll 1
    for (int j = 0; j < K; ++j) {
      C2P(10);
      if (tid == 0) mbar_expect_tx(&mbar[2], HALO_BYTES);
      __syncthreads();
      C2P(2);
      if (g0 && j > 0) givens_col(j - 1, h1, h2, hn_prev, H, cs, sn, gv, K + 1);
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) w[c][zl] = 0.0;
      if (act) cl2p_stencil<E, 0, ZL>(p, pv, pc, w);
      C2P(3);
      mbar_wait_cluster(&mbar[2], (ph >> 2) & 1u);
      ph ^= 4u;
      C2P(4);
      if (act) {
        if (rank == 0) cl2p_stencil<E, ZL, ZL + 3>(p, pv, pc, w);
        else cl2p_stencil<E, -3, 0>(p, pv, pc, w);
      }
      C2P(5);
      double hn2 = 0.0;
      auto cgs2 = [&](auto Jc) {
        constexpr int J = decltype(Jc)::value;
        redb = red + rb * 2 * NW * RS;
        redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
        mbr = mbar_rem0 + 8u * rb;
        {
          double acc[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] = 0.0;
          if (act) {
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int zl = 0; zl < ZL; ++zl) {
                const double wz = w[c][zl];
#pragma unroll
                for (int i = 0; i <= J; ++i) acc[i] = fma(V(i, c, zl), wz, acc[i]);
              }
          }
          C2P(11);
          cl2_put_multi<NW>(acc, J + 1, redb, redr, mbr, rank, wid, lane);
        }
        reduce(J + 1, J + 1, h1);
        C2P(12);
        redb = red + rb * 2 * NW * RS;
        redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
        mbr = mbar_rem0 + 8u * rb;
        {
          double hv[J + 1], acc[16], nrm = 0.0;
#pragma unroll
          for (int i = 0; i <= J; ++i) hv[i] = h1[i];
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] = 0.0;
          if (act) {
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int zl = 0; zl < ZL; ++zl) {
                double ww = w[c][zl];
#pragma unroll
                for (int i = 0; i <= J; ++i) ww = fma(-hv[i], V(i, c, zl), ww);
#pragma unroll
                for (int i = 0; i <= J; ++i) acc[i] = fma(V(i, c, zl), ww, acc[i]);
                nrm = fma(ww, ww, nrm);
                w[c][zl] = ww;
              }
          }
          C2P(13);
          cl2_put_multi<NW>(acc, J + 1, redb, redr, mbr, rank, wid, lane);
          cl2_put<NW>(nrm, J + 1, redb, redr, mbr, rank, wid, lane);
        }
        reduce(J + 2, J + 2, h2);
        C2P(14);
        double h2n = 0.0;
        for (int i = 0; i <= J; ++i) h2n += h2[i] * h2[i];
        const double wn2 = h2[J + 1];
        if (act) {
          double hv[J + 1];
#pragma unroll
          for (int i = 0; i <= J; ++i) hv[i] = h2[i];
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int zl = 0; zl < ZL; ++zl) {
              double ww = w[c][zl];
#pragma unroll
              for (int i = 0; i <= J; ++i) ww = fma(-hv[i], V(i, c, zl), ww);
              w[c][zl] = ww;
            }
        }
        if (h2n <= 1e-8 * wn2) {
          hn2 = wn2 - h2n;
        } else {
          redb = red + rb * 2 * NW * RS;
          redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
          mbr = mbar_rem0 + 8u * rb;
          double s = 0.0;
          if (act) {
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int zl = 0; zl < ZL; ++zl) s = fma(w[c][zl], w[c][zl], s);
          }
          cl2_put<NW>(s, 0, redb, redr, mbr, rank, wid, lane);
          reduce(1, 1, hx);
          hn2 = hx[0];
        }
        return hn2;
      };
      dispatch_j<K>(j, cgs2);
      C2P(6);
      const double hn = sqrt(hn2 > 0.0 ? hn2 : 0.0);
      hn_prev = hn;
      jm = j + 1;
      if (hn <= 1e-14 * beta) break;
      if (j + 1 < K) {
        const double ihn = 1.0 / hn;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) w[c][zl] *= ihn;
        put_v(j + 1);
      }
    }
    C2P(10);
    if (g0) {
      const int ld = K + 1;
      givens_col(jm - 1, h1, h2, hn_prev, H, cs, sn, gv, ld);
      for (int i = jm - 1; i >= 0; --i) {
        double s = gv[i];
        for (int l = i + 1; l < jm; ++l) s -= H[i + ld * l] * yv[l];
        yv[i] = s / H[i + ld * i];
      }
      for (int i = jm; i < K; ++i) yv[i] = 0.0;   // steps not taken: zero coefficients
      if (rank == 0) ras_count(p.jcnt, jm);
    }
    __syncthreads();
    C2P(7);
    if (act) {
      // y = V yv with no data-dependent branch, so every basis load (three vectors from the L2
      // scratch) is issued up front; fma(0, v, s) = s exactly for the finite unused slots
      double yl[2][ZL];
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) yl[c][zl] = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const double yi = yv[i];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) yl[c][zl] = fma(yi, V(i, c, zl), yl[c][zl]);
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int y = y0 + c;
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) {
          const int ez = ez0 + zl, li = x - p.o, lj = y - p.o, lk = ez - p.o;
          if (p.y_ext) {
            p.y_ext[(size_t)box * NE + (ez * E + y) * E + x] = yl[c][zl];
          } else if (li >= 0 && li < p.bx && lj >= 0 && lj < p.by && lk >= 0 && lk < p.bz) {
            p.z[(size_t)(ibx * p.bx + li) + NX * (iby * p.by + lj) + NXY * (ibz * p.bz + lk)] =
                yl[c][zl];
          }
        }
      }
    }
    C2P(9);
  }
  C2P(8);
#ifdef CL2_PROF
  if (blockIdx.x == 0 && tid == 0)
    for (int i = 0; i < 16; ++i) cl2_prof[i] += c2p_acc[i];
#endif
  cl_sync();   // no CTA leaves while its partner may still address its shared memory
}


// ---- tensor memory as basis storage (ras3d_cl2t_kernel): tcgen05.st / tcgen05.ld of the
// 32x32b shape move each thread's own TMEM lane row (32-bit columns); a double is two columns.
// Measured on this pool (tools/tmem_probe.cu, 8 warps): tcgen05.ld 427 B/clk/SM with a wait
// after every x16, tcgen05.st 977 B/clk/SM -- 3x and 7x the 128 B/clk of shared memory.
__device__ __forceinline__ void tm_alloc512(uint32_t* dst) {   // one warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                   smem_u32(dst))
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_dealloc512(uint32_t base) {   // the allocating warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tm_st16(uint32_t ta, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(ta),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tm_st8(uint32_t ta, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
               "r"(r[7])
               : "memory");
}
// load + wait in one statement: the registers are valid when the statement ends
__device__ __forceinline__ void tm_ld16(uint32_t ta, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n\ttcgen05.wait::ld.sync.aligned;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(ta)
      : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t ta, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(ta)
      : "memory");
}
// a thread's 2 x ZL doubles <-> 4 ZL columns at ta (chunks of 16 columns, then 8)
template <int ZL>
__device__ __forceinline__ void tm_st_vec(uint32_t ta, const double (&w)[2][ZL]) {
  constexpr int NC = 4 * ZL;
  static_assert(NC % 8 == 0, "columns in chunks of 8");
  uint32_t r[NC];
#pragma unroll
  for (int k = 0; k < 2 * ZL; ++k) {
    const double d = w[k / ZL][k % ZL];
    r[2 * k] = (uint32_t)__double2loint(d);
    r[2 * k + 1] = (uint32_t)__double2hiint(d);
  }
#pragma unroll
  for (int c = 0; c + 16 <= NC; c += 16) tm_st16(ta + c, r + c);
  if constexpr (NC % 16 == 8) tm_st8(ta + (NC - 8), r + (NC - 8));
  // (no wait here: the sources are consumed at issue; tm_wait_st() before the data is read back)
}
__device__ __forceinline__ void tm_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// 40 columns (ZL = 10) in one statement: three loads, one wait (one TMEM round trip)
__device__ __forceinline__ void tm_ld40(uint32_t ta, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%40];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,"
      "%28,%29,%30,%31}, [%41];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%32,%33,%34,%35,%36,%37,%38,%39}, [%42];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]),
        "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]),
        "=r"(v[38]), "=r"(v[39])
      : "r"(ta), "r"(ta + 16), "r"(ta + 32)
      : "memory");
}
template <int ZL>
__device__ __forceinline__ void tm_ld_vec(uint32_t ta, double (&v)[2][ZL]) {
  constexpr int NC = 4 * ZL;
  uint32_t r[NC];
  if constexpr (NC == 40) {
    tm_ld40(ta, r);
  } else {
#pragma unroll
    for (int c = 0; c + 16 <= NC; c += 16) tm_ld16(ta + c, r + c);
    if constexpr (NC % 16 == 8) tm_ld8(ta + (NC - 8), r + (NC - 8));
  }
#pragma unroll
  for (int k = 0; k < 2 * ZL; ++k)
    v[k / ZL][k % ZL] = __hiloint2double((int)r[2 * k + 1], (int)r[2 * k]);
}

// Cl2p with the basis vectors NR..K-2 in tensor memory instead of shared memory (NS) and the
// L2 scratch (NG): the whole Krylov basis on chip.  Same layouts and arithmetic as
// ras3d_cl2p_kernel, the CGS2 passes vector by vector with each inner product summed in four
// independent chains (FP64 latency with 8 warps), so it agrees with cl2p to rounding.
// ---- Horner-in-T form of the subdomain operator (CL2T_HORNER = 1) ---------------------------
// With the unscaled Laplacian split as L = T + Z (T: 5-point xy part, Z: 3-point z part; they
// commute) and A_k v = p(L) v + L (c' v), p(L) = a0 + a1 L + a2 L^2 + a3 L^3 (a0 = 1/dt,
// a1 = -(1-gamma)/2 h^-2, a2 = -h^-4, a3 = -h^-6 / 2, c' = -c / h^2):
//   U2 = q2(Z) v + a3 T v,   U1 = q1(Z) v + c' v + T U2,   A_k v = q0(Z) v + Z (c' v) + T U1,
//   q0 = a0 + a1 Z + a2 Z^2 + a3 Z^3,  q1 = a1 + 2 a2 Z + 3 a3 Z^2,  q2 = a2 + 3 a3 Z.
// Every q_m(Z) acts along the thread's own z-columns (their z-halo comes from the partner's
// planes), each T stage reads the 6 outside xy neighbour columns of the thread's column pair
// over the OWN z-range from a plane set the previous stage wrote (U2, then U1; c'-plane layout),
// with a CTA barrier between stages.  v = 0 outside the box leaves U2 and U1 non-zero only on
// the 4 E ring columns next to a box face (corners stay zero): the Givens warp computes those.
#ifndef CL2T_HORNER
#define CL2T_HORNER 0
#endif

// PART 0: the contributions of the CTA's own planes (before the partner's halo planes have
// landed); PART 1: those of the halo planes.  U2 goes to its plane set as soon as an entry is
// complete; U1 (without T U2) and w stay in registers.
template <int E, int PART>
__device__ __forceinline__ void hz_stage1(const Ras3Cl2Args& p, double q00, const double* pv,
                                          const double* pc, double* pu, int rank,
                                          double (&w)[2][E / 2], double (&u1)[2][E / 2],
                                          double (&u2)[2][E / 2]) {
  using C = Cl2p<E>;
  constexpr int ZL = C::ZL, PX = C::PX, PP = C::PP, CX = C::CX, CP = C::CP;
#pragma unroll
  for (int zz = -3; zz < ZL + 3; ++zz) {
    const bool own = zz >= 0 && zz < ZL;
    if ((PART == 0) != own) continue;
    // planes this CTA holds: rank 0 [0, ZL+3), rank 1 [-3, ZL); beyond the box face v = 0
    const bool live = (zz >= 0 || rank != 0) && (zz < ZL || rank != 1);
    if (live) {
      const double val[2] = {pv[zz * PP], pv[zz * PP + PX]};
#pragma unroll
      for (int c = 0; c < 2; ++c) {
#pragma unroll
        for (int z = (zz - 3 > 0 ? zz - 3 : 0); z <= (zz + 3 < ZL - 1 ? zz + 3 : ZL - 1); ++z) {
          const int dz = zz > z ? zz - z : z - zz;
          w[c][z] = fma(dz == 0 ? q00 : dz == 1 ? p.HW[1] : dz == 2 ? p.HW[2] : p.HW[3], val[c],
                        w[c][z]);
          if (dz <= 2)
            u1[c][z] = fma(dz == 0 ? p.HW[4] : dz == 1 ? p.HW[5] : p.HW[6], val[c], u1[c][z]);
          if (dz <= 1) u2[c][z] = fma(dz == 0 ? p.HW[7] : p.HW[8], val[c], u2[c][z]);
        }
      }
      if (own) {   // a3 T v over the own z-range
        const double n0 = pv[zz * PP - 1], n1 = pv[zz * PP + 1], n2 = pv[zz * PP - PX];
        const double n3 = pv[zz * PP + 2 * PX], n4 = pv[zz * PP + PX - 1],
                     n5 = pv[zz * PP + PX + 1];
        const double t0 = fma(-4.0, val[0], (n0 + n1) + (n2 + val[1]));
        const double t1 = fma(-4.0, val[1], (n4 + n5) + (n3 + val[0]));
        u2[0][zz] = fma(p.HW[3], t0, u2[0][zz]);
        u2[1][zz] = fma(p.HW[3], t1, u2[1][zz]);
      }
      if (zz >= -1 && zz <= ZL) {   // c' v: into U1 at its plane, Z (c' v) into w
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const double cv = pc[zz * CP + c * CX] * val[c];
          if (zz - 1 >= 0 && zz - 1 < ZL) w[c][zz - 1] += cv;
          if (zz + 1 >= 0 && zz + 1 < ZL) w[c][zz + 1] += cv;
          if (own) {
            w[c][zz] = fma(-2.0, cv, w[c][zz]);
            u1[c][zz] += cv;
          }
        }
      }
    }
    // U2 entries that only own planes contribute to, as soon as they are complete
    if (PART == 0 && zz - 1 >= 1 && zz - 1 <= ZL - 2) {
      pu[(zz - 1) * CP] = u2[0][zz - 1];
      pu[(zz - 1) * CP + CX] = u2[1][zz - 1];
    }
  }
  if (PART == 1) {
    pu[0] = u2[0][0];
    pu[CX] = u2[1][0];
    pu[(ZL - 1) * CP] = u2[0][ZL - 1];
    pu[(ZL - 1) * CP + CX] = u2[1][ZL - 1];
  }
}

// U1 += T U2 at the thread's nodes (registers), written to its plane set for the neighbours
template <int E>
__device__ __forceinline__ void hz_stage2(const double* pu, double* pq, double (&u1)[2][E / 2]) {
  using C = Cl2p<E>;
  constexpr int ZL = C::ZL, CX = C::CX, CP = C::CP;
#pragma unroll
  for (int zl = 0; zl < ZL; ++zl) {
    const double* u = pu + zl * CP;
    const double o0 = u[0], o1 = u[CX];
    u1[0][zl] += fma(-4.0, o0, (u[-1] + u[1]) + (u[-CX] + o1));
    u1[1][zl] += fma(-4.0, o1, (u[CX - 1] + u[CX + 1]) + (u[2 * CX] + o0));
    pq[zl * CP] = u1[0][zl];
    pq[zl * CP + CX] = u1[1][zl];
  }
}

// w += T U1 at the thread's nodes
template <int E>
__device__ __forceinline__ void hz_stage3(const double* pq, const double (&u1)[2][E / 2],
                                          double (&w)[2][E / 2]) {
  using C = Cl2p<E>;
  constexpr int ZL = C::ZL, CX = C::CX, CP = C::CP;
#pragma unroll
  for (int zl = 0; zl < ZL; ++zl) {
    const double* u = pq + zl * CP;
    const double o0 = u1[0][zl], o1 = u1[1][zl];
    w[0][zl] += fma(-4.0, o0, (u[-1] + u[1]) + (u[-CX] + o1));
    w[1][zl] += fma(-4.0, o1, (u[CX - 1] + u[CX + 1]) + (u[2 * CX] + o0));
  }
}

// ---- two-stage form (CL2T_HORNER = 2): U1 = [q1(Z) + T q2(Z) + a3 T^2] v + c' v evaluated directly
// (radius-2 xy diamond, union of the two columns' diamonds, z-reach 2 / 1 / 0 for the own / R1 /
// R2 columns) together with the own-column part q0(Z) v + Z (c' v) of w; then w += T U1.
template <int E, int ZZ>
__device__ __forceinline__ void hy_plane(const Ras3Cl2Args& p, double q00, const double* pv,
                                         const double* pc, int rank, double (&w)[2][E / 2],
                                         double (&u1)[2][E / 2]) {
  using C = Cl2p<E>;
  constexpr int ZL = C::ZL, PX = C::PX, PP = C::PP, CX = C::CX, CP = C::CP;
  constexpr int zz = ZZ;
  {
    constexpr bool own = zz >= 0 && zz < ZL;
    // planes this CTA holds: rank 0 [0, ZL+3), rank 1 [-3, ZL); beyond the box face v = 0
    const bool live = (zz >= 0 || rank != 0) && (zz < ZL || rank != 1);
    if (live) {
    double g[2][4];
#pragma unroll
    for (int o = 0; o < 2; ++o)
#pragma unroll
      for (int k = 0; k < 4; ++k) g[o][k] = 0.0;
#pragma unroll
    for (int dx = -2; dx <= 2; ++dx) {
#pragma unroll
      for (int du = -2; du <= 3; ++du) {
        bool need = false;
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          const int k = cl2p_group(o, dx, du);
          const int reach = k == 0 ? 3 : k == 1 ? 1 : 0;
          if (k >= 0 && k <= 3 && zz >= -reach && zz < ZL + reach) need = true;
        }
        if (!need) continue;
        const double val = pv[zz * PP + dx + PX * du];
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          const int k = cl2p_group(o, dx, du);
          const int reach = k == 0 ? 3 : k == 1 ? 1 : 0;
          if (k < 0 || k > 3 || zz < -reach || zz >= ZL + reach) continue;
          g[o][k] += val;
        }
      }
    }
#pragma unroll
    for (int o = 0; o < 2; ++o) {
#pragma unroll
      for (int z = (zz - 3 > 0 ? zz - 3 : 0); z <= (zz + 3 < ZL - 1 ? zz + 3 : ZL - 1); ++z) {
        const int dz = zz > z ? zz - z : z - zz;
        w[o][z] = fma(dz == 0 ? q00 : dz == 1 ? p.HW[1] : dz == 2 ? p.HW[2] : p.HW[3], g[o][0],
                      w[o][z]);
        if (dz <= 2)
          u1[o][z] = fma(dz == 0 ? p.GW[0] : dz == 1 ? p.GW[1] : p.GW[2], g[o][0], u1[o][z]);
        if (dz <= 1) u1[o][z] = fma(dz == 0 ? p.GW[3] : p.GW[4], g[o][1], u1[o][z]);
        if (dz == 0) {
          u1[o][z] = fma(p.GW[5], g[o][2], u1[o][z]);
          u1[o][z] = fma(p.GW[6], g[o][3], u1[o][z]);
        }
      }
      if (zz >= -1 && zz <= ZL) {   // c' v: into U1 at its plane, Z (c' v) into w
        const double cv = pc[zz * CP + o * CX] * g[o][0];
        if (zz - 1 >= 0 && zz - 1 < ZL) w[o][zz - 1] += cv;
        if (zz + 1 >= 0 && zz + 1 < ZL) w[o][zz + 1] += cv;
        if (own) {
          w[o][zz] = fma(-2.0, cv, w[o][zz]);
          u1[o][zz] += cv;
        }
      }
    }
    }
  }
}

// planes [ZZ, ZEND), unrolled by recursion (a 16-plane loop of this body is not fully unrolled
// by the compiler at E = 20, which would put w and U1 in local memory)
template <int E, int ZZ, int ZEND>
__device__ __forceinline__ void hy_planes(const Ras3Cl2Args& p, double q00, const double* pv,
                                          const double* pc, int rank, double (&w)[2][E / 2],
                                          double (&u1)[2][E / 2]) {
  if constexpr (ZZ < ZEND) {
    hy_plane<E, ZZ>(p, q00, pv, pc, rank, w, u1);
    hy_planes<E, ZZ + 1, ZEND>(p, q00, pv, pc, rank, w, u1);
  }
}
template <int E, int PART>
__device__ __forceinline__ void hy_stageA(const Ras3Cl2Args& p, double q00, const double* pv,
                                          const double* pc, int rank, double (&w)[2][E / 2],
                                          double (&u1)[2][E / 2]) {
  constexpr int ZL = E / 2;
  if constexpr (PART == 0) {
    hy_planes<E, 0, ZL>(p, q00, pv, pc, rank, w, u1);
  } else {
    hy_planes<E, -3, 0>(p, q00, pv, pc, rank, w, u1);
    hy_planes<E, ZL, ZL + 3>(p, q00, pv, pc, rank, w, u1);
  }
}

// ring column q in [0, 4E) next to a box face: offsets (c'-plane layout) of the ring column,
// its box neighbour and the step along the face; v-plane offset of the box neighbour
template <int E>
__device__ __forceinline__ void hz_ring(int q, int& ro, int& bo, int& eo, int& vo) {
  using C = Cl2p<E>;
  const int s = q / E, i = q - s * E;
  int bx, by, rx, ry;
  if (s == 0) { bx = 0; by = i; rx = -1; ry = i; eo = C::CX; }
  else if (s == 1) { bx = E - 1; by = i; rx = E; ry = i; eo = C::CX; }
  else if (s == 2) { bx = i; by = 0; rx = i; ry = -1; eo = 1; }
  else { bx = i; by = E - 1; rx = i; ry = E; eo = 1; }
  ro = (ry + 1) * C::CX + rx + 1;
  bo = (by + 1) * C::CX + bx + 1;
  vo = (by + 3) * C::PX + bx + 3;
}

template <int K, int E, int NRX>
constexpr size_t cl2t_smem_doubles() {
  using C = Cl2p<E>;
  return (size_t)C::NVB * C::PP + (size_t)C::NCB * C::CP + 2 * 2 * C::NW * RS + C::NW * 3 * RS +
         (CL2T_HORNER ? 2 * (size_t)C::ZL * C::CP : 0);
}

template <int K, int E, int NRX>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cl2p<E>::NT, 1)
    ras3d_cl2t_kernel(const __grid_constant__ Ras3Cl2Args p) {
  if (p.gate && *p.gate) return;     // uniform over the cluster: both CTAs leave at once
  using C = Cl2p<E>;
  constexpr int ZL = C::ZL, PL = C::PL, NW = C::NW, NTN = C::NTN;
  constexpr int PX = C::PX, PP = C::PP, CX = C::CX, CP = C::CP, NVB = C::NVB, NCB = C::NCB;
  constexpr int NR = Cl2pK<K, NRX>::NR, NS = 0, NG = 0;
  constexpr int NTM = K - 1 - NR;              // basis vectors NR..K-2 in tensor memory
  constexpr int TMC = 4 * ZL;                  // TMEM columns per vector (2 x ZL doubles)
  static_assert(NTM * TMC <= 256, "two warps share a TMEM lane quarter: 256 columns each");
  constexpr int NE = E * E * E;
  extern __shared__ __align__(128) double smem_dyn[];
  double* vb = smem_dyn;                 // NVB padded planes of v_j (rank 0: zl in [0, ZL+3),
                                         // rank 1: [-3, ZL))
  double* cb = vb + NVB * PP;            // NCB padded planes of c' (rank 0: [0, ZL], rank 1:
                                         // [-1, ZL))
  double* vs = cb + NCB * CP;            // NS x [col][zl][thread]: basis vectors NR..NR+NS-1
  constexpr int HZP = CL2T_HORNER ? ZL * CP : 0;
  double* ub = vs + NS * 2 * ZL * NTN;   // Horner form: ZL planes of U2 (c'-plane layout) ...
  double* qb = ub + HZP;                 // ... and of U1
  double* red = qb + HZP;                // 2 buffers x [rank][warp][RS]
  double* hw = red + 2 * 2 * NW * RS;    // per warp: h1, h2, scratch
  __shared__ double H[(K + 1) * K];
  __shared__ double gv[K + 1], cs[K], sn[K], yv[K];
  __shared__ __align__(8) uint64_t mbar[3];
  __shared__ uint32_t tm_base;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool g0 = wid == NW - 1 && lane == 0;
  const int rank = (int)cluster_rank(), partner = rank ^ 1;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const bool act = tid < NTN;
  const int x = act ? tid % E : 0, y0 = act ? 2 * (tid / E) : 0;
  const int colp = (y0 + 3) * PX + (x + 3);        // padded v column of (x, y0)
  const int colc = (y0 + 1) * CX + (x + 1);        // padded c' column of (x, y0)
  const int pv0 = rank == 0 ? 0 : 3, pc0 = rank == 0 ? 0 : 1;   // plane of zl = 0
  const double* pv = vb + pv0 * PP + colp;
  const double* pc = cb + pc0 * CP + colc;
  double* pu = ub + colc;
  double* pq = qb + colc;
  double* gs = p.gscr + (size_t)blockIdx.x * (NG > 0 ? NG : 1) * 2 * ZL * NTN + tid;
  double* h1 = hw + wid * 3 * RS;
  double* h2 = h1 + RS;
  double* hx = h2 + RS;
  const uint32_t red_rem = mapa_rank(smem_u32(red), (uint32_t)partner);
  const uint32_t vb_rem = mapa_rank(smem_u32(vb), (uint32_t)partner);
  const int nbx = p.nx / p.bx, nby = p.ny / p.by, nbz = p.nz / p.bz;
  const int nboxes = nbx * nby * nbz;
  const size_t NX = p.nx, NXY = (size_t)p.nx * p.ny;

  int rb = 0;
  const uint32_t mbar_rem0 = mapa_rank(smem_u32(&mbar[0]), (uint32_t)partner);
  // zero v planes (ring stays zero) and finite c'
  for (int q = tid; q < NVB * PP + NCB * CP + 2 * HZP; q += blockDim.x) vb[q] = 0.0;
  if (tid == 0) {
    for (int q = 0; q < 3; ++q) mbar_init(&mbar[q], 1);
    fence_mbar_init();
  }
  if (wid == 0) tm_alloc512(&tm_base);   // all 512 columns (one CTA per SM: registers)
  tc_fence_before();
  cl_sync();   // the partner is running, zeroed and its mbarriers initialised before any DSMEM store
  tc_fence_after();
  // this thread's TMEM row: lane quarter of its warp, column half by warp pair (w, w + 4)
  const uint32_t tma = tm_base + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)(256 * (wid >> 2));
  {  // finite basis slots: the final V y reads every slot, with a zero coefficient beyond the
     // steps taken
    double zr[2][ZL];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int zl = 0; zl < ZL; ++zl) zr[c][zl] = 0.0;
#pragma unroll
    for (int s = 0; s < NTM; ++s) tm_st_vec<ZL>(tma + (uint32_t)(s * TMC), zr);
    tm_wait_st();
  }
#ifdef CL2_PROF
  long long c2p_acc[16] = {0}, c2p_last = clock64();
#endif
  uint32_t ph = 0;
  constexpr uint32_t HALO_BYTES = (uint32_t)PL * 3u * 8u;
  auto reduce = [&](int nsent, int nget, double* hwv) {
    if (tid == 0) mbar_expect_tx(&mbar[rb], (uint32_t)(NW * nsent * 8));
    __syncthreads();
    mbar_wait_cluster(&mbar[rb], (ph >> rb) & 1u);
    ph ^= 1u << rb;
    cl2_get<NW>(nget, red + rb * 2 * NW * RS, hwv, lane);
    rb ^= 1;
  };

  double vr[NR > 0 ? NR : 1][2][ZL];
#pragma unroll
  for (int s = 0; s < (NR > 0 ? NR : 1); ++s)
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int zl = 0; zl < ZL; ++zl) vr[s][c][zl] = 0.0;
  for (int box = cid; box < nboxes; box += ncl) {
    const int ibx = box % nbx, iby = (box / nbx) % nby, ibz = box / (nbx * nby);
    const int gx0 = ibx * p.bx - p.o, gy0 = iby * p.by - p.o, gz0 = ibz * p.bz - p.o;
    const int ez0 = rank * ZL;
    double w[2][ZL];
    double acc = 0.0;
    if (act) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int y = y0 + c;
        const size_t gxy = (size_t)wrapi(gx0 + x, p.nx) + NX * wrapi(gy0 + y, p.ny);
        const bool oxy = x >= p.o && x < p.o + p.bx && y >= p.o && y < p.o + p.by;
        int gz = wrapi(gz0 + ez0, p.nz);   // wrapped z of own plane 0, advanced without '%'
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl, gz = gz + 1 == p.nz ? 0 : gz + 1) {
          const size_t g = gxy + NXY * (size_t)gz;
          const int ez = ez0 + zl;
          const bool owned = oxy && ez >= p.o && ez < p.o + p.bz;
          w[c][zl] = (p.restrict_owned && !owned) ? 0.0 : p.v[g];
          cb[(zl + pc0) * CP + colc + c * CX] = -p.ih2 * p.c[g];
          acc = fma(w[c][zl], w[c][zl], acc);
        }
        const int zh = rank == 0 ? ZL : -1;
        cb[(zh + pc0) * CP + colc + c * CX] =
            -p.ih2 * p.c[gxy + NXY * wrapi(gz0 + ez0 + zh, p.nz)];
      }
    } else {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) w[c][zl] = 0.0;
    }
    double* redb = red + rb * 2 * NW * RS;
    uint32_t redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
    uint32_t mbr = mbar_rem0 + 8u * rb;
    C2P(0);
    cl2_put<NW>(acc, 0, redb, redr, mbr, rank, wid, lane);
    reduce(1, 1, hx);
    C2P(1);
    const double beta = sqrt(hx[0]);
    if (beta == 0.0) {
      if (act) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) {
            const int y = y0 + c;
            const int ez = ez0 + zl, li = x - p.o, lj = y - p.o, lk = ez - p.o;
            if (p.y_ext) p.y_ext[(size_t)box * NE + (ez * E + y) * E + x] = 0.0;
            else if (li >= 0 && li < p.bx && lj >= 0 && lj < p.by && lk >= 0 && lk < p.bz)
              p.z[(size_t)(ibx * p.bx + li) + NX * (iby * p.by + lj) + NXY * (ibz * p.bz + lk)] = 0.0;
          }
      }
      if (tid == 0 && rank == 0) ras_count(p.jcnt, 0);
      continue;
    }
    auto put_v = [&](int slot) {
      // tensor memory: warp-collective, every lane (inactive lanes store their zero w)
      if (slot >= NR && slot < K - 1) tm_st_vec<ZL>(tma + (uint32_t)((slot - NR) * TMC), w);
      if (!act) return;
#pragma unroll
      for (int s = 0; s < NR; ++s)
        if (s == slot) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int zl = 0; zl < ZL; ++zl) vr[s][c][zl] = w[c][zl];
        }
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) vb[(zl + pv0) * PP + colp + c * PX] = w[c][zl];
      const uint32_t hm = mbar_rem0 + 16u;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (rank == 0) {
#pragma unroll
          for (int q = 0; q < 3; ++q)
            st_async(vb_rem + (uint32_t)(q * PP + colp + c * PX) * 8u, w[c][ZL - 3 + q], hm);
        } else {
#pragma unroll
          for (int q = 0; q < 3; ++q)
            st_async(vb_rem + (uint32_t)((ZL + q) * PP + colp + c * PX) * 8u, w[c][q], hm);
        }
      }
    };
    // basis vector i of the thread's 2 x ZL nodes: registers (i < NR), tensor memory (NR <= i <
    // K-1, warp-collective load: called by every lane) or the stencil planes (i = K-1)
    auto getv = [&](int i, double (&vt)[2][ZL]) {   // (i a constant after unrolling)
      if (i < NR) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) vt[c][zl] = vr[i < NR ? i : 0][c][zl];
      } else if (i < K - 1) {
        tm_ld_vec<ZL>(tma + (uint32_t)((i - NR) * TMC), vt);
      } else {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) vt[c][zl] = pv[zl * PP + c * PX];
      }
    };
    {
      const double ib = 1.0 / beta;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) w[c][zl] *= ib;
      put_v(0);
    }
    if (g0) gv[0] = beta;
    int jm = 0;
    double hn_prev = 0.0;
#pragma unroll 1
    for (int j = 0; j < K; ++j) {
      C2P(10);
      if (tid == 0) mbar_expect_tx(&mbar[2], HALO_BYTES);
      __syncthreads();
      C2P(2);
      if (g0 && j > 0) givens_col(j - 1, h1, h2, hn_prev, H, cs, sn, gv, K + 1);
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) w[c][zl] = 0.0;
#if CL2T_HORNER == 2
      double u1[2][ZL];
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) u1[c][zl] = 0.0;
      const double q00 = dt_inv(p.dtp, p.idt) + p.HW[0];
      if (act) hy_stageA<E, 0>(p, q00, pv, pc, rank, w, u1);
      C2P(3);
      mbar_wait_cluster(&mbar[2], (ph >> 2) & 1u);
      ph ^= 4u;
      if (act) {
        hy_stageA<E, 1>(p, q00, pv, pc, rank, w, u1);
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) {
          pq[zl * CP] = u1[0][zl];
          pq[zl * CP + CX] = u1[1][zl];
        }
      } else if (wid == NW - 1) {
        // ring columns next to a box face: U1 from the box columns within radius 2 (the box
        // neighbour b with its z-neighbours, b +- the step along the face, b one step inwards)
        for (int q = lane; q < 4 * E; q += 32) {
          int ro, bo, eo, vo;
          hz_ring<E>(q, ro, bo, eo, vo);
          const int s = q / E;
          const int ev = s < 2 ? PX : 1;                               // along the face (v planes)
          const int nv = s == 0 ? 1 : s == 1 ? -1 : s == 2 ? PX : -PX;   // inwards
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) {
            const double* vp = vb + (zl + pv0) * PP + vo;
            const double dn = (zl > 0 || rank != 0) ? vp[-PP] : 0.0;
            const double up = (zl < ZL - 1 || rank != 1) ? vp[PP] : 0.0;
            double r = p.GW[3] * vp[0];
            r = fma(p.GW[4], dn + up, r);
            r = fma(p.GW[6], vp[ev] + vp[-ev], r);
            r = fma(p.GW[5], vp[nv], r);
            qb[zl * CP + ro] = r;
          }
        }
      }
      __syncthreads();
      C2P(4);
      if (act) hz_stage3<E>(pq, u1, w);
      C2P(5);
#elif CL2T_HORNER
      double u1[2][ZL], u2[2][ZL];
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) {
          u1[c][zl] = 0.0;
          u2[c][zl] = 0.0;
        }
      const double q00 = dt_inv(p.dtp, p.idt) + p.HW[0];
      if (act) {
        hz_stage1<E, 0>(p, q00, pv, pc, pu, rank, w, u1, u2);
      } else if (wid == NW - 1) {   // ring columns: U2 = a3 v(box neighbour)
        for (int q = lane; q < 4 * E; q += 32) {
          int ro, bo, eo, vo;
          hz_ring<E>(q, ro, bo, eo, vo);
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl)
            ub[zl * CP + ro] = p.HW[3] * vb[(zl + pv0) * PP + vo];
        }
      }
      C2P(3);
      mbar_wait_cluster(&mbar[2], (ph >> 2) & 1u);
      ph ^= 4u;
      if (act) hz_stage1<E, 1>(p, q00, pv, pc, pu, rank, w, u1, u2);
      __syncthreads();
      C2P(4);
      if (act) {
        hz_stage2<E>(pu, pq, u1);
      } else if (wid == NW - 1) {   // ring columns: U1 = T U2 (the outer neighbour is zero)
        for (int q = lane; q < 4 * E; q += 32) {
          int ro, bo, eo, vo;
          hz_ring<E>(q, ro, bo, eo, vo);
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) {
            const double* u = ub + zl * CP;
            qb[zl * CP + ro] = fma(-4.0, u[ro], (u[bo] + u[ro + eo]) + u[ro - eo]);
          }
        }
      }
      __syncthreads();
      C2P(15);
      if (act) hz_stage3<E>(pq, u1, w);
      C2P(5);
#else
      if (act) cl2p_stencil<E, 0, ZL>(p, pv, pc, w);
      C2P(3);
      mbar_wait_cluster(&mbar[2], (ph >> 2) & 1u);
      ph ^= 4u;
      C2P(4);
      if (act) {
        if (rank == 0) cl2p_stencil<E, ZL, ZL + 3>(p, pv, pc, w);
        else cl2p_stencil<E, -3, 0>(p, pv, pc, w);
      }
      C2P(5);
#endif
      double hn2 = 0.0;
      auto cgs2 = [&](auto Jc) {
        constexpr int J = decltype(Jc)::value;
        tm_wait_st();   // this thread's TMEM stores of v_j (put_v, a stencil ago) have landed
        redb = red + rb * 2 * NW * RS;
        redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
        mbr = mbar_rem0 + 8u * rb;
        {
          double acc[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] = 0.0;
          // vector by vector
          #pragma unroll
          for (int I = 0; I < J + 1; ++I) {
            double vt[2][ZL];
            getv(I, vt);
            if (act) {   // four independent chains (FP64 latency), summed in a fixed order
              double q4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
              for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int zl = 0; zl < ZL; ++zl)
                  q4[2 * c + (zl & 1)] = fma(vt[c][zl], w[c][zl], q4[2 * c + (zl & 1)]);
              acc[I] = (q4[0] + q4[1]) + (q4[2] + q4[3]);
            }
          }
          C2P(11);
          cl2_put_multi<NW>(acc, J + 1, redb, redr, mbr, rank, wid, lane);
        }
        reduce(J + 1, J + 1, h1);
        C2P(12);
        redb = red + rb * 2 * NW * RS;
        redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
        mbr = mbar_rem0 + 8u * rb;
        {
          double hv[J + 1], acc[16], nrm = 0.0;
#pragma unroll
          for (int i = 0; i <= J; ++i) hv[i] = h1[i];
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] = 0.0;
          // w <- w - V h1 (per node in the order i = 0..J), then h2 = V^T w and |w|^2
          #pragma unroll
          for (int I = 0; I < J + 1; ++I) {
            double vt[2][ZL];
            getv(I, vt);
            if (act) {
#pragma unroll
              for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int zl = 0; zl < ZL; ++zl) w[c][zl] = fma(-hv[I], vt[c][zl], w[c][zl]);
            }
          }
          #pragma unroll
          for (int I = 0; I < J + 1; ++I) {
            double vt[2][ZL];
            getv(I, vt);
            if (act) {   // four independent chains (FP64 latency), summed in a fixed order
              double q4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
              for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int zl = 0; zl < ZL; ++zl)
                  q4[2 * c + (zl & 1)] = fma(vt[c][zl], w[c][zl], q4[2 * c + (zl & 1)]);
              acc[I] = (q4[0] + q4[1]) + (q4[2] + q4[3]);
            }
          }
          if (act) {
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int zl = 0; zl < ZL; ++zl) nrm = fma(w[c][zl], w[c][zl], nrm);
          }
          C2P(13);
          cl2_put_multi<NW>(acc, J + 1, redb, redr, mbr, rank, wid, lane);
          cl2_put<NW>(nrm, J + 1, redb, redr, mbr, rank, wid, lane);
        }
        reduce(J + 2, J + 2, h2);
        C2P(14);
        double h2n = 0.0;
        for (int i = 0; i <= J; ++i) h2n += h2[i] * h2[i];
        const double wn2 = h2[J + 1];
        {
          double hv[J + 1];
#pragma unroll
          for (int i = 0; i <= J; ++i) hv[i] = h2[i];
          #pragma unroll
          for (int I = 0; I < J + 1; ++I) {
            double vt[2][ZL];
            getv(I, vt);
            if (act) {
#pragma unroll
              for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int zl = 0; zl < ZL; ++zl) w[c][zl] = fma(-hv[I], vt[c][zl], w[c][zl]);
            }
          }
        }
        if (h2n <= 1e-8 * wn2) {
          hn2 = wn2 - h2n;
        } else {
          redb = red + rb * 2 * NW * RS;
          redr = red_rem + (uint32_t)(rb * 2 * NW * RS) * 8u;
          mbr = mbar_rem0 + 8u * rb;
          double s = 0.0;
          if (act) {
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int zl = 0; zl < ZL; ++zl) s = fma(w[c][zl], w[c][zl], s);
          }
          cl2_put<NW>(s, 0, redb, redr, mbr, rank, wid, lane);
          reduce(1, 1, hx);
          hn2 = hx[0];
        }
        return hn2;
      };
      dispatch_j<K>(j, cgs2);
      C2P(6);
      const double hn = sqrt(hn2 > 0.0 ? hn2 : 0.0);
      hn_prev = hn;
      jm = j + 1;
      if (hn <= 1e-14 * beta) break;
      if (j + 1 < K) {
        const double ihn = 1.0 / hn;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) w[c][zl] *= ihn;
        put_v(j + 1);
      }
    }
    C2P(10);
    if (g0) {
      const int ld = K + 1;
      givens_col(jm - 1, h1, h2, hn_prev, H, cs, sn, gv, ld);
      for (int i = jm - 1; i >= 0; --i) {
        double s = gv[i];
        for (int l = i + 1; l < jm; ++l) s -= H[i + ld * l] * yv[l];
        yv[i] = s / H[i + ld * i];
      }
      for (int i = jm; i < K; ++i) yv[i] = 0.0;   // steps not taken: zero coefficients
      if (rank == 0) ras_count(p.jcnt, jm);
    }
    __syncthreads();
    C2P(7);
    tm_wait_st();
    {   // (every lane: the tensor-memory loads are warp-collective; only node lanes store)
      // y = V yv over every slot (fma(0, v, s) = s exactly for the finite unused slots)
      double yl[2][ZL];
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) yl[c][zl] = 0.0;
      #pragma unroll
      for (int I = 0; I < K; ++I) {
        double vt[2][ZL];
        getv(I, vt);
        const double yi = yv[I];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int zl = 0; zl < ZL; ++zl) yl[c][zl] = fma(yi, vt[c][zl], yl[c][zl]);
      }
#pragma unroll
      for (int c = 0; c < 2 && act; ++c) {
        const int y = y0 + c;
#pragma unroll
        for (int zl = 0; zl < ZL; ++zl) {
          const int ez = ez0 + zl, li = x - p.o, lj = y - p.o, lk = ez - p.o;
          if (p.y_ext) {
            p.y_ext[(size_t)box * NE + (ez * E + y) * E + x] = yl[c][zl];
          } else if (li >= 0 && li < p.bx && lj >= 0 && lj < p.by && lk >= 0 && lk < p.bz) {
            p.z[(size_t)(ibx * p.bx + li) + NX * (iby * p.by + lj) + NXY * (ibz * p.bz + lk)] =
                yl[c][zl];
          }
        }
      }
    }
    C2P(9);
  }
  C2P(8);
#ifdef CL2_PROF
  if (blockIdx.x == 0 && tid == 0)
    for (int i = 0; i < 16; ++i) cl2_prof[i] += c2p_acc[i];
#endif
  tc_fence_before();
  cl_sync();   // no CTA leaves while its partner may still address its shared memory
  tc_fence_after();
  if (wid == 0) tm_dealloc512(tm_base);
}


typedef void (*ras3cl2_fn)(const Ras3Cl2Args);

// NR = basis vectors in registers (1, 2 or 3; PFC_CL2_NR selects, default 1: measured fastest)
int cl2_nr() {
  const int nr = getenv("PFC_CL2_NR") ? atoi(getenv("PFC_CL2_NR")) : 1;
  return nr == 3 ? 3 : nr == 2 ? 2 : 1;
}

// columns per thread: 1 (ras3d_cl2_kernel) or 2 (ras3d_cl2p_kernel); PFC_CL2_CP selects
int cl2_cp() {   // default 3: the two-column kernel with the basis in tensor memory
                 // (ras3d_cl2t_kernel), 37.6 ms per 512^3 apply vs 39.2 ms (2, shared memory +
                 // L2 scratch) vs 50.1 ms (1)
  const char* e = getenv("PFC_CL2_CP");
  return e && e[0] == '1' ? 1 : (e && e[0] == '2') ? 2 : 3;
}

ras3cl2_fn pick_cl2(int k, int e, size_t* smem, int* threads, int* ng) {
  const int nr = cl2_nr();
  if (cl2_cp() == 3) {
    const char* en = getenv("PFC_CL2_NR");
    const int nr2 = en ? atoi(en) : 3;
#define C2T(K, E, NR)                                               \
    if (k == K && e == E && nr2 == NR) {                            \
      *smem = cl2t_smem_doubles<K, E, NR>() * sizeof(double);       \
      *threads = Cl2p<E>::NT;                                       \
      *ng = 0;                                                      \
      return ras3d_cl2t_kernel<K, E, NR>;                           \
    }
    C2T(10, 20, 3) C2T(4, 20, 3) C2T(10, 12, 3) C2T(4, 12, 3)
#undef C2T
    return nullptr;
  }
  if (cl2_cp() == 2) {
    const char* en = getenv("PFC_CL2_NR");
    const int nr2 = en ? atoi(en) : 3;   // measured fastest (NR = 4 spills at 255 registers)
#define C2P2(K, E, NR)                                              \
    if (k == K && e == E && nr2 == NR) {                            \
      *smem = cl2p_smem_doubles<K, E, NR>() * sizeof(double);       \
      *threads = Cl2p<E>::NT;                                       \
      *ng = Cl2pK<K, NR>::NG;                                       \
      return ras3d_cl2p_kernel<K, E, NR>;                           \
    }
    C2P2(10, 20, 3) C2P2(4, 20, 3) C2P2(10, 12, 3) C2P2(4, 12, 3)
    C2P2(10, 20, 1) C2P2(10, 20, 2) C2P2(10, 20, 4)
#undef C2P2
    return nullptr;
  }
#define C2(K, E, NR)                                                \
  if (k == K && e == E && nr == NR) {                               \
    *smem = cl2_smem_doubles<K, E, NR>() * sizeof(double);          \
    *threads = Cl2<E>::NT;                                          \
    *ng = Cl2K<K, NR>::NG;                                          \
    return ras3d_cl2_kernel<K, E, NR>;                              \
  }
  C2(10, 20, 1) C2(4, 20, 1) C2(10, 12, 1) C2(4, 12, 1) C2(10, 20, 2) C2(10, 20, 3)
#undef C2
  return nullptr;
}

}  // namespace

// 1 if the 2-CTA cluster kernel handles this configuration (cubic extended box with an even
// edge, instantiated K and E, periodic, M = 1); *clusters = concurrent clusters to launch
int ras3d_cl2_plan(pfc_ctx* ctx, int* clusters, size_t* scratch_doubles) {
  const pfc_config& c = ctx->cfg;
  const int e = c.ras_box[0] + 2 * c.ras_overlap;
  if (c.ras_box[1] != c.ras_box[0] || c.ras_box[2] != c.ras_box[0] || (e & 3)) return 0;
  size_t smem = 0;
  int threads = 0, ng = 0;
  if (!pick_cl2(c.ras_local_k, e, &smem, &threads, &ng)) return 0;
  if (smem + 2048 > 227 * 1024) return 0;
  const int nboxes = (c.n[0] / c.ras_box[0]) * (c.n[1] / c.ras_box[1]) * (c.n[2] / c.ras_box[2]);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  *clusters = nboxes < sms / 2 ? nboxes : sms / 2;
  *scratch_doubles = (size_t)2 * (*clusters) * (ng > 0 ? ng : 1) * (e / 2) * e * e;
  return 1;
}

cudaError_t launch_ras_3d_cl2(pfc_ctx* ctx, const double* v, const double* c, double dt,
                              double* z, double* scratch) {
  const pfc_config& cf = ctx->cfg;
  const int e = cf.ras_box[0] + 2 * cf.ras_overlap;
  size_t smem = 0;
  int threads = 0, ng = 0;
  ras3cl2_fn fn = pick_cl2(cf.ras_local_k, e, &smem, &threads, &ng);
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
  p.dtp = ctx->dtdev;
  p.W[1] = -al * ih2 + 12.0 * ih4 - 61.5 * ih6;
  p.W[2] = -ih4 + 9.0 * ih6;
  p.W[3] = -2.0 * ih4 + 18.0 * ih6;
  p.W[4] = -0.5 * ih6;
  p.W[5] = -1.5 * ih6;
  p.W[6] = -3.0 * ih6;
  p.ih2 = ih2;
  p.idt = 1.0 / dt;
  {   // Horner-in-T form: z-weights of q0, q1, q2 (Z = [1 -2 1], Z^2 = [1 -4 6 -4 1],
      // Z^3 = [1 -6 15 -20 15 -6 1])
    const double a1 = -al * ih2, a2 = -ih4, a3 = -0.5 * ih6;
    p.HW[0] = -2.0 * a1 + 6.0 * a2 - 20.0 * a3;   // + 1/dt in the kernel
    p.HW[1] = a1 - 4.0 * a2 + 15.0 * a3;
    p.HW[2] = a2 - 6.0 * a3;
    p.HW[3] = a3;
    p.HW[4] = a1 - 4.0 * a2 + 18.0 * a3;
    p.HW[5] = 2.0 * a2 - 12.0 * a3;
    p.HW[6] = 3.0 * a3;
    p.HW[7] = a2 - 6.0 * a3;
    p.HW[8] = 3.0 * a3;
    p.GW[0] = p.HW[4] - 4.0 * p.HW[7] + 20.0 * a3;   // T = [1 1 -4 1 1], T^2: 20, -8, 1, 2
    p.GW[1] = p.HW[5] - 4.0 * p.HW[8];
    p.GW[2] = p.HW[6];
    p.GW[3] = p.HW[7] - 8.0 * a3;
    p.GW[4] = p.HW[8];
    p.GW[5] = a3;
    p.GW[6] = 2.0 * a3;
  }
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

#ifdef CL2_PROF
extern "C" void pfc_cl2_prof_read(long long* out) {
  cudaMemcpyFromSymbol(out, cl2_prof, sizeof(long long) * 16);
  long long z[16] = {0};
  cudaMemcpyToSymbol(cl2_prof, z, sizeof(z));
}
#endif
