// stencil3d.cu -- fused 3D DVD residual (K1) and Jacobian-vector product (K2), sm_100a.
//
// Same operators as stencil2d.cu (Eq. NSOP, Eq. discretedG, Eq. Jacobi
// P:351-356), the 7-point Delta_d composed three times (a radius-3, 63-point stencil).  With
// the UNSCALED Laplacian  Lt f = sum of the 6 neighbours - 6 f  (Delta_d = ih2 * Lt, ih2 = 1/h^2):
//   resid: s = Phi + psi (= 2u),  N = (Phi^3 + Phi^2 psi + Phi psi^2 + psi^3)/4 = s (Phi^2+psi^2)/4
//          A = (1-gamma)/2 s + ih2 Lt s + ih2^2/2 Lt Lt s + N   (= (1-gamma)u + 2 Delta u + Delta^2 u + N)
//          F = (Phi - psi)/dt - ih2 Lt A
//   jv:    B = ((1-gamma)/2 + c) v + ih2 Lt v + ih2^2/2 Lt Lt v,   Jv = v/dt - ih2 Lt B
//
// 2.5D z-march.  A CTA owns a 32 x 32 column of outputs and a chunk of z-planes; input planes
// z0-3 .. z0+zc+2 stream through a RING-slot ring per field.  The input window of a plane is
// loaded by TMA (cp.async.bulk.tensor.3d) as two 42 x 20 boxes (rows 0..19 | 20..39).
// Periodic wrap without any fix-up: when n_x, n_y are multiples of 32 the tile origins are
// shifted to x0 = 32k - 18, y0 = 32j - 16, so the periodic seam y = 0 falls on the boxes' row
// boundary (row 20), and in the one tile column that straddles x = 0 the window is loaded as
// four 22 x 20 boxes split at col 22, where the seam x = 0 falls: every box is one in-range
// rectangle at wrapped coordinates (TMA has no wrap mode).  Other grids (ragged or too small
// for TMA) use unshifted tiles, and the producer warp re-reads the out-of-range cells (or all
// cells) with wrapped indices.  Warp specialisation:
//  * the producer warp issues every TMA load (full / empty mbarriers per slot) and, on such
//    grids, makes the periodic fix-up (fixd mbarrier);
//  * compute thread i < 324 owns the 2 x 2 point block (pair column p, row strip s), p, s in
//    1..18, of the window, i.e. the halo-2 region; at streamed plane t it computes
//        Lt s|v (t-1)  ->  A|B (t-2)  ->  F|Jv (t-3)
//    with z-neighbours, block-internal neighbours and the block's own values in registers (every
//    queue has period 3, so the 3x-unrolled loop rotates it by register renaming) and only the
//    block's 8 outside neighbours read from shared memory.  The intermediate planes Lt and A|B
//    are kept in an even/odd-column split layout with a row pitch of 25 doubles, which makes
//    every shared access of a warp conflict-free.  Each stage reads planes written in the
//    previous iteration: a split-phase mbarrier (arrive after the plane stores, wait before the
//    neighbour loads) separates iterations, and the neighbour-free parts of the three Laplacians
//    are computed before the wait.  Optional fused ||F||^2 partial per CTA.
#include "pfc_device.cuh"
#include "pfc_internal.h"

#include <algorithm>
#include <functional>
#include <queue>
#include <vector>

#ifndef ST3_TWO_PHASE
#define ST3_TWO_PHASE 1   // 0: chunks only (the round-1 plan), diagnostic
#endif

#ifndef ST3_RES_SHFL
#define ST3_RES_SHFL 0    // 1: residual takes the left / right stage-1 neighbours of s by warp
                          // shuffles (diagnostic: bitwise equal, but 68 B of spills in the z-march
                          // loop at the 168-register cap: 0.736 -> 1.172 ms at 512^3, not kept)
#endif

namespace {

constexpr int TX = 32, TY = 32;
constexpr int WY = 40;              // window rows y0-4 .. y0+35
constexpr int BH = 20;              // TMA box rows (upper / lower half of the window)
// natural layout (every tile except the x-seam column): two 42 x 20 boxes, row pitch 42
constexpr int NW = 42, NYB = 848;   // box width; offset of the lower box (128-B aligned)
// split layout (x-seam tiles): four 22 x 20 boxes, cols 0..21 | 22..43, row pitch 22
constexpr int BW = 22, BOXN = 448;  // box width; doubles per box incl. padding (22 x 20 = 440)
constexpr int XB = BOXN, YB = 2 * BOXN;    // offsets of the right-hand and lower boxes
constexpr int WS = 4 * BOXN;        // doubles per ring slot (14336 B), either layout
constexpr int NPB = 18;             // stage region: pair columns 1..18 x strips 1..18
constexpr int NBLK = NPB * NPB;     // 324 blocks
constexpr int NTC = 352;            // 11 compute warps
constexpr int NWC = NTC / 32;
constexpr int NT = NTC + 32;        // + 1 producer warp (TMA issue, periodic fix-up)
// ring depth per operator.  LAG: a plane's slot is released LAG iterations after the plane's
// own iteration (J v reads the input ring's plane t-1 for the stage-1 neighbours: LAG 1; the
// residual takes them from its s = Phi + psi split planes: LAG 0); PF <= RING - 1 - LAG.
template <int OP> struct Cfg { static constexpr int RING = 5, PF = 3, NSPL = 4, LAG = 1; };
constexpr int SP = 25;              // split-plane row pitch (doubles)
constexpr int SROWS = WY;
constexpr int SO = SROWS * SP;      // offset of the odd-column half
constexpr int SPLANE = 2 * SO;      // doubles per split plane
template <int OP> constexpr int smem_bytes() {
  return (2 * Cfg<OP>::RING * WS + Cfg<OP>::NSPL * SPLANE) * (int)sizeof(double);
}

// slot offset of window cell (row r, col c)
__host__ __device__ constexpr int woff_nat(int r, int c) {
  return (r < BH ? r * NW : NYB + (r - BH) * NW) + c;
}
__host__ __device__ constexpr int woff_split(int r, int c) {
  return (r < BH ? r * BW : YB + (r - BH) * BW) + (c < BW ? c : XB + (c - BW));
}
__device__ __forceinline__ int woff(bool split, int r, int c) {
  return split ? woff_split(r, c) : woff_nat(r, c);
}

enum { OP_RESID = 0, OP_JV = 1 };
template <> struct Cfg<OP_RESID> { static constexpr int RING = 4, PF = 3, NSPL = 6, LAG = 0; };

struct S3Args {
  const double* a;   // Phi | v
  const double* b;   // psi | c
  double* out;
  double* partials;
  int nx, ny, nz;
  int zc;            // planes per chunk (items beyond the first n1)
  double idt, k0, k1, k2, kout;   // (1-gamma)/2, ih2, ih2^2/2, -ih2
  int mode;          // 0: plain loads; 1: TMA + wrapped re-reads; 2: seam-aligned TMA tiles
  const int* gate;   // device-resident FGMRES: skip the launch when *gate != 0 (f1)
  const double* dtp; // graph path (f1): dt on the device
  int n1;            // the first n1 items are whole z-columns of tiles 0..n1-1 (two-phase plan)
  int ntiles;
};

struct q4 { double a, b, c, d; };   // (row0,col0) (row0,col1) (row1,col0) (row1,col1)

__device__ __forceinline__ double2 lds2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}
__device__ __forceinline__ void stg2(double* p, double x, double y) {
  *reinterpret_cast<double2*>(p) = make_double2(x, y);
}

// window-relative offsets of one block's accesses; row 1 of a pair / scalar: + pitch
struct boff { int own, l, r, t, d, pitch; };

// sums of the outside xy neighbours of the block from a ring slot
__device__ __forceinline__ q4 out_ring(const double* f, const boff& o) {
  const double L0 = f[o.l], R0 = f[o.r], L1 = f[o.l + o.pitch], R1 = f[o.r + o.pitch];
  const double2 T = lds2(f + o.t), D = lds2(f + o.d);
  return {L0 + T.x, R0 + T.y, L1 + D.x, R1 + D.y};
}
// split layout: E(r,k) = P[r*SP + k] (window col 2k), O(r,k) = P[SO + r*SP + k] (col 2k+1)
__device__ __forceinline__ q4 out_split(const double* P, int e0) {
  const double L0 = P[SO + e0 - 1], L1 = P[SO + e0 + SP - 1];
  const double R0 = P[e0 + 1], R1 = P[e0 + SP + 1];
  const double Ta = P[e0 - SP], Tb = P[SO + e0 - SP];
  const double Da = P[e0 + 2 * SP], Db = P[SO + e0 + 2 * SP];
  return {L0 + Ta, R0 + Tb, L1 + Da, R1 + Db};
}
__device__ __forceinline__ void st_split(double* P, int e0, const q4& v) {
  P[e0] = v.a;
  P[SO + e0] = v.b;
  P[e0 + SP] = v.c;
  P[SO + e0 + SP] = v.d;
}
// unscaled 7-point Laplacian of the block WITHOUT its outside xy neighbours: in-block xy
// neighbours, z-neighbours m and p (p omitted when it is added later), -6 times the centre f
__device__ __forceinline__ q4 lap_own(const q4& f, const q4& m, const q4& p) {
  q4 o;
  o.a = fma(-6.0, f.a, (f.b + f.c) + (m.a + p.a));
  o.b = fma(-6.0, f.b, (f.a + f.d) + (m.b + p.b));
  o.c = fma(-6.0, f.c, (f.d + f.a) + (m.c + p.c));
  o.d = fma(-6.0, f.d, (f.c + f.b) + (m.d + p.d));
  return o;
}
__device__ __forceinline__ q4 lap_own(const q4& f, const q4& m) {
  q4 o;
  o.a = fma(-6.0, f.a, (f.b + f.c) + m.a);
  o.b = fma(-6.0, f.b, (f.a + f.d) + m.b);
  o.c = fma(-6.0, f.c, (f.d + f.a) + m.c);
  o.d = fma(-6.0, f.d, (f.c + f.b) + m.d);
  return o;
}
__device__ __forceinline__ q4 add4(const q4& x, const q4& y) {
  return {x.a + y.a, x.b + y.b, x.c + y.c, x.d + y.d};
}

struct S3Maps {   // 42 x 20 (natural) and 22 x 20 (split) boxes of both fields
  CUtensorMap a, b, a22, b22;
};

template <int OP>
__global__ void __launch_bounds__(NT, 1) stencil3d_kernel(const __grid_constant__ S3Maps m,
                                                          const __grid_constant__ S3Args p) {
  constexpr int RING = Cfg<OP>::RING, PF = Cfg<OP>::PF, LAG = Cfg<OP>::LAG;
  extern __shared__ __align__(128) double smem_dyn[];
  double* ringA = smem_dyn;                 // RING slots: Phi | v
  double* ringB = ringA + RING * WS;        // RING slots: psi | c
  double* Lsp = ringB + RING * WS;          // 2 split planes: Lt s | Lt v
  double* Bsp = Lsp + 2 * SPLANE;           // 2 split planes: A | B
  double* Ssp = Bsp + 2 * SPLANE;           // resid: 2 split planes of s = Phi + psi
  __shared__ uint64_t full[RING];   // the slot's TMA boxes landed (transaction bytes)
  __shared__ uint64_t fixd[RING];   // the producer finished the periodic fix-up of the slot
  __shared__ uint64_t empty[RING];  // every compute warp finished reading the slot
  __shared__ uint64_t itbar;        // compute warps: split-phase iteration barrier
  __shared__ double red[64];

  if (p.gate && *p.gate) return;
  const double idt = dt_inv(p.dtp, p.idt);
  const int tid = threadIdx.x, lane = tid & 31;
  const int nx = p.nx, ny = p.ny, nz = p.nz;
  const int ntx = (nx + TX - 1) / TX;
  const bool tma = p.mode != 0, seam = p.mode == 2;
  // seam-aligned tiles (mode 2): the periodic seam lies on the boxes' shared edge; only the
  // tile column that straddles x = 0 needs the split (four-box) layout
  // work item -> (tile, z-chunk).  J v (1D grid): whole columns first, then the other tiles
  // chunk by chunk.  The residual keeps the chunk-only plan on a (tiles, chunks) grid: the
  // item decode costs it registers it does not have (24 B of spills in the z-march loop,
  // 0.735 -> 0.80 ms at 512^3).
  int tile = blockIdx.x, z0 = 0, zc = nz;
  if (OP == OP_RESID) {
    z0 = blockIdx.y * p.zc;
    zc = min(p.zc, nz - z0);
  } else if ((int)blockIdx.x >= p.n1) {
    const int r = blockIdx.x - p.n1, nt2 = p.ntiles - p.n1;
    tile = p.n1 + r % nt2;
    z0 = (r / nt2) * p.zc;
    zc = min(p.zc, nz - z0);
  }
  const bool split = seam && tile % ntx == 0;
  const int x0 = (tile % ntx) * TX - (seam ? 18 : 0);
  const int y0 = (tile / ntx) * TY - (seam ? 16 : 0);
  const int gx0 = x0 - 4, gy0 = y0 - 4;     // global coordinates of window cell (0,0)
  const size_t plane = (size_t)nx * ny;
  const int T = zc + 6;
  const int Tp = (T + 2) / 3 * 3;           // padded to the unroll factor; extra planes are inert
  // does a window cell the stencil reads (rows and cols 1..38) need a fix-up?
  const bool edge = !tma || (!seam && (x0 < 3 || y0 < 3 || x0 + 34 >= nx || y0 + 34 >= ny));

  if (tid == 0) {
    for (int i = 0; i < RING; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&fixd[i], 1);
      mbar_init(&empty[i], NWC);
    }
    mbar_init(&itbar, NWC);
    fence_mbar_init();
  }
  __syncthreads();
  double nrm = 0.0;

  if (tid >= NTC) {
    // ================= producer warp: TMA issue (and periodic fix-up) of every plane =========
    const int xa = seam ? wrapi(gx0, nx) : gx0, xb = seam ? wrapi(x0 + 18, nx) : x0 + 18;
    const int ya = seam ? wrapi(gy0, ny) : gy0, yb = seam ? wrapi(y0 + 16, ny) : y0 + 16;
    auto zof = [&](int q) { return wrapi(z0 - 3 + q, nz); };
    auto wait_empty = [&](int q) {   // plane q - RING released by every compute warp
      if (q >= RING) mbar_wait(&empty[q % RING], (uint32_t)((q / RING - 1) & 1));
    };
    auto issue = [&](int q) {
      const int sl = q % RING, zi = zof(q);
      wait_empty(q);
      if (lane == 0) {
        double* da = ringA + sl * WS;
        double* db = ringB + sl * WS;
        if (split) {
          mbar_expect_tx(&full[sl], 2u * 4u * BW * BH * (uint32_t)sizeof(double));
          tma_load_3d(da, &m.a22, &full[sl], xa, ya, zi);
          tma_load_3d(da + XB, &m.a22, &full[sl], xb, ya, zi);
          tma_load_3d(da + YB, &m.a22, &full[sl], xa, yb, zi);
          tma_load_3d(da + YB + XB, &m.a22, &full[sl], xb, yb, zi);
          tma_load_3d(db, &m.b22, &full[sl], xa, ya, zi);
          tma_load_3d(db + XB, &m.b22, &full[sl], xb, ya, zi);
          tma_load_3d(db + YB, &m.b22, &full[sl], xa, yb, zi);
          tma_load_3d(db + YB + XB, &m.b22, &full[sl], xb, yb, zi);
        } else {
          mbar_expect_tx(&full[sl], 2u * 2u * NW * BH * (uint32_t)sizeof(double));
          tma_load_3d(da, &m.a, &full[sl], xa, ya, zi);
          tma_load_3d(da + NYB, &m.a, &full[sl], xa, yb, zi);
          tma_load_3d(db, &m.b, &full[sl], xa, ya, zi);
          tma_load_3d(db + NYB, &m.b, &full[sl], xa, yb, zi);
        }
      }
    };
    // periodic fix-up of plane q (ragged / small grids only): every cell of rows/cols 1..38
    // outside the grid (no TMA: every cell) re-read with wrapped indices
    auto fix = [&](int q) {
      const int sl = q % RING;
      if (tma) mbar_wait(&full[sl], (uint32_t)((q / RING) & 1));
      else wait_empty(q);
      double* ra = ringA + sl * WS;
      double* rb = ringB + sl * WS;
      const size_t zo = plane * (size_t)zof(q);
#pragma unroll 4
      for (int i = lane; i < 38 * 38; i += 32) {
        const int r = 1 + i / 38, c = 1 + i % 38;
        const int x = gx0 + c, y = gy0 + r;
        if (!tma || x < 0 || x >= nx || y < 0 || y >= ny) {
          const size_t g = (size_t)wrapi(x, nx) + (size_t)nx * wrapi(y, ny) + zo;
          ra[woff_nat(r, c)] = p.a[g];
          rb[woff_nat(r, c)] = p.b[g];
        }
      }
      if (tma) fence_proxy_async();   // generic writes before a later TMA overwrite
      __syncwarp();
      if (lane == 0) mbar_arrive(&fixd[sl]);
    };
    if (tma)
      for (int q = 0; q < PF && q < Tp; ++q) issue(q);
    if (!edge) {
      for (int q = PF; q < Tp; ++q) issue(q);
    } else if (!tma) {
      for (int q = 0; q < Tp; ++q) fix(q);
    } else {
      fix(0);
      for (int t = 0; t < Tp; ++t) {
        if (t + PF < Tp) issue(t + PF);
        if (t + 1 < Tp) fix(t + 1);
      }
    }
  } else {
    // ================= compute warps =================
    // this thread's block (pair column pc, strip sr) of the halo-2 region
    const bool valid = tid < NBLK;
    const int bi = valid ? tid : 0;
    const int pc = 1 + bi % NPB, sr = 1 + bi / NPB;
    const boff bo{woff(split, 2 * sr, 2 * pc), woff(split, 2 * sr, 2 * pc - 1),
                  woff(split, 2 * sr, 2 * pc + 2), woff(split, 2 * sr - 1, 2 * pc),
                  woff(split, 2 * sr + 2, 2 * pc), split ? BW : NW};
    const int e0 = 2 * sr * SP + pc;          // split offset of the block's point a
    // resid: s = Phi + psi of one outer-ring cell of the window (rows / cols 1 and 38, which no
    // block owns) per thread tid < 148, written with the block values into the s plane
    int rc_q = 0, rc_e = -1;
    if (OP == OP_RESID && tid < 2 * 38 + 2 * 36) {
      int rr, cc;
      if (tid < 76) { rr = tid < 38 ? 1 : 38; cc = 1 + tid % 38; }
      else { const int k = tid - 76; cc = k < 36 ? 1 : 38; rr = 2 + k % 36; }
      rc_q = woff(split, rr, cc);
      rc_e = ((cc & 1) ? SO : 0) + rr * SP + (cc >> 1);
    }
    const int xg = gx0 + 2 * pc, yg = gy0 + 2 * sr;   // global coords of point a (unwrapped)
    // outputs: pair columns / strips 2..17 inside the (possibly ragged) grid; a pair never
    // straddles the seam (x, y0 even)
    const bool outblk = valid && pc >= 2 && pc <= 17 && sr >= 2 && sr <= 17;
    const bool o_a = outblk && xg < nx && yg < ny, o_b = outblk && xg + 1 < nx && yg < ny;
    const bool o_c = outblk && xg < nx && yg + 1 < ny, o_d = outblk && xg + 1 < nx && yg + 1 < ny;
    const size_t g0 = (size_t)wrapi(xg, nx) + (size_t)nx * wrapi(yg, ny);
    const size_t g1 = (size_t)wrapi(xg, nx) + (size_t)nx * wrapi(yg + 1, ny);
    const bool vec0 = o_a && o_b && (nx % 2 == 0) && ((reinterpret_cast<uintptr_t>(p.out + g0) & 15u) == 0);
    const bool vec1 = o_c && o_d && (nx % 2 == 0) && ((reinterpret_cast<uintptr_t>(p.out + g1) & 15u) == 0);
    uint64_t* wbar = edge ? fixd : full;      // plane ready: fixed up (edge tiles) or landed

    int slot = 0;
    uint32_t phase = 0;
    const q4 Z{0, 0, 0, 0};
    // queues (period 3):  A1,A2 = Phi|v at t-1,t-2;  B1,B2 = psi|c at t-1,t-2;
    // L2,L3 = Lt at t-2,t-3;  M3,M4 = A|B at t-3,t-4;  P2,P3 = (Phi-psi)/dt | v/dt at t-2,t-3
    q4 A1 = Z, A2 = Z, B1 = Z, B2 = Z, L2 = Z, L3 = Z, M3 = Z, M4 = Z, P2 = Z, P3 = Z;
    double* out0 = p.out + plane * (size_t)z0 + g0;
    const ptrdiff_t d1 = (ptrdiff_t)g1 - (ptrdiff_t)g0;

#pragma unroll 3
    for (int t = 0; t < Tp; ++t) {
      const double* ra = ringA + slot * WS;
      const double* rb = ringB + slot * WS;
      const int prv = slot == 0 ? RING - 1 : slot - 1;   // ring slot of plane t-1
      const double* Lr = Lsp + ((t - 2) & 1) * SPLANE;   // Lt at t-2
      const double* Mr = Bsp + ((t - 3) & 1) * SPLANE;   // A|B at t-3
      double* Lw = Lsp + ((t - 1) & 1) * SPLANE;
      double* Mw = Bsp + ((t - 2) & 1) * SPLANE;
      mbar_wait(&wbar[slot], phase);

      q4 A0, B0;   // own inputs of plane t
      {
        const double2 a0 = lds2(ra + bo.own), a1 = lds2(ra + bo.own + bo.pitch);
        const double2 b0 = lds2(rb + bo.own), b1 = lds2(rb + bo.own + bo.pitch);
        A0 = {a0.x, a0.y, a1.x, a1.y};
        B0 = {b0.x, b0.y, b1.x, b1.y};
      }
      q4 Pnew;     // pointwise part of the output at plane t-1
      if (OP == OP_RESID)
        Pnew = {(A1.a - B1.a) * idt, (A1.b - B1.b) * idt, (A1.c - B1.c) * idt,
                (A1.d - B1.d) * idt};
      else
        Pnew = {A1.a * idt, A1.b * idt, A1.c * idt, A1.d * idt};
      // everything that needs no outside neighbour, while other warps finish iteration t-1:
      // the centre and z parts of the three Laplacians and the pointwise part of A|B
      const q4 c1 = (OP == OP_RESID) ? lap_own(add4(A1, B1), add4(A2, B2), add4(A0, B0))
                                     : lap_own(A1, A2, A0);
      double srng = 0.0;   // resid: s at this thread's outer-ring cell of plane t
      if (OP == OP_RESID && rc_e >= 0) srng = ra[rc_q] + rb[rc_q];
      const q4 c2 = lap_own(L2, L3), c3 = lap_own(M3, M4);
      q4 r2;       // pointwise part of A|B at t-2 plus ih2 Lt at t-2
      {
        q4 base;
        if (OP == OP_RESID) {   // (1-gamma)/2 s + N,  N = s (Phi^2 + psi^2) / 4
          auto nb = [&](double ph, double ps) {
            const double s = ph + ps;
            return s * fma(0.25, fma(ph, ph, ps * ps), p.k0);
          };
          base = {nb(A2.a, B2.a), nb(A2.b, B2.b), nb(A2.c, B2.c), nb(A2.d, B2.d)};
        } else {                // ((1-gamma)/2 + c) v
          base = {(p.k0 + B2.a) * A2.a, (p.k0 + B2.b) * A2.b, (p.k0 + B2.c) * A2.c,
                  (p.k0 + B2.d) * A2.d};
        }
        r2 = {fma(p.k1, L2.a, base.a), fma(p.k1, L2.b, base.b), fma(p.k1, L2.c, base.c),
              fma(p.k1, L2.d, base.d)};
      }
      // ---- every compute warp has finished iteration t-1 (its reads and its plane stores)
      if (t > 0) mbar_wait(&itbar, (uint32_t)((t - 1) & 1));
      // outside neighbours of the planes produced in iteration t-1 (all loads before any store)
      q4 x1;
      if constexpr (OP == OP_RESID) {
#if ST3_RES_SHFL
        // left / right neighbours of s = Phi + psi at plane t-1 from the adjacent lanes'
        // registers (the same sums the s plane holds), top / bottom from the s plane
        const double* S = Ssp + ((t - 1) & 1) * SPLANE;
        // (recomputed here by opaque adds: sharing them with c1's sums would keep four more
        // doubles live across the iteration barrier, which spills at the 168-register cap)
        double sa, sb, sc, sd;
        asm volatile("add.f64 %0, %1, %2;" : "=d"(sa) : "d"(A1.a), "d"(B1.a));
        asm volatile("add.f64 %0, %1, %2;" : "=d"(sb) : "d"(A1.b), "d"(B1.b));
        asm volatile("add.f64 %0, %1, %2;" : "=d"(sc) : "d"(A1.c), "d"(B1.c));
        asm volatile("add.f64 %0, %1, %2;" : "=d"(sd) : "d"(A1.d), "d"(B1.d));
        double L0 = __shfl_up_sync(0xffffffffu, sb, 1);
        double L1 = __shfl_up_sync(0xffffffffu, sd, 1);
        double R0 = __shfl_down_sync(0xffffffffu, sa, 1);
        double R1 = __shfl_down_sync(0xffffffffu, sc, 1);
        if (!(pc > 1 && lane > 0)) {
          L0 = S[SO + e0 - 1];
          L1 = S[SO + e0 + SP - 1];
        }
        if (!(pc < NPB && lane < 31)) {
          R0 = S[e0 + 1];
          R1 = S[e0 + SP + 1];
        }
        const double Ta = S[e0 - SP], Tb = S[SO + e0 - SP];
        const double Da = S[e0 + 2 * SP], Db = S[SO + e0 + 2 * SP];
        x1 = {L0 + Ta, R0 + Tb, L1 + Da, R1 + Db};
#else
        x1 = out_split(Ssp + ((t - 1) & 1) * SPLANE, e0);
#endif
      } else {
        // left / right neighbours of the block are the adjacent lanes' own plane-(t-1) values
        // (shuffles; the stride-2 ring loads were 2-way bank conflicts), from the ring only at
        // the region edge and across warps; top / bottom pairs from the ring
        const double* f = ringA + prv * WS;
        const double lb = __shfl_up_sync(0xffffffffu, A1.b, 1);
        const double ld = __shfl_up_sync(0xffffffffu, A1.d, 1);
        const double ra = __shfl_down_sync(0xffffffffu, A1.a, 1);
        const double rc = __shfl_down_sync(0xffffffffu, A1.c, 1);
        double L0 = lb, L1 = ld, R0 = ra, R1 = rc;
        if (!(pc > 1 && lane > 0)) {   // (predicated: only these lanes touch shared memory)
          L0 = f[bo.l];
          L1 = f[bo.l + bo.pitch];
        }
        if (!(pc < NPB && lane < 31)) {
          R0 = f[bo.r];
          R1 = f[bo.r + bo.pitch];
        }
        const double2 T = lds2(f + bo.t), D = lds2(f + bo.d);
        x1 = {L0 + T.x, R0 + T.y, L1 + D.x, R1 + D.y};
      }
      const q4 x2 = out_split(Lr, e0);
      const q4 x3 = out_split(Mr, e0);
      // ---- stage 1: Lt s | Lt v at plane t-1
      const q4 Lnew = add4(c1, x1);
      // ---- stage 2: A | B at plane t-2  (z+ neighbour of Lt: the new plane t-1)
      const q4 LL = add4(add4(c2, x2), Lnew);
      const q4 Mnew = {fma(p.k2, LL.a, r2.a), fma(p.k2, LL.b, r2.b), fma(p.k2, LL.c, r2.c),
                       fma(p.k2, LL.d, r2.d)};
      // ---- stage 3: F | Jv at plane t-3
      const q4 LM = add4(add4(c3, x3), Mnew);
      const double oa = fma(p.kout, LM.a, P3.a), ob = fma(p.kout, LM.b, P3.b);
      const double oc = fma(p.kout, LM.c, P3.c), od = fma(p.kout, LM.d, P3.d);
      // ---- plane stores, then this warp's arrivals: iteration done, plane t-1 released
      if (valid) {
        st_split(Lw, e0, Lnew);
        st_split(Mw, e0, Mnew);
        if (OP == OP_RESID) st_split(Ssp + (t & 1) * SPLANE, e0, add4(A0, B0));
      }
      if (OP == OP_RESID && rc_e >= 0) Ssp[(t & 1) * SPLANE + rc_e] = srng;
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&itbar);
        if (LAG == 0) mbar_arrive(&empty[slot]);
        else if (t > 0) mbar_arrive(&empty[prv]);
      }
      // ---- queue rotation (renames under the 3x unroll)
      A2 = A1; A1 = A0; B2 = B1; B1 = B0;
      L3 = L2; L2 = Lnew;
      M4 = M3; M3 = Mnew;
      P3 = P2; P2 = Pnew;
      if (t >= 6 && t - 6 < zc) {
        double* o = out0 + plane * (size_t)(t - 6);
        if (vec0) {
          stg2(o, oa, ob);
          nrm += oa * oa + ob * ob;
        } else {
          if (o_a) { o[0] = oa; nrm += oa * oa; }
          if (o_b) { o[1] = ob; nrm += ob * ob; }
        }
        if (vec1) {
          stg2(o + d1, oc, od);
          nrm += oc * oc + od * od;
        } else {
          if (o_c) { o[d1] = oc; nrm += oc * oc; }
          if (o_d) { o[d1 + 1] = od; nrm += od * od; }
        }
      }
      slot = slot + 1 == RING ? 0 : slot + 1;
      phase ^= (slot == 0) ? 1u : 0u;
    }
  }
  if (p.partials) {   // all 12 warps (the producer contributes 0)
    const double sblk = block_sum(nrm, red);
    if (tid == 0) p.partials[blockIdx.y * gridDim.x + blockIdx.x] = sblk;
  }
}

// Work plan: the first n1 tiles are streamed as whole z-columns (one item each, 6 halo planes
// per 512 instead of per chunk), the other tiles in nzc chunks, launched chunk by chunk with the
// tile index fastest, so the CTAs resident at any time march neighbouring tiles through the same
// planes (their halos hit in L2).  n1 is 0 or a multiple of the SM count (a full wave of
// columns); the plan minimising the makespan of in-order list scheduling on nsm SMs wins
// (cost of an item = its streamed planes, padded to the unroll factor).
struct Plan3 { int n1, nzc, zc, nitems; long makespan; };
Plan3 choose_plan(int ntiles, int nz, int nsm, bool two_phase) {
  auto makespan = [&](int n1, int nzc, int zc) {
    std::priority_queue<long, std::vector<long>, std::greater<long>> fin;   // SM finish times
    for (int i = 0; i < nsm; ++i) fin.push(0);
    long m = 0;
    auto put = [&](int planes) {
      const long f = fin.top() + (planes + 6 + 2) / 3 * 3;
      fin.pop();
      fin.push(f);
      m = std::max(m, f);
    };
    for (int i = 0; i < n1; ++i) put(nz);
    for (int c = 0; c < nzc; ++c)
      for (int i = n1; i < ntiles; ++i) put(std::min(zc, nz - c * zc));
    return m;
  };
  Plan3 best{0, 1, nz, ntiles, 0};
  long best_cost = -1;
  for (int n1 = 0; n1 <= ntiles; n1 += nsm) {
    for (int nzc = 1; nzc <= nz && nzc <= 64; ++nzc) {
      const int zc = (nz + nzc - 1) / nzc;
      if ((nz + zc - 1) / zc != nzc) continue;
      if (n1 == ntiles && nzc > 1) break;
      const long cost = makespan(n1, nzc, zc);
      if (best_cost < 0 || cost < best_cost) {
        best_cost = cost;
        best = {n1, nzc, zc, n1 + (ntiles - n1) * nzc, cost};
      }
    }
    if (!two_phase) break;
  }
  return best;
}

template <int OP>
cudaError_t launch3d(pfc_ctx* ctx, const double* a, const double* b, double dt, double* out,
                     double* partials, int* nparts) {
  static bool attr_set = false;
  static int nsm = 148;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(stencil3d_kernel<OP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem_bytes<OP>());
    if (e != cudaSuccess) return e;
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      nsm = v;
    attr_set = true;
  }
  const int nx = ctx->cfg.n[0], ny = ctx->cfg.n[1], nz = ctx->cfg.n[2];
  const int ntiles = ((nx + TX - 1) / TX) * ((ny + TY - 1) / TY);
  static Plan3 plan{-1, 0, 0, 0, 0};
  static int plan_key[3] = {0, 0, 0};
  if (plan.n1 < 0 || plan_key[0] != ntiles || plan_key[1] != nz || plan_key[2] != nsm) {
    plan = choose_plan(ntiles, nz, nsm, OP == OP_JV && ST3_TWO_PHASE);
    plan_key[0] = ntiles; plan_key[1] = nz; plan_key[2] = nsm;
  }
  const int zc = plan.zc;
  const double ih2 = ctx->ih2;
  S3Args p{a, b, out, partials, nx, ny, nz, zc, 1.0 / dt, 0.5 * (1.0 - ctx->cfg.gamma), ih2,
           0.5 * ih2 * ih2, -ih2, 0, OP == OP_JV ? ctx->gate : nullptr};
  p.n1 = plan.n1;
  p.ntiles = ntiles;
  p.dtp = ctx->dtdev;
  S3Maps m;
  memset(&m, 0, sizeof(m));
  const int box[3] = {NW, BH, 1}, box22[3] = {BW, BH, 1};
  // TMA: 16-B aligned rows and base; a box must fit the grid
  if (nx % 2 == 0 && nx >= NW && ny >= BH && tma_usable(a) && tma_usable(b) &&
      tma_encode(&m.a, a, 3, ctx->cfg.n, box) && tma_encode(&m.b, b, 3, ctx->cfg.n, box) &&
      tma_encode(&m.a22, a, 3, ctx->cfg.n, box22) && tma_encode(&m.b22, b, 3, ctx->cfg.n, box22))
    p.mode = (nx % TX == 0 && ny % TY == 0) ? 2 : 1;
  const dim3 grid = OP == OP_JV ? dim3(plan.nitems) : dim3(ntiles, plan.nzc);
  if (nparts) *nparts = plan.nitems;
  stencil3d_kernel<OP><<<grid, NT, smem_bytes<OP>(), ctx->stream>>>(m, p);
  ctx->launches++;
  pfc_account(ctx, OP == OP_RESID ? PFC_K_RESIDUAL : PFC_K_JV, 24.0 * ctx->N,
              (OP == OP_RESID ? 42.0 : 31.0) * ctx->N);
  return cudaGetLastError();
}

}  // namespace

pfc_status pfc_plan_stencil3d(int ntiles, int nz, int nsm, int two_phase, long long plan[5]) {
  if (ntiles < 1 || nz < 1 || nsm < 1 || !plan) return PFC_EINVAL;
  const Plan3 pl = choose_plan(ntiles, nz, nsm, two_phase != 0);
  plan[0] = pl.n1; plan[1] = pl.nzc; plan[2] = pl.zc; plan[3] = pl.nitems; plan[4] = pl.makespan;
  return PFC_OK;
}

cudaError_t launch_residual_3d(pfc_ctx* ctx, const double* phi_new, const double* phi_old,
                               double dt, double* F, double* partials, int* nparts) {
  return launch3d<OP_RESID>(ctx, phi_new, phi_old, dt, F, partials, nparts);
}

cudaError_t launch_jv_3d(pfc_ctx* ctx, const double* v, const double* c, double dt,
                         double* out) {
  return launch3d<OP_JV>(ctx, v, c, dt, out, nullptr, nullptr);
}
