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
// z0-3 .. z0+zc+2 stream through a RING-slot ring per field (one 42 x 40 TMA box per field and
// plane, cp.async.bulk.tensor.3d, PF planes in flight).  Warp specialisation:
//  * the producer warp issues every TMA load and makes the periodic wrap: TMA zero-fills
//    out-of-range cells and has no wrap mode, so edge tiles also load small x-strip, y-strip and
//    corner boxes at the wrapped coordinates into a staging area and the producer copies those
//    cells into the window (ragged grids: wrapped global re-reads; no-TMA grids: every cell);
//    full / fixd / empty mbarriers per slot order TMA -> wrap -> compute -> re-fill;
//  * compute thread i < 324 owns the 2 x 2 point block (pair column p, row strip s), p, s in
//    1..18, of the window, i.e. the halo-2 region; at streamed plane t it computes
//        Lt s|v (t-1)  ->  A|B (t-2)  ->  F|Jv (t-3)
//    with z-neighbours, block-internal neighbours and the block's own values in registers (every
//    queue has period 3, so the 3x-unrolled loop rotates it by register renaming) and only the
//    block's 8 outside neighbours read from shared memory.  The intermediate planes Lt and A|B
//    are kept in an even/odd-column split layout with a row pitch of 25 doubles, which makes
//    every shared access of a warp conflict-free; the input window uses a row pitch of 42 for the
//    same reason.  Each stage reads planes written in the previous iteration: a split-phase
//    mbarrier (arrive after the plane stores, wait before the neighbour loads) separates
//    iterations, and the neighbour-free parts of the three Laplacians are computed before the
//    wait.  Optional fused ||F||^2 partial per CTA.
#include "pfc_device.cuh"
#include "pfc_internal.h"

namespace {

constexpr int TX = 32, TY = 32;
constexpr int WX = 42, WY = 40;     // window: cols x0-4 .. x0+37, rows y0-4 .. y0+35
constexpr int WS = WX * WY;         // doubles per ring slot (13440 B, a multiple of 128)
constexpr int NPB = 18;             // stage region: pair columns 1..18 x strips 1..18
constexpr int NBLK = NPB * NPB;     // 324 blocks
constexpr int NTC = 352;            // 11 compute warps (324 blocks)
constexpr int NWC = NTC / 32;
constexpr int NT = NTC + 32;        // + 1 producer warp (TMA issue, periodic wrap)
#ifndef ST3_RING                    // diagnostic builds may override the ring depth
#define ST3_RING 5
#define ST3_PF 3
#endif
constexpr int RING = ST3_RING, PF = ST3_PF;   // PF <= RING - 2: re-fill after the last reader
constexpr int SP = 25;              // split-plane row pitch (doubles)
constexpr int SROWS = WY;
constexpr int SO = SROWS * SP;      // offset of the odd-column half
constexpr int SPLANE = 2 * SO;      // doubles per split plane
// wrap staging (mode 2): per field and slot an x-strip box 4 x 40, a y-strip box 42 x 4 (padded
// to 176 for 128-B aligned TMA destinations) and a corner box 4 x 4
constexpr int XS_N = 4 * WY, YS_N = WX * 4, YS_PAD = 176, CS_N = 16;
constexpr int STG = XS_N + YS_PAD + CS_N;   // 352 doubles per field and slot
constexpr int SMEM_BYTES = (2 * RING * WS + 4 * SPLANE + 2 * RING * STG) * (int)sizeof(double);

enum { OP_RESID = 0, OP_JV = 1 };

struct S3Args {
  const double* a;   // Phi | v
  const double* b;   // psi | c
  double* out;
  double* partials;
  int nx, ny, nz;
  int zc;            // planes per chunk
  double idt, k0, k1, k2, kout;   // (1-gamma)/2, ih2, ih2^2/2, -ih2
  int mode;          // 0: plain loads; 1: TMA + wrapped global re-reads; 2: TMA + staged wrap
  const int* gate;   // device-resident FGMRES: skip the launch when *gate != 0 (f1)
};

struct q4 { double a, b, c, d; };   // (row0,col0) (row0,col1) (row1,col0) (row1,col1)

__device__ __forceinline__ double2 lds2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}
__device__ __forceinline__ void stg2(double* p, double x, double y) {
  *reinterpret_cast<double2*>(p) = make_double2(x, y);
}

// sums of the outside xy neighbours of the block, natural (ring) layout, qa = row-0 offset
__device__ __forceinline__ q4 out_ring(const double* f, int qa) {
  const double L0 = f[qa - 1], R0 = f[qa + 2], L1 = f[qa + WX - 1], R1 = f[qa + WX + 2];
  const double2 T = lds2(f + qa - WX), D = lds2(f + qa + 2 * WX);
  return {L0 + T.x, R0 + T.y, L1 + D.x, R1 + D.y};
}
// same for Phi + psi from both rings (resid stage 1)
__device__ __forceinline__ q4 out_ring2(const double* f, const double* g, int qa) {
  const double L0 = f[qa - 1] + g[qa - 1], R0 = f[qa + 2] + g[qa + 2];
  const double L1 = f[qa + WX - 1] + g[qa + WX - 1], R1 = f[qa + WX + 2] + g[qa + WX + 2];
  const double2 T = lds2(f + qa - WX), D = lds2(f + qa + 2 * WX);
  const double2 Tg = lds2(g + qa - WX), Dg = lds2(g + qa + 2 * WX);
  return {L0 + (T.x + Tg.x), R0 + (T.y + Tg.y), L1 + (D.x + Dg.x), R1 + (D.y + Dg.y)};
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

struct S3Maps {   // main window box, x-strip, y-strip and corner boxes, per field
  CUtensorMap a, b, xa, xb, ya, yb, ca, cb;
};

template <int OP>
__global__ void __launch_bounds__(NT, 1) stencil3d_kernel(const __grid_constant__ S3Maps m,
                                                          const __grid_constant__ S3Args p) {
  extern __shared__ __align__(128) double smem_dyn[];
  double* ringA = smem_dyn;                 // RING slots: Phi | v
  double* ringB = ringA + RING * WS;        // RING slots: psi | c
  double* Lsp = ringB + RING * WS;          // 2 split planes: Lt s | Lt v
  double* Bsp = Lsp + 2 * SPLANE;           // 2 split planes: A | B
  double* stg = Bsp + 2 * SPLANE;           // RING x (field a, field b) wrap staging
  __shared__ uint64_t full[RING];   // the slot's TMA boxes landed (transaction bytes)
  __shared__ uint64_t fixd[RING];   // the producer finished the periodic wrap of the slot
  __shared__ uint64_t empty[RING];  // every compute warp finished reading the slot
  __shared__ uint64_t itbar;        // compute warps: split-phase iteration barrier
  __shared__ double red[64];

  if (p.gate && *p.gate) return;
  const int tid = threadIdx.x, lane = tid & 31;
  const int nx = p.nx, ny = p.ny, nz = p.nz;
  const int ntx = (nx + TX - 1) / TX;
  const int x0 = (blockIdx.x % ntx) * TX, y0 = (blockIdx.x / ntx) * TY;
  const int z0 = blockIdx.y * p.zc;
  const int zc = min(p.zc, nz - z0);
  const int gx0 = x0 - 4, gy0 = y0 - 4;     // global coordinates of window cell (0,0)
  const size_t plane = (size_t)nx * ny;
  const int T = zc + 6;
  const int Tp = (T + 2) / 3 * 3;           // padded to the unroll factor; extra planes are inert
  const bool tma = p.mode != 0, staged = p.mode == 2;
  // does a window cell the stencil reads (rows and cols 1..38) lie outside the grid?
#ifdef ST3_NOEDGE   // diagnostic timing build: no periodic wrap at all (wrong edge values)
  const bool edge = false;
#else
  const bool edge = !tma || x0 < 3 || y0 < 3 || x0 + 34 >= nx || y0 + 34 >= ny;
#endif

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
    // ================= producer warp: TMA issue and periodic wrap of every plane =================
    const bool xl = x0 == 0, xr = x0 + TX >= nx, yt = y0 == 0, yb = y0 + TY >= ny;
    const bool xe = edge && staged && (xl || xr), ye = edge && staged && (yt || yb);
    const int xs = xl ? nx - 4 : 0, cb0 = xl ? 0 : 36;   // strip origins: global x, window col
    const int ys = yt ? ny - 4 : 0, rb0 = yt ? 0 : 36;
    const uint32_t tx_bytes = 2u * sizeof(double) *
        (WS + (xe ? XS_N : 0) + (ye ? YS_N : 0) + (xe && ye ? CS_N : 0));
    auto zof = [&](int q) { return wrapi(z0 - 3 + q, nz); };
    auto wait_empty = [&](int q) {   // plane q - RING released by every compute warp
      if (q >= RING) mbar_wait(&empty[q % RING], (uint32_t)((q / RING - 1) & 1));
    };
    auto issue = [&](int q) {
      const int sl = q % RING, zi = zof(q);
      wait_empty(q);
      if (lane == 0) {
        mbar_expect_tx(&full[sl], tx_bytes);
        tma_load_3d(ringA + sl * WS, &m.a, &full[sl], gx0, gy0, zi);
        tma_load_3d(ringB + sl * WS, &m.b, &full[sl], gx0, gy0, zi);
        double* sa = stg + sl * 2 * STG;
        double* sb = sa + STG;
        if (xe) {
          tma_load_3d(sa, &m.xa, &full[sl], xs, gy0, zi);
          tma_load_3d(sb, &m.xb, &full[sl], xs, gy0, zi);
        }
        if (ye) {
          tma_load_3d(sa + XS_N, &m.ya, &full[sl], gx0, ys, zi);
          tma_load_3d(sb + XS_N, &m.yb, &full[sl], gx0, ys, zi);
        }
        if (xe && ye) {
          tma_load_3d(sa + XS_N + YS_PAD, &m.ca, &full[sl], xs, ys, zi);
          tma_load_3d(sb + XS_N + YS_PAD, &m.cb, &full[sl], xs, ys, zi);
        }
      }
    };
    // periodic wrap of plane q: every cell of rows/cols 1..38 outside the grid.  Mode 2: copied
    // from the slot's staging boxes, (window, staging) offsets precomputed per lane (<= 7 cells:
    // at most 3 x 38 + 3 x 35 = 219 per tile); mode 1: re-read with wrapped indices; mode 0:
    // every cell re-read (the last two only on ragged or small grids)
    constexpr int MAXC = 7;
    int cdst[MAXC], csrc[MAXC];
    {
      const int nxc = xe ? 3 : 0, nyr = ye ? 3 : 0, w = 38 - nxc;
      const int cnt = nxc * 38 + nyr * w;
#pragma unroll
      for (int k = 0; k < MAXC; ++k) {
        const int i = lane + 32 * k;
        int r = 0, c = 0;
        if (i < nxc * 38) { r = 1 + i / nxc; c = (xl ? 1 : 36) + i % nxc; }
        else if (i < cnt) {
          const int j = i - nxc * 38;
          r = (yt ? 1 : 36) + j / w;
          c = (xe && xl ? 4 : 1) + j % w;
        }
        const bool ix = xe && (xl ? c < 4 : c >= 36), iy = ye && (yt ? r < 4 : r >= 36);
        cdst[k] = i < cnt ? r * WX + c : -1;
        csrc[k] = (ix && iy) ? XS_N + YS_PAD + (r - rb0) * 4 + (c - cb0)
                  : ix ? r * 4 + (c - cb0) : XS_N + (r - rb0) * WX + c;
      }
    }
    auto fix_body = [&](int q) {
      const int sl = q % RING;
      double* ra = ringA + sl * WS;
      double* rb = ringB + sl * WS;
      if (staged) {
        const double* sa = stg + sl * 2 * STG;
        const double* sb = sa + STG;
        double va[MAXC], vb[MAXC];
#pragma unroll
        for (int k = 0; k < MAXC; ++k)
          if (cdst[k] >= 0) { va[k] = sa[csrc[k]]; vb[k] = sb[csrc[k]]; }
#pragma unroll
        for (int k = 0; k < MAXC; ++k)
          if (cdst[k] >= 0) { ra[cdst[k]] = va[k]; rb[cdst[k]] = vb[k]; }
      } else {
        const size_t zo = plane * (size_t)zof(q);
#pragma unroll 4
        for (int i = lane; i < 38 * 38; i += 32) {
          const int r = 1 + i / 38, c = 1 + i % 38;
          const int x = gx0 + c, y = gy0 + r;
          if (!tma || x < 0 || x >= nx || y < 0 || y >= ny) {
            const size_t g = (size_t)wrapi(x, nx) + (size_t)nx * wrapi(y, ny) + zo;
            ra[r * WX + c] = p.a[g];
            rb[r * WX + c] = p.b[g];
          }
        }
      }
      if (tma) fence_proxy_async();   // generic writes before a later TMA overwrite
      __syncwarp();
      if (lane == 0) mbar_arrive(&fixd[sl]);
    };
    auto fix = [&](int q) {   // blocking
      if (tma) mbar_wait(&full[q % RING], (uint32_t)((q / RING) & 1));
      else wait_empty(q);
      fix_body(q);
    };
    if (tma)
      for (int q = 0; q < PF && q < Tp; ++q) issue(q);
    if (!edge) {
      for (int q = PF; q < Tp; ++q) issue(q);
    } else if (!tma) {
      for (int q = 0; q < Tp; ++q) fix(q);
    } else {
      // issue and wrap decoupled: whichever is ready first (never block the TMA pipeline
      // behind a plane that has not landed yet)
      fix(0);
      int qi = PF, qf = 1;
      while (qi < Tp || qf < Tp) {
        if (qi < Tp && (qi < RING || mbar_test(&empty[qi % RING], (uint32_t)((qi / RING - 1) & 1)))) {
          issue(qi);
          ++qi;
        } else if (qf < qi && qf < Tp && mbar_test(&full[qf % RING], (uint32_t)((qf / RING) & 1))) {
          fix_body(qf);
          ++qf;
        } else {
          __nanosleep(64);
        }
      }
    }
  } else {
    // ================= compute warps =================
    // this thread's block (pair column pc, strip sr) of the halo-2 region
    const bool valid = tid < NBLK;
    const int bi = valid ? tid : 0;
    const int pc = 1 + bi % NPB, sr = 1 + bi / NPB;
    const int qa = 2 * sr * WX + 2 * pc;      // ring offset of (row 2sr, col 2pc)
    const int e0 = 2 * sr * SP + pc;          // split offset of the same point
    const int xa = gx0 + 2 * pc, ya = gy0 + 2 * sr;   // global coords of point a
    // outputs: pair columns / strips 2..17 inside the (possibly ragged) grid
    const bool outblk = valid && pc >= 2 && pc <= 17 && sr >= 2 && sr <= 17;
    const bool o_a = outblk && xa < nx && ya < ny, o_b = outblk && xa + 1 < nx && ya < ny;
    const bool o_c = outblk && xa < nx && ya + 1 < ny, o_d = outblk && xa + 1 < nx && ya + 1 < ny;
    const size_t ga = (size_t)xa + (size_t)nx * ya;   // meaningful only for output points
    const bool vec0 = o_a && o_b && (nx % 2 == 0) && ((reinterpret_cast<uintptr_t>(p.out + ga) & 15u) == 0);
    const bool vec1 = o_c && o_d && (nx % 2 == 0) &&
                      ((reinterpret_cast<uintptr_t>(p.out + ga + nx) & 15u) == 0);
    uint64_t* wbar = edge ? fixd : full;      // plane ready: wrapped (edge tiles) or just landed

    int slot = 0;
    uint32_t phase = 0;
    const q4 Z{0, 0, 0, 0};
    // queues (period 3):  A1,A2 = Phi|v at t-1,t-2;  B1,B2 = psi|c at t-1,t-2;
    // L2,L3 = Lt at t-2,t-3;  M3,M4 = A|B at t-3,t-4;  P2,P3 = (Phi-psi)/dt | v/dt at t-2,t-3
    q4 A1 = Z, A2 = Z, B1 = Z, B2 = Z, L2 = Z, L3 = Z, M3 = Z, M4 = Z, P2 = Z, P3 = Z;
    double* outp = p.out + plane * (size_t)z0 + ga;

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
        const double2 a0 = lds2(ra + qa), a1 = lds2(ra + qa + WX);
        const double2 b0 = lds2(rb + qa), b1 = lds2(rb + qa + WX);
        A0 = {a0.x, a0.y, a1.x, a1.y};
        B0 = {b0.x, b0.y, b1.x, b1.y};
      }
      q4 Pnew;     // pointwise part of the output at plane t-1
      if (OP == OP_RESID)
        Pnew = {(A1.a - B1.a) * p.idt, (A1.b - B1.b) * p.idt, (A1.c - B1.c) * p.idt,
                (A1.d - B1.d) * p.idt};
      else
        Pnew = {A1.a * p.idt, A1.b * p.idt, A1.c * p.idt, A1.d * p.idt};
      // everything that needs no outside neighbour, while other warps finish iteration t-1:
      // the centre and z parts of the three Laplacians and the pointwise part of A|B
      const q4 c1 = (OP == OP_RESID) ? lap_own(add4(A1, B1), add4(A2, B2), add4(A0, B0))
                                     : lap_own(A1, A2, A0);
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
      const q4 x1 = (OP == OP_RESID) ? out_ring2(ringA + prv * WS, ringB + prv * WS, qa)
                                     : out_ring(ringA + prv * WS, qa);
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
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&itbar);
        if (t > 0) mbar_arrive(&empty[prv]);
      }
      // ---- queue rotation (renames under the 3x unroll)
      A2 = A1; A1 = A0; B2 = B1; B1 = B0;
      L3 = L2; L2 = Lnew;
      M4 = M3; M3 = Mnew;
      P3 = P2; P2 = Pnew;
      if (t >= 6 && t - 6 < zc) {
        double* o = outp + plane * (size_t)(t - 6);
        if (vec0) {
          stg2(o, oa, ob);
          nrm += oa * oa + ob * ob;
        } else {
          if (o_a) { o[0] = oa; nrm += oa * oa; }
          if (o_b) { o[1] = ob; nrm += ob * ob; }
        }
        if (vec1) {
          stg2(o + nx, oc, od);
          nrm += oc * oc + od * od;
        } else {
          if (o_c) { o[nx] = oc; nrm += oc * oc; }
          if (o_d) { o[nx + 1] = od; nrm += od * od; }
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

// z chunking: minimise (waves of resident CTAs) x (planes streamed per CTA)
int choose_chunks(int ntiles, int nz, int nsm) {
  int best = 1;
  double best_cost = 1e300;
  for (int nzc = 1; nzc <= nz && nzc <= 256; ++nzc) {
    const int zc = (nz + nzc - 1) / nzc;
    if ((nz + zc - 1) / zc != nzc) continue;
    const double waves = (double)((ntiles * nzc + nsm - 1) / nsm);
    const double cost = waves * (zc + 6);
    if (cost < best_cost - 1e-9) { best_cost = cost; best = nzc; }
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
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      nsm = v;
    attr_set = true;
  }
  const int nx = ctx->cfg.n[0], ny = ctx->cfg.n[1], nz = ctx->cfg.n[2];
  const int ntiles = ((nx + TX - 1) / TX) * ((ny + TY - 1) / TY);
  const int nzc = choose_chunks(ntiles, nz, nsm);
  const int zc = (nz + nzc - 1) / nzc;
  const double ih2 = ctx->ih2;
  S3Args p{a, b, out, partials, nx, ny, nz, zc, 1.0 / dt, 0.5 * (1.0 - ctx->cfg.gamma), ih2,
           0.5 * ih2 * ih2, -ih2, 0, OP == OP_JV ? ctx->gate : nullptr};
  S3Maps m;
  memset(&m, 0, sizeof(m));
  const int* n = ctx->cfg.n;
  const int box[3] = {WX, WY, 1}, xbox[3] = {4, WY, 1}, ybox[3] = {WX, 4, 1}, cbox[3] = {4, 4, 1};
  if (nx % 2 == 0 && nx >= WX && ny >= WY && tma_usable(a) && tma_usable(b) &&
      tma_encode(&m.a, a, 3, n, box) && tma_encode(&m.b, b, 3, n, box)) {
    p.mode = 1;
    if (nx % TX == 0 && ny % TY == 0 && nx >= 2 * TX && ny >= 2 * TY &&
        tma_encode(&m.xa, a, 3, n, xbox) && tma_encode(&m.xb, b, 3, n, xbox) &&
        tma_encode(&m.ya, a, 3, n, ybox) && tma_encode(&m.yb, b, 3, n, ybox) &&
        tma_encode(&m.ca, a, 3, n, cbox) && tma_encode(&m.cb, b, 3, n, cbox))
      p.mode = 2;
  }
  dim3 grid(ntiles, nzc);
  if (nparts) *nparts = grid.x * grid.y;
  stencil3d_kernel<OP><<<grid, NT, SMEM_BYTES, ctx->stream>>>(m, p);
  ctx->launches++;
  pfc_account(ctx, OP == OP_RESID ? PFC_K_RESIDUAL : PFC_K_JV, 24.0 * ctx->N,
              (OP == OP_RESID ? 42.0 : 31.0) * ctx->N);
  return cudaGetLastError();
}

}  // namespace

int stencil3d_tiles(int nx, int ny) { return ((nx + TX - 1) / TX) * ((ny + TY - 1) / TY); }

cudaError_t launch_residual_3d(pfc_ctx* ctx, const double* phi_new, const double* phi_old,
                               double dt, double* F, double* partials, int* nparts) {
  return launch3d<OP_RESID>(ctx, phi_new, phi_old, dt, F, partials, nparts);
}

cudaError_t launch_jv_3d(pfc_ctx* ctx, const double* v, const double* c, double dt,
                         double* out) {
  return launch3d<OP_JV>(ctx, v, c, dt, out, nullptr, nullptr);
}
