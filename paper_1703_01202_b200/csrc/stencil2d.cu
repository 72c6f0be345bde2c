// stencil2d.cu -- fused 2D DVD residual (K1) and Jacobian-vector product (K2), sm_100a.
//
// Residual, Eq. (NSOP) P:257-263 with M = 1, and A from Eq. (discretedG) P:250-255:
//   F = (Phi - psi)/dt - Delta_d[(1-gamma)u + 2 Delta_d u + Delta_d^2 u + N(Phi,psi)],
//   u = (Phi+psi)/2, N = (Phi^3 + Phi^2 psi + Phi psi^2 + psi^3)/4.
// Jacobian (Eq. Jacobi):
//   Jv = v/dt - Delta_d[(1/2)(1-gamma)v + c v + Delta_d v + (1/2) Delta_d^2 v].
// Delta_d (1+Delta_d)^2 is a radius-3 stencil ("3 is the stencil width"), applied by
// composing the UNSCALED 5-point Laplacian Lt f = sum of the 4 neighbours - 4 f three times
// (Delta_d = ih2 Lt, the h^-2 factors folded into the coefficients, as in stencil3d.cu):
//   resid: s = Phi + psi,  A = (1-gamma)/2 s + ih2 Lt s + ih2^2/2 Lt Lt s + s (Phi^2+psi^2)/4,
//          F = (Phi - psi)/dt - ih2 Lt A
//   jv:    B = ((1-gamma)/2 + c) v + ih2 Lt v + ih2^2/2 Lt Lt v,   Jv = v/dt - ih2 Lt B
//
// Barrier-free warp-per-strip y-march (no shared memory).  A warp owns a strip of 64 columns
// (window cols 0..63 <-> x = 56k - 4 + col; outputs are cols 4..59, 56 per strip) and a chunk
// of rows; lane l holds the column pair (2l, 2l+1).  Streaming row t it computes
//     Lt s|v (row t-1)  ->  A|B (t-2)  ->  F|Jv (t-3)
// with y-neighbours in register queues (period 3, renamed under a 3x unroll) and x-neighbours
// from the adjacent lanes by warp shuffles; the strip's outer 3 columns carry the halo (the
// values computed there at the warp edge are never consumed by an output).  Input rows are
// read as coalesced 16-byte pairs (periodic wrap per lane and per row; a pair never straddles
// the seam since x is even), PF rows ahead of use.  Optional fused ||F||^2 partial per warp.
#include "pfc_device.cuh"
#include "pfc_internal.h"

#include <algorithm>
#include <cstdlib>

namespace {

constexpr int SO = 56, HLO = 4;            // outputs per 64-column strip, left halo
constexpr int NT = 256;                    // 8 independent warps per CTA
constexpr int PF = 3;                      // rows in flight ahead of use (= queue period)
// grids below this many nodes use the tile kernel (measured crossover)
#ifndef ST2_STRIP_MIN
#define ST2_STRIP_MIN (2048L * 2048L)
#endif
constexpr long kStripMinNodes = ST2_STRIP_MIN;

enum { OP_RESID = 0, OP_JV = 1 };

struct S2Args {
  const double* a;   // Phi (resid) | v (jv)
  const double* b;   // psi (resid) | c (jv)
  double* out;
  double* partials;  // per-warp ||out||^2 or nullptr
  int nx, ny;
  int nstrips, nchunks, chunk;
  double idt, k0, k1, k2, kout;   // (1-gamma)/2, ih2, ih2^2/2, -ih2
  int vec;           // 16-byte pair loads / stores (n_x even, aligned bases)
  const int* gate;   // device-resident FGMRES: skip the launch when *gate != 0 (f1)
  const double* dtp; // graph path (f1): dt on the device
};

struct p2 { double x, y; };   // the lane's two columns

__device__ __forceinline__ p2 add2(p2 a, p2 b) { return {a.x + b.x, a.y + b.y}; }

// unscaled 5-point Laplacian of the lane's pair: x-neighbours from the adjacent lanes,
// y-neighbours m (row above in the march) and p (row below)
__device__ __forceinline__ p2 lap_pair(p2 f, p2 m, p2 p) {
  const double lft = __shfl_up_sync(0xffffffffu, f.y, 1);
  const double rgt = __shfl_down_sync(0xffffffffu, f.x, 1);
  return {fma(-4.0, f.x, (lft + f.y) + (m.x + p.x)), fma(-4.0, f.y, (f.x + rgt) + (m.y + p.y))};
}

template <int OP>
__global__ void __launch_bounds__(NT, 2) stencil2d_kernel(const __grid_constant__ S2Args p) {
  if (p.gate && *p.gate) return;
  const double idt = dt_inv(p.dtp, p.idt);
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
  if (item >= p.nstrips * p.nchunks) return;   // whole warps only
  const int strip = item % p.nstrips, ck = item / p.nstrips;
  const int nx = p.nx, ny = p.ny;
  const int xw = strip * SO - HLO + 2 * lane;   // global x of the lane's first column
  const int y0 = ck * p.chunk;
  const int rows = min(p.chunk, ny - y0);
  const int T = rows + 6;
  const int Tp = (T + 2) / 3 * 3;
  const int xa = wrapi(xw, nx), xb = wrapi(xw + 1, nx);
  // outputs: window cols 4..59 inside the (possibly ragged) grid
  const bool oa = lane >= 2 && lane < 30 && xw < nx, ob = lane >= 2 && lane < 30 && xw + 1 < nx;

  auto load = [&](const double* f, int t) {   // the lane's pair of input row y0 - 3 + t
    const size_t rowo = (size_t)nx * wrapi(y0 - 3 + t, ny);
    if (p.vec) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(f + rowo + xa));
      return p2{v.x, v.y};
    }
    return p2{__ldg(f + rowo + xa), __ldg(f + rowo + xb)};
  };
  // prefetch queue: rows t .. t+PF-1 (period PF = 3 like every other queue)
  p2 fa0 = load(p.a, 0), fa1 = load(p.a, 1), fa2 = load(p.a, 2);
  p2 fb0 = load(p.b, 0), fb1 = load(p.b, 1), fb2 = load(p.b, 2);
  const p2 Z{0.0, 0.0};
  // queues: A1,A2 = Phi|v at t-1,t-2;  B1,B2 = psi|c;  L2,L3 = Lt at t-2,t-3;  M3,M4 = A|B
  // at t-3,t-4;  P2,P3 = (Phi-psi)/dt | v/dt at t-2,t-3
  p2 A1 = Z, A2 = Z, B1 = Z, B2 = Z, L2 = Z, L3 = Z, M3 = Z, M4 = Z, P2 = Z, P3 = Z;
  double nrm = 0.0;
  double* outp = p.out + (size_t)xa;

#pragma unroll 3
  for (int t = 0; t < Tp; ++t) {
    const p2 A0 = fa0, B0 = fb0;              // row t
    fa0 = fa1; fa1 = fa2; fb0 = fb1; fb1 = fb2;
    fa2 = load(p.a, t + PF);                  // rows past the end wrap harmlessly
    fb2 = load(p.b, t + PF);
    // ---- stage 1: Lt s | Lt v at row t-1, pointwise output part of row t-1
    p2 Lnew, Pnew;
    if (OP == OP_RESID) {
      Lnew = lap_pair(add2(A1, B1), add2(A2, B2), add2(A0, B0));
      Pnew = {(A1.x - B1.x) * idt, (A1.y - B1.y) * idt};
    } else {
      Lnew = lap_pair(A1, A2, A0);
      Pnew = {A1.x * idt, A1.y * idt};
    }
    // ---- stage 2: A | B at row t-2
    p2 Mnew;
    {
      const p2 LL = lap_pair(L2, L3, Lnew);
      p2 base;
      if (OP == OP_RESID) {   // (1-gamma)/2 s + s (Phi^2 + psi^2) / 4
        auto nb = [&](double ph, double ps) {
          const double s = ph + ps;
          return s * fma(0.25, fma(ph, ph, ps * ps), p.k0);
        };
        base = {nb(A2.x, B2.x), nb(A2.y, B2.y)};
      } else {
        base = {(p.k0 + B2.x) * A2.x, (p.k0 + B2.y) * A2.y};
      }
      Mnew = {fma(p.k2, LL.x, fma(p.k1, L2.x, base.x)), fma(p.k2, LL.y, fma(p.k1, L2.y, base.y))};
    }
    // ---- stage 3: F | Jv at row t-3
    const p2 LM = lap_pair(M3, M4, Mnew);
    const double o0 = fma(p.kout, LM.x, P3.x), o1 = fma(p.kout, LM.y, P3.y);
    A2 = A1; A1 = A0; B2 = B1; B1 = B0;
    L3 = L2; L2 = Lnew;
    M4 = M3; M3 = Mnew;
    P3 = P2; P2 = Pnew;
    if (t >= 6 && t - 6 < rows) {
      double* o = outp + (size_t)nx * (y0 + t - 6);
      if (p.vec && oa && ob) {
        *reinterpret_cast<double2*>(o) = make_double2(o0, o1);
        nrm += o0 * o0 + o1 * o1;
      } else {
        if (oa) { o[0] = o0; nrm += o0 * o0; }
        if (ob) { o[xb - xa] = o1; nrm += o1 * o1; }
      }
    }
  }
  if (p.partials) {
    const double s = warp_sum(nrm);
    if (lane == 0) p.partials[item] = s;
  }
}


// ---------------------------------------------------------------------------------------
// Tile variant for small (L2-resident) grids, where the strip march has too few rows per
// warp to hide latency: one CTA per 32 x 16 output tile, its (40 x 22) input window staged
// by one TMA tile load per field (mbarrier completion; zero-filled out-of-range cells re-read
// with wrapped indices), then three in-shared-memory 5-point stages shrinking the halo
// 3 -> 2 -> 1 -> 0.  Same operators (composed in the order of the definition).
namespace tile {


constexpr int TX = 32, TY = 16;          // output tile
constexpr int HX = 4, HY = 3;            // loaded halo (x: 3 + 1 slack for 16-B rows)
constexpr int WX = TX + 2 * HX;          // 40
constexpr int WY = TY + 2 * HY;          // 22
constexpr int WN = WX * WY;
constexpr int NT = 256;


struct S2TArgs {
  const double* a;   // Phi (resid) | v (jv)
  const double* b;   // psi (resid) | c (jv)
  double* out;
  double* partials;  // per-tile ||out||^2 or nullptr
  int nx, ny;
  double idt, gamma, ih2;
  int use_tma;
  const int* gate;   // device-resident FGMRES: skip the launch when *gate != 0 (f1)
  const double* dtp; // graph path (f1): dt on the device
};

__device__ __forceinline__ double lap5(const double* f, int q, double ih2) {
  return ih2 * ((f[q - 1] + f[q + 1]) + (f[q - WX] + f[q + WX]) - 4.0 * f[q]);
}

template <int OP>
__global__ void __launch_bounds__(NT) stencil2d_tile_kernel(const __grid_constant__ CUtensorMap ma,
                                                       const __grid_constant__ CUtensorMap mb,
                                                       S2TArgs p) {
  // declared as a shared array (not re-derived through an integer) so that every access
  // compiles to LDS/STS with 32-bit shared addressing; 128-B aligned for TMA destinations
  extern __shared__ __align__(128) double smem_dyn[];
  double* base = smem_dyn;
  double* A0 = base;            // Phi | v
  double* B0 = A0 + WN;         // psi | c
  double* U = B0 + WN;          // u (resid only)
  double* L1 = U + WN;          // Delta u | Delta v
  double* AA = L1 + WN;         // A | bracket of J
  __shared__ uint64_t bar;
  __shared__ double red[64];

  if (p.gate && *p.gate) return;
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int gx0 = x0 - HX, gy0 = y0 - HY;
  const int nx = p.nx, ny = p.ny;

  if (p.use_tma) {
    if (tid == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
      mbar_expect_tx(&bar, 2u * WN * sizeof(double));
      tma_load_2d(A0, &ma, &bar, gx0, gy0);
      tma_load_2d(B0, &mb, &bar, gx0, gy0);
    }
    mbar_wait(&bar, 0);
    const bool edge = gx0 < 0 || gy0 < 0 || gx0 + WX > nx || gy0 + WY > ny;
    if (edge) {  // periodic wrap of the zero-filled out-of-range cells
      for (int q = tid; q < WN; q += NT) {
        int gx = gx0 + q % WX, gy = gy0 + q / WX;
        if (gx < 0 || gx >= nx || gy < 0 || gy >= ny) {
          size_t g = (size_t)wrapi(gx, nx) + (size_t)nx * wrapi(gy, ny);
          A0[q] = p.a[g];
          B0[q] = p.b[g];
        }
      }
    }
  } else {
    for (int q = tid; q < WN; q += NT) {
      int gx = gx0 + q % WX, gy = gy0 + q / WX;
      size_t g = (size_t)wrapi(gx, nx) + (size_t)nx * wrapi(gy, ny);
      A0[q] = p.a[g];
      B0[q] = p.b[g];
    }
  }
  __syncthreads();

  const double ih2 = p.ih2;
  const double* Lin;   // field whose Laplacian feeds stage r=2
  if (OP == OP_RESID) {
    // r = 3: u = (Phi + psi)/2 on columns [1, WX-1), all rows
    for (int q = tid; q < (WX - 2) * WY; q += NT) {
      int f = (q / (WX - 2)) * WX + 1 + q % (WX - 2);
      U[f] = 0.5 * (A0[f] + B0[f]);
    }
    __syncthreads();
    Lin = U;
  } else {
    Lin = A0;
  }
  // r = 2: L1 = Delta_d (u | v)
  for (int q = tid; q < (WX - 4) * (WY - 2); q += NT) {
    int f = (1 + q / (WX - 4)) * WX + 2 + q % (WX - 4);
    L1[f] = lap5(Lin, f, ih2);
  }
  __syncthreads();
  // r = 1
  for (int q = tid; q < (WX - 6) * (WY - 4); q += NT) {
    int f = (2 + q / (WX - 6)) * WX + 3 + q % (WX - 6);
    if (OP == OP_RESID) {
      double a = A0[f], b = B0[f];
      double N = 0.25 * (a * a * a + a * a * b + a * b * b + b * b * b);
      AA[f] = (1.0 - p.gamma) * U[f] + 2.0 * L1[f] + lap5(L1, f, ih2) + N;
    } else {
      double v = A0[f];
      AA[f] = (0.5 * (1.0 - p.gamma) + B0[f]) * v + L1[f] + 0.5 * lap5(L1, f, ih2);
    }
  }
  __syncthreads();
  // r = 0: outputs
  double nrm = 0.0;
  for (int q = tid; q < TX * TY; q += NT) {
    int r = q / TX, cc = q % TX;
    int f = (HY + r) * WX + HX + cc;
    int gx = x0 + cc, gy = y0 + r;
    double o;
    if (OP == OP_RESID) o = (A0[f] - B0[f]) * dt_inv(p.dtp, p.idt) - lap5(AA, f, ih2);
    else o = A0[f] * dt_inv(p.dtp, p.idt) - lap5(AA, f, ih2);
    if (gx < nx && gy < ny) {
      p.out[(size_t)gx + (size_t)nx * gy] = o;
      nrm += o * o;
    }
  }
  if (p.partials) {
    double s = block_sum(nrm, red);
    if (tid == 0) p.partials[blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}

constexpr int SMEM_BYTES = 5 * WN * (int)sizeof(double) + 128;

template <int OP>
cudaError_t launch2d_tile(pfc_ctx* ctx, const double* a, const double* b, double dt, double* out,
                     double* partials, int* nparts) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(stencil2d_tile_kernel<OP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int nx = ctx->cfg.n[0], ny = ctx->cfg.n[1];
  S2TArgs p{a, b, out, partials, nx, ny, 1.0 / dt, ctx->cfg.gamma, ctx->ih2, 0,
           OP == OP_JV ? ctx->gate : nullptr};
  p.dtp = ctx->dtdev;
  CUtensorMap ma, mb;
  memset(&ma, 0, sizeof(ma));
  memset(&mb, 0, sizeof(mb));
  const int box[2] = {WX, WY};
  if (nx % 2 == 0 && nx >= WX && ny >= WY && tma_usable(a) && tma_usable(b) &&
      tma_encode(&ma, a, 2, ctx->cfg.n, box) && tma_encode(&mb, b, 2, ctx->cfg.n, box))
    p.use_tma = 1;
  dim3 grid((nx + TX - 1) / TX, (ny + TY - 1) / TY);
  if (nparts) *nparts = grid.x * grid.y;
  stencil2d_tile_kernel<OP><<<grid, NT, SMEM_BYTES, ctx->stream>>>(ma, mb, p);
  ctx->launches++;
  // algorithmic: 2 fields in, 1 out; flops of the composed operator per node (2D)
  pfc_account(ctx, OP == OP_RESID ? PFC_K_RESIDUAL : PFC_K_JV, 24.0 * ctx->N,
              (OP == OP_RESID ? 36.0 : 25.0) * ctx->N);
  return cudaGetLastError();
}

}  // namespace tile

template <int OP>
cudaError_t launch2d(pfc_ctx* ctx, const double* a, const double* b, double dt, double* out,
                     double* partials, int* nparts) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0, v = 0;
    nsm = (cudaGetDevice(&dev) == cudaSuccess &&
           cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
              ? v : 148;
  }
  const int nx = ctx->cfg.n[0], ny = ctx->cfg.n[1];
  // PFC_ST2_KERNEL=strip|tile overrides the size rule (tests of both paths on every shape)
  const char* force = getenv("PFC_ST2_KERNEL");
  const bool use_tile = force ? force[0] == 't' : (long)nx * ny < kStripMinNodes;
  if (use_tile) return tile::launch2d_tile<OP>(ctx, a, b, dt, out, partials, nparts);
  const int nstrips = (nx + SO - 1) / SO;
  // rows per chunk: halved (not below 32: 6 warm-up rows per chunk) until ~16 warps per SM
  int chunk = ny;
  while (chunk > 32 && (long)nstrips * ((ny + chunk - 1) / chunk) < 16L * nsm) chunk = (chunk + 1) / 2;
  const long maxitems = (long)ctx->npartials - 64;
  while ((long)nstrips * ((ny + chunk - 1) / chunk) > maxitems && chunk < ny) chunk *= 2;
  chunk = std::min(chunk, ny);
  const int nchunks = (ny + chunk - 1) / chunk;
  const double ih2 = ctx->ih2;
  const bool vec = nx % 2 == 0 && tma_usable(a) && tma_usable(b) && tma_usable(out);
  S2Args p{a, b, out, partials, nx, ny, nstrips, nchunks, chunk, 1.0 / dt,
           0.5 * (1.0 - ctx->cfg.gamma), ih2, 0.5 * ih2 * ih2, -ih2, vec ? 1 : 0,
           OP == OP_JV ? ctx->gate : nullptr};
  p.dtp = ctx->dtdev;
  const int items = nstrips * nchunks;
  if (nparts) *nparts = items;
  stencil2d_kernel<OP><<<(items + NT / 32 - 1) / (NT / 32), NT, 0, ctx->stream>>>(p);
  ctx->launches++;
  // algorithmic: 2 fields in, 1 out; flops of the composed operator per node (2D)
  pfc_account(ctx, OP == OP_RESID ? PFC_K_RESIDUAL : PFC_K_JV, 24.0 * ctx->N,
              (OP == OP_RESID ? 36.0 : 25.0) * ctx->N);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_residual_2d(pfc_ctx* ctx, const double* phi_new, const double* phi_old,
                               double dt, double* F, double* partials, int* nparts) {
  return launch2d<OP_RESID>(ctx, phi_new, phi_old, dt, F, partials, nparts);
}

cudaError_t launch_jv_2d(pfc_ctx* ctx, const double* v, const double* c, double dt,
                         double* out) {
  return launch2d<OP_JV>(ctx, v, c, dt, out, nullptr, nullptr);
}
