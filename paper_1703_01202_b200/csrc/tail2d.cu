// tail2d.cu -- the Arnoldi step after the preconditioner in ONE cooperative kernel (2D grids up
// to ~4M nodes: configs 1-3), sm_100a.
//
// Step j of the right-preconditioned FGMRES(m) of P:369-380, after z_j = M^{-1} v_j (the RAS
// apply) has been computed:
//   w   = J z_j                                 (Eq. Jacobi, matrix-free)
//   h1  = V^T w,  w <- w - V h1                 (CGS2 pass 1)
//   h2  = V^T w,  w <- w - V h2,  |w|^2         (CGS2 pass 2)
//   v_{j+1} = w / |w|                           (the next basis vector; the host decides from
//                                                h1 + h2 and |w| whether the cycle continues)
// On the small 2D grids these five operations were five kernels of a few microseconds each
// (launch latency and an L2 round trip of w per kernel).  Here each thread keeps its MAXP
// nodes of w in registers through all phases; the three inner-product reductions are grid-wide
// (cooperative launch, grid.sync between phases) in a FIXED order, so results are bitwise
// reproducible run to run and identical in every block:
//   per block: warp xor-butterflies -> shared memory -> fixed warp order -> partials[block][i]
//   after grid.sync: warp w sums value i = w, w+nw, ... over the blocks (lane-strided, fixed
//   butterfly) -> shared h[i] in every block.
// J z uses the direct 25-point class-weight form of the linear part (the same weights as the 2D
// subdomain kernels) plus the 5-point -Delta(c z), with periodic wrap.
#include <cooperative_groups.h>

#include "pfc_device.cuh"
#include "pfc_internal.h"
#include "gmres_close.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int TT = 256;            // threads per block
constexpr int NWT = TT / 32;
constexpr int HS = 40;             // partial slots per block (>= PFC_MAX_RESTART + 1)

struct TailArgs {
  const double* V;     // basis, ldv = N
  const double* z;     // z_j = M^{-1} v_j
  const double* c;     // Jacobian coefficient
  double* vnext;       // v_{j+1}
  double* partials;    // gridDim.x x HS
  double* out;         // host scalars: h1 at [0, 32), h2 at [32, 64), |w|^2 at [64]
  size_t N;
  int nx, ny, j;
  double W[6];         // classes (0,0) (0,1) (0,2) (1,1) (0,3) (1,2) of the linear part
  double ih2;
  // device-resident FGMRES (row f1): skip when *gate != 0 (a speculative step after the cycle
  // stopped); gm != null: block 0 closes the Arnoldi step on the device (Givens, stop flag)
  const int* gate;
  pfc_gmres_dev* gm;
  const double* dtp;   // graph path (f1): dt-dependent scalars on the device (dt_w0)
};

// J z at node (x, y): sum over the radius-3 diamond of W_class z + the 5-point -Delta(c z)
__device__ __forceinline__ double jz_point(const TailArgs& p, double W0, int x, int y) {
  const int nx = p.nx, ny = p.ny;
  int xs[7], ys[7];
#pragma unroll
  for (int d = -3; d <= 3; ++d) {
    int a = x + d, b = y + d;
    a += a < 0 ? nx : (a >= nx ? -nx : 0);
    b += b < 0 ? ny : (b >= ny ? -ny : 0);
    xs[d + 3] = a;
    ys[d + 3] = b * nx;
  }
  const double* z = p.z;
  const double* c = p.c;
  auto Z = [&](int dx, int dy) { return __ldg(z + ys[dy + 3] + xs[dx + 3]); };
  auto Cc = [&](int dx, int dy) { return __ldg(c + ys[dy + 3] + xs[dx + 3]); };
  const double z0 = Z(0, 0);
  const double s01 = (Z(-1, 0) + Z(1, 0)) + (Z(0, -1) + Z(0, 1));
  const double s02 = (Z(-2, 0) + Z(2, 0)) + (Z(0, -2) + Z(0, 2));
  const double s11 = (Z(-1, -1) + Z(1, -1)) + (Z(-1, 1) + Z(1, 1));
  const double s03 = (Z(-3, 0) + Z(3, 0)) + (Z(0, -3) + Z(0, 3));
  const double s12 = ((Z(-1, -2) + Z(1, -2)) + (Z(-2, -1) + Z(2, -1))) +
                     ((Z(-2, 1) + Z(2, 1)) + (Z(-1, 2) + Z(1, 2)));
  double r = W0 * z0;
  r = fma(p.W[1], s01, r);
  r = fma(p.W[2], s02, r);
  r = fma(p.W[3], s11, r);
  r = fma(p.W[4], s03, r);
  r = fma(p.W[5], s12, r);
  // -Delta(c z) = -ih2 (sum of the 4 neighbours' c z - 4 c z)
  const double cz = (Cc(-1, 0) * Z(-1, 0) + Cc(1, 0) * Z(1, 0)) +
                    (Cc(0, -1) * Z(0, -1) + Cc(0, 1) * Z(0, 1));
  return fma(-p.ih2, fma(-4.0, Cc(0, 0) * z0, cz), r);
}

__device__ __forceinline__ double warp_total(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// block partial of value i (every thread passes its contribution s): warp totals in red[warp]
__device__ __forceinline__ void block_put(double s, int i, double* red) {
  s = warp_total(s);
  if ((threadIdx.x & 31) == 0) red[(threadIdx.x >> 5) * HS + i] = s;
}
// after __syncthreads: thread i < nv writes the block partial of value i (fixed warp order)
__device__ __forceinline__ void block_flush(int nv, const double* red, double* partials) {
  if (threadIdx.x < nv) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NWT; ++w) t += red[w * HS + threadIdx.x];
    partials[(size_t)blockIdx.x * HS + threadIdx.x] = t;
  }
}
// after grid.sync: the grid totals of values 0..nv-1 into h[] (shared), identical in every block
__device__ __forceinline__ void grid_total(int nv, const double* partials, double* h) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = wid; i < nv; i += NWT) {
    double t = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) t += __ldcg(partials + (size_t)b * HS + i);
    t = warp_total(t);
    if (lane == 0) h[i] = t;
  }
  __syncthreads();
}

template <int MAXP>
__global__ void __launch_bounds__(TT) k_arnoldi_tail(const __grid_constant__ TailArgs p) {
  if (p.gate && *p.gate) return;   // uniform: every block reads the same flag
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[NWT * HS];
  __shared__ double h1[HS], h2[HS], hx[2];
  const size_t N = p.N;
  const size_t G = (size_t)gridDim.x * TT;
  const size_t g = (size_t)blockIdx.x * TT + threadIdx.x;
  const int j = p.j;
  const double W0 = dt_w0<2>(p.dtp, p.W[0]);
  double w[MAXP];
  // ---- w = J z_j
#pragma unroll
  for (int k = 0; k < MAXP; ++k) {
    const size_t q = g + k * G;
    w[k] = 0.0;
    if (q < N) w[k] = jz_point(p, W0, (int)(q % p.nx), (int)(q / p.nx));
  }
  // ---- pass 1: h1 = V^T w
  for (int i = 0; i <= j; ++i) {
    const double* Vi = p.V + (size_t)i * N;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < MAXP; ++k) {
      const size_t q = g + k * G;
      if (q < N) s = fma(__ldcg(Vi + q), w[k], s);
    }
    block_put(s, i, red);
  }
  __syncthreads();
  block_flush(j + 1, red, p.partials);
  grid.sync();
  grid_total(j + 1, p.partials, h1);
  // ---- pass 2: w <- w - V h1, h2 = V^T w, |w|^2
  for (int i = 0; i <= j; ++i) {
    const double* Vi = p.V + (size_t)i * N;
    const double hi = h1[i];
#pragma unroll
    for (int k = 0; k < MAXP; ++k) {
      const size_t q = g + k * G;
      if (q < N) w[k] = fma(-hi, __ldcg(Vi + q), w[k]);
    }
  }
  for (int i = 0; i <= j; ++i) {
    const double* Vi = p.V + (size_t)i * N;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < MAXP; ++k) {
      const size_t q = g + k * G;
      if (q < N) s = fma(__ldcg(Vi + q), w[k], s);
    }
    block_put(s, i, red);
  }
  {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < MAXP; ++k) s = fma(w[k], w[k], s);
    block_put(s, j + 1, red);
  }
  __syncthreads();
  block_flush(j + 2, red, p.partials);
  grid.sync();
  grid_total(j + 2, p.partials, h2);
  // ---- pass 3: w <- w - V h2, |w|^2
  for (int i = 0; i <= j; ++i) {
    const double* Vi = p.V + (size_t)i * N;
    const double hi = h2[i];
#pragma unroll
    for (int k = 0; k < MAXP; ++k) {
      const size_t q = g + k * G;
      if (q < N) w[k] = fma(-hi, __ldcg(Vi + q), w[k]);
    }
  }
  {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < MAXP; ++k) s = fma(w[k], w[k], s);
    block_put(s, 0, red);
  }
  __syncthreads();
  block_flush(1, red, p.partials);
  grid.sync();
  grid_total(1, p.partials, hx);
  // ---- v_{j+1} = w / |w| (written unless |w| = 0; the host checks breakdown)
  const double nrm2 = hx[0];
  if (nrm2 > 0.0) {
    const double ihn = 1.0 / sqrt(nrm2);
#pragma unroll
    for (int k = 0; k < MAXP; ++k) {
      const size_t q = g + k * G;
      if (q < N) p.vnext[q] = ihn * w[k];
    }
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i <= j; i += TT) {
      p.out[i] = h1[i];
      p.out[32 + i] = h2[i];
    }
    if (threadIdx.x == 0) {
      p.out[64] = nrm2;
      if (p.gm) arnoldi_close(p.gm, j, h1, h2, nrm2);
    }
  }
}

// Tiled variant (grids with n_x % 64 == 0): block b owns the 64 x 4RS tile (x0, y0) of the
// grid, thread t the column x0 + t % 64, rows y0 + RS (t / 64) .. + RS - 1.  z (halo 3) and c
// (halo 1) of the tile are staged in shared memory once, so J z is evaluated column by column
// (the direct 25-point class weights + the 5-point -Delta(c z)) from shared memory with the
// column's y-neighbours in registers, instead of 30 gathers per node through L1 with 64-bit
// index arithmetic; the CGS2 passes then read V row-coalesced at the thread's own nodes.
constexpr int TXT = 64;
template <int RS>
struct TileGeom {
  static constexpr int TYT = 4 * RS, ZW = TXT + 6, ZH = TYT + 6, CW = TXT + 2, CH = TYT + 2;
  static constexpr int SMEM = (ZW * ZH + CW * CH) * (int)sizeof(double);
};

template <int RS>
__global__ void __launch_bounds__(TT, 2) k_arnoldi_tail_tile(const __grid_constant__ TailArgs p) {
  if (p.gate && *p.gate) return;   // uniform: every block reads the same flag
  using TG = TileGeom<RS>;
  constexpr int TYT = TG::TYT, ZW = TG::ZW, ZH = TG::ZH, CW = TG::CW, CH = TG::CH;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double tile_sm[];
  double* zt = tile_sm;             // z on the tile + halo 3
  double* ct = tile_sm + ZW * ZH;   // c on the tile + halo 1
  __shared__ double red[NWT * HS];
  __shared__ double h1[HS], h2[HS], hx[2];
  const int nx = p.nx, ny = p.ny;
  const size_t N = p.N;
  const int ntx = nx / TXT;
  const int x0 = (blockIdx.x % ntx) * TXT, y0 = (blockIdx.x / ntx) * TYT;
  for (int q = threadIdx.x; q < ZW * ZH; q += TT) {
    const int r = q / ZW, cc = q - r * ZW;
    const int gx = wrapi(x0 + cc - 3, nx), gy = wrapi(y0 + r - 3, ny);
    zt[q] = __ldcg(p.z + (size_t)gx + (size_t)nx * gy);
  }
  for (int q = threadIdx.x; q < CW * CH; q += TT) {
    const int r = q / CW, cc = q - r * CW;
    const int gx = wrapi(x0 + cc - 1, nx), gy = wrapi(y0 + r - 1, ny);
    ct[q] = __ldcg(p.c + (size_t)gx + (size_t)nx * gy);
  }
  const int j = p.j;
  const double W0 = dt_w0<2>(p.dtp, p.W[0]);
  const int tx = threadIdx.x % TXT, yr = (threadIdx.x / TXT) * RS;
  const size_t g0 = (size_t)(x0 + tx) + (size_t)nx * (size_t)(y0 + yr);
  __syncthreads();
  double w[RS];
  // ---- w = J z_j: linear part, column by column (rows yr - a .. yr + RS - 1 + a of column
  // dx in registers), then -Delta(c z) from the 5-point neighbours
  {
#pragma unroll
    for (int r = 0; r < RS; ++r) w[r] = 0.0;
    const double* zc = zt + (yr + 3) * ZW + tx + 3;   // (row yr, column tx) of the z tile
#pragma unroll
    for (int dx = -3; dx <= 3; ++dx) {
      const int a = 3 - (dx < 0 ? -dx : dx);
      double col[RS + 6];
#pragma unroll
      for (int rr = -a; rr < RS + a; ++rr) col[rr + a] = zc[rr * ZW + dx];
#pragma unroll
      for (int r = 0; r < RS; ++r)
#pragma unroll
        for (int dy = -a; dy <= a; ++dy) {
          const int ax = dx < 0 ? -dx : dx, ay = dy < 0 ? -dy : dy;
          const int cls = (ax + ay == 0) ? 0 : (ax + ay == 1) ? 1 : (ax == 1 && ay == 1) ? 3
                          : (ax + ay == 2) ? 2 : (ax + ay == 3 && (ax == 0 || ay == 0)) ? 4 : 5;
          w[r] = fma(cls == 0 ? W0 : p.W[cls], col[r + dy + a], w[r]);
        }
    }
    const double* cc = ct + (yr + 1) * CW + tx + 1;
    double czo[RS + 2];   // c z of the own column, rows -1 .. RS
#pragma unroll
    for (int rr = -1; rr <= RS; ++rr) czo[rr + 1] = cc[rr * CW] * zc[rr * ZW];
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      const double lap = (cc[r * CW - 1] * zc[r * ZW - 1] + cc[r * CW + 1] * zc[r * ZW + 1]) +
                         (czo[r] + czo[r + 2]) - 4.0 * czo[r + 1];
      w[r] = fma(-p.ih2, lap, w[r]);
    }
  }
  // ---- pass 1: h1 = V^T w
  for (int i = 0; i <= j; ++i) {
    const double* Vi = p.V + (size_t)i * N + g0;
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < RS; ++r) s = fma(__ldcg(Vi + (size_t)r * nx), w[r], s);
    block_put(s, i, red);
  }
  __syncthreads();
  block_flush(j + 1, red, p.partials);
  grid.sync();
  grid_total(j + 1, p.partials, h1);
  // ---- pass 2: w <- w - V h1, h2 = V^T w, |w|^2
  for (int i = 0; i <= j; ++i) {
    const double* Vi = p.V + (size_t)i * N + g0;
    const double hi = h1[i];
#pragma unroll
    for (int r = 0; r < RS; ++r) w[r] = fma(-hi, __ldcg(Vi + (size_t)r * nx), w[r]);
  }
  for (int i = 0; i <= j; ++i) {
    const double* Vi = p.V + (size_t)i * N + g0;
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < RS; ++r) s = fma(__ldcg(Vi + (size_t)r * nx), w[r], s);
    block_put(s, i, red);
  }
  {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < RS; ++r) s = fma(w[r], w[r], s);
    block_put(s, j + 1, red);
  }
  __syncthreads();
  block_flush(j + 2, red, p.partials);
  grid.sync();
  grid_total(j + 2, p.partials, h2);
  // ---- pass 3: w <- w - V h2, |w|^2
  for (int i = 0; i <= j; ++i) {
    const double* Vi = p.V + (size_t)i * N + g0;
    const double hi = h2[i];
#pragma unroll
    for (int r = 0; r < RS; ++r) w[r] = fma(-hi, __ldcg(Vi + (size_t)r * nx), w[r]);
  }
  {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < RS; ++r) s = fma(w[r], w[r], s);
    block_put(s, 0, red);
  }
  __syncthreads();
  block_flush(1, red, p.partials);
  grid.sync();
  grid_total(1, p.partials, hx);
  // ---- v_{j+1} = w / |w| (written unless |w| = 0; the host checks breakdown)
  const double nrm2 = hx[0];
  if (nrm2 > 0.0) {
    const double ihn = 1.0 / sqrt(nrm2);
#pragma unroll
    for (int r = 0; r < RS; ++r) p.vnext[g0 + (size_t)r * nx] = ihn * w[r];
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i <= j; i += TT) {
      p.out[i] = h1[i];
      p.out[32 + i] = h2[i];
    }
    if (threadIdx.x == 0) {
      p.out[64] = nrm2;
      if (p.gm) arnoldi_close(p.gm, j, h1, h2, nrm2);
    }
  }
}

typedef void (*tail_tile_fn)(const TailArgs);

tail_tile_fn pick_tail_tile(int rs, int* smem) {
  switch (rs) {
#define TTC(R) case R: *smem = TileGeom<R>::SMEM; return k_arnoldi_tail_tile<R>;
    TTC(1) TTC(2) TTC(4) TTC(8) TTC(16)
#undef TTC
  }
  return nullptr;
}

// tiled plan: the smallest rows-per-thread RS whose tiles are all co-resident; 0 if none
int tail_tile_plan(pfc_ctx* ctx, int* blocks, int* rs_out, int* smem_out) {
  const int nx = ctx->cfg.n[0], ny = ctx->cfg.n[1];
  const char* e = getenv("PFC_TAIL_TILE");
  if ((e && e[0] == '0') || nx % TXT != 0) return 0;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  // PFC_TAIL_RS=r forces r rows per thread (A/B probes); small grids prefer ONE tile (the grid
  // syncs become block barriers of a single co-resident block)
  const char* fr = getenv("PFC_TAIL_RS");
  const int rforce = fr ? atoi(fr) : 0;
  for (int rs = 1; rs <= 16; rs *= 2) {
    if (ny % (4 * rs) != 0) continue;
    if (rforce && rs != rforce) continue;
    int smem = 0;
    tail_tile_fn fn = pick_tail_tile(rs, &smem);
    if (!fn) continue;
    if (cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, TT, smem) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      continue;
    }
    const long need = (long)(nx / TXT) * (ny / (4 * rs));
    if (need <= (long)sms * per_sm) {
      *blocks = (int)need;
      *rs_out = rs;
      *smem_out = smem;
      return 1;
    }
  }
  return 0;
}

typedef void (*tail_fn)(const TailArgs);

tail_fn pick_tail(int maxp) {
  switch (maxp) {
    case 1: return k_arnoldi_tail<1>;
    case 2: return k_arnoldi_tail<2>;
    case 4: return k_arnoldi_tail<4>;
    case 8: return k_arnoldi_tail<8>;
    case 16: return k_arnoldi_tail<16>;
    case 32: return k_arnoldi_tail<32>;
  }
  return nullptr;
}

// launch plan: blocks (co-resident) and nodes per thread
bool tail_plan(pfc_ctx* ctx, int* blocks, int* maxp) {
  const size_t N = ctx->N;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  for (int mp = 1; mp <= 32; mp *= 2) {
    tail_fn fn = pick_tail(mp);
    if (!fn) continue;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, TT, 0) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      continue;
    }
    const size_t cap = (size_t)sms * per_sm;             // co-resident blocks
    const size_t need = (N + (size_t)TT * mp - 1) / ((size_t)TT * mp);
    if (need <= cap) {
      *blocks = (int)need;
      *maxp = mp;
      return true;
    }
  }
  return false;
}

}  // namespace

// 1 if the fused Arnoldi tail serves this context (2D, periodic, M = 1, N within the plan)
int tail_enabled(pfc_ctx* ctx) {
  const pfc_config& c = ctx->cfg;
  const char* e = getenv("PFC_TAIL");
  if (e && e[0] == '0') return 0;
  if (c.ndim != 2 || generic_path(c) || c.gmres_restart + 1 > HS) return 0;
  int b = 0, mp = 0, sm = 0;
  ctx->tail_rs = 0;
  if (tail_tile_plan(ctx, &b, &mp, &sm)) {
    ctx->tail_rs = mp;
    ctx->tail_blocks = b;
    return 1;
  }
  return tail_plan(ctx, &b, &mp) ? 1 : 0;
}

// Arnoldi step j after the preconditioner: w = J z, CGS2 against V_0..V_j, v_{j+1} = w/|w|;
// h1 -> out[0..j], h2 -> out[32..32+j], |w|^2 -> out[64] (device scalars)
cudaError_t launch_arnoldi_tail(pfc_ctx* ctx, const double* V, const double* z, const double* c,
                                double dt, int j, double* vnext, double* out,
                                pfc_gmres_dev* gm) {
  const pfc_config& cf = ctx->cfg;
  int blocks = 0, maxp = 0;
  if (!ctx->tail_rs && !tail_plan(ctx, &blocks, &maxp)) return cudaErrorInvalidValue;
  TailArgs p{};
  p.V = V; p.z = z; p.c = c; p.vnext = vnext; p.partials = ctx->partials; p.out = out;
  p.N = ctx->N; p.nx = cf.n[0]; p.ny = cf.n[1]; p.j = j;
  const double ih2 = ctx->ih2, ih4 = ih2 * ih2, ih6 = ih4 * ih2;
  const double al = 0.5 * (1.0 - cf.gamma);
  // class weights of v/dt - alpha Delta v - Delta^2 v - Delta^3 v / 2
  p.W[0] = 1.0 / dt + 4.0 * al * ih2 - 20.0 * ih4 + 56.0 * ih6;
  p.dtp = ctx->dtdev;
  p.W[1] = -al * ih2 + 8.0 * ih4 - 28.5 * ih6;
  p.W[2] = -ih4 + 6.0 * ih6;
  p.W[3] = -2.0 * ih4 + 12.0 * ih6;
  p.W[4] = -0.5 * ih6;
  p.W[5] = -1.5 * ih6;
  p.ih2 = ih2;
  p.gate = ctx->gate;
  p.gm = gm;
  void* args[] = {&p};
  cudaError_t e;
  if (ctx->tail_rs) {   // tiled J z (shared memory; plan made once by tail_enabled)
    int tsm = 0;
    tail_tile_fn fn = pick_tail_tile(ctx->tail_rs, &tsm);
    e = cudaLaunchCooperativeKernel((const void*)fn, dim3(ctx->tail_blocks), dim3(TT), args,
                                    (size_t)tsm, ctx->stream);
  }
  else
    e = cudaLaunchCooperativeKernel((const void*)pick_tail(maxp), dim3(blocks), dim3(TT), args, 0,
                                    ctx->stream);
  ctx->launches++;
  {  // algorithmic: z (25-pt) + c read once, V read 3 (j+1) times, v_{j+1} written
    const double n = (double)ctx->N, jj = j + 1;
    pfc_account(ctx, PFC_K_ORTH, 8.0 * n * (2.0 + 3.0 * jj + 1.0),
                n * (50.0 + 12.0 + 8.0 * jj + 6.0));
  }
  return e;
}
