// stencil3d.cu -- fused 3D DVD residual (K1) and Jacobian-vector product (K2), sm_100a.
//
// Same operators as stencil2d.cu (Eq. NSOP, Eq. discretedG, Eq. Jacobi
// P:351-356), 7-point Delta_d composed three times: a radius-3, 63-point stencil.
//
// 2.5D z-march.  A CTA owns a TX x TY column of outputs and a chunk of ZC z-planes.  It streams
// the input planes z0-3 .. z0+ZC+2 through a ring of RING plane buffers per field, filled by
// TMA (cp.async.bulk.tensor.3d, one (TX+8) x (TY+6) x 1 box per field and plane, PREFETCH
// planes ahead, one mbarrier per ring slot).  Every thread owns fixed xy positions of the
// plane window ("slots") for all stages; at plane t it computes
//     u(t) [halo 3]  ->  L1(t-1) [halo 2]  ->  A(t-2) [halo 1]  ->  F(t-3) [halo 0]
// where the xy-neighbours come from one shared-memory plane per stage (double-buffered) and
// the z-neighbours from per-thread register queues of the thread's own slots.  Periodic x/y
// wrap: TMA zero-fills out-of-range cells and edge tiles reload exactly those own-slot cells
// with wrapped loads; z wraps by plane index.  Optional fused ||F||^2 partial per CTA.
#include "pfc_device.cuh"
#include "pfc_internal.h"

namespace {

constexpr int TX = 32, TY = 16;
constexpr int HX = 4, HY = 3;
constexpr int WX = TX + 2 * HX;   // 40
constexpr int WY = TY + 2 * HY;   // 22
constexpr int WN = WX * WY;       // 880
constexpr int NT = 512;
constexpr int NS = (WN + NT - 1) / NT;  // slots per thread (2)
constexpr int RING = 6;
constexpr int PREFETCH = 3;

enum { OP_RESID = 0, OP_JV = 1 };

struct S3Args {
  const double* a;   // Phi | v
  const double* b;   // psi | c
  double* out;
  double* partials;
  int nx, ny, nz;
  int zc;            // planes per chunk
  double idt, gamma, ih2;
  int use_tma;
};

__device__ __forceinline__ bool in_region(int q, int r) {
  int qx = q % WX, qy = q / WX;
  return qx >= HX - r && qx < HX + TX + r && qy >= HY - r && qy < HY + TY + r;
}

__device__ __forceinline__ double lap_xy(const double* f, int q) {
  return (f[q - 1] + f[q + 1]) + (f[q - WX] + f[q + WX]) - 4.0 * f[q];
}

template <int OP>
__global__ void __launch_bounds__(NT, 1) stencil3d_kernel(const __grid_constant__ CUtensorMap ma,
                                                          const __grid_constant__ CUtensorMap mb,
                                                          S3Args p) {
  extern __shared__ unsigned char smem_raw[];
  double* base = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                           ~uintptr_t(127));
  double* ringA = base;                    // RING planes
  double* ringB = ringA + RING * WN;       // RING planes
  double* Ub = ringB + RING * WN;          // 2 planes (resid only)
  double* L1b = Ub + 2 * WN;               // 2 planes
  double* AAb = L1b + 2 * WN;              // 2 planes
  __shared__ uint64_t bars[RING];
  __shared__ double red[64];

  const int tid = threadIdx.x;
  const int ntx = (p.nx + TX - 1) / TX;
  const int x0 = (blockIdx.x % ntx) * TX, y0 = (blockIdx.x / ntx) * TY;
  const int z0 = blockIdx.y * p.zc;
  const int zc = min(p.zc, p.nz - z0);
  const int gx0 = x0 - HX, gy0 = y0 - HY;
  const int nx = p.nx, ny = p.ny, nz = p.nz;
  const size_t plane = (size_t)nx * ny;
  const int T = zc + 6;                    // planes streamed
  const bool edge = gx0 < 0 || gy0 < 0 || gx0 + WX > nx || gy0 + WY > ny;
  const double ih2 = p.ih2;

  // slot geometry
  int qs[NS];
  bool r3[NS], r2[NS], r1[NS], r0[NS], valid[NS];
  size_t gofs[NS];  // in-plane global offset (wrapped) of the slot
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    int q = tid + s * NT;
    valid[s] = q < WN;
    qs[s] = valid[s] ? q : 0;
    r3[s] = valid[s] && in_region(q, 3) && (OP == OP_RESID);
    r2[s] = valid[s] && in_region(q, 2);
    r1[s] = valid[s] && in_region(q, 1);
    r0[s] = valid[s] && in_region(q, 0);
    int gx = gx0 + qs[s] % WX, gy = gy0 + qs[s] / WX;
    gofs[s] = (size_t)wrapi(gx, nx) + (size_t)nx * wrapi(gy, ny);
    if (r0[s] && (gx >= nx || gy >= ny)) r0[s] = false;   // ragged tile: no output
  }

  auto issue = [&](int t) {   // TMA of streamed plane t into ring slot t % RING
    int zp = wrapi(z0 - 3 + t, nz);
    int slot = t % RING;
    mbar_expect_tx(&bars[slot], 2u * WN * sizeof(double));
    tma_load_3d(ringA + slot * WN, &ma, &bars[slot], gx0, gy0, zp);
    tma_load_3d(ringB + slot * WN, &mb, &bars[slot], gx0, gy0, zp);
  };

  if (p.use_tma) {
    if (tid == 0) {
      for (int i = 0; i < RING; ++i) mbar_init(&bars[i], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0)
      for (int t = 0; t < PREFETCH && t < T; ++t) issue(t);
  }

  // register z-queues: index 0 = oldest
  double qU[NS][3], qL[NS][3], qA[NS][3], qa[NS][4], qb[NS][4];
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i < 3) qU[s][i] = qL[s][i] = qA[s][i] = 0.0;
      qa[s][i] = qb[s][i] = 0.0;
    }
  double nrm = 0.0;

  for (int t = 0; t < T; ++t) {
    const int slot = t % RING;
    double* pa = ringA + slot * WN;
    double* pb = ringB + slot * WN;
    const int zp = wrapi(z0 - 3 + t, nz);
    if (p.use_tma) {
      if (tid == 0 && t + PREFETCH < T) issue(t + PREFETCH);
      mbar_wait(&bars[slot], (t / RING) & 1);
    }
    // own-slot inputs of plane t (wrapped reload of out-of-range cells on edge tiles)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
#pragma unroll
      for (int i = 0; i < 3; ++i) { qa[s][i] = qa[s][i + 1]; qb[s][i] = qb[s][i + 1]; }
      double va = 0.0, vb = 0.0;
      if (valid[s]) {
        if (!p.use_tma || edge) {
          int gx = gx0 + qs[s] % WX, gy = gy0 + qs[s] / WX;
          bool oob = !p.use_tma || gx < 0 || gx >= nx || gy < 0 || gy >= ny;
          if (oob) {
            size_t g = gofs[s] + plane * zp;
            va = p.a[g];
            vb = p.b[g];
            pa[qs[s]] = va;
            pb[qs[s]] = vb;
          } else {
            va = pa[qs[s]];
            vb = pb[qs[s]];
          }
        } else {
          va = pa[qs[s]];
          vb = pb[qs[s]];
        }
      }
      qa[s][3] = va;
      qb[s][3] = vb;
    }
    // generic-proxy patch writes must be ordered before later TMA writes to the same slot
    if (p.use_tma && edge) fence_proxy_async();
    double* Lin;   // plane buffer whose xy-Laplacian feeds L1(t-1)
    if (OP == OP_RESID) {
      // u(t) on halo 3
      double* Ucur = Ub + (t & 1) * WN;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        qU[s][0] = qU[s][1]; qU[s][1] = qU[s][2];
        double u = 0.5 * (qa[s][3] + qb[s][3]);
        qU[s][2] = u;
        if (r3[s]) Ucur[qs[s]] = u;
      }
      Lin = Ub + ((t - 1) & 1) * WN;
    } else {
      // v planes t-2, t-1, t live in qa[.][1..3]; xy-neighbours of plane t-1 in the ring
#pragma unroll
      for (int s = 0; s < NS; ++s) { qU[s][0] = qa[s][1]; qU[s][1] = qa[s][2]; qU[s][2] = qa[s][3]; }
      Lin = ringA + ((t + RING - 1) % RING) * WN;
    }
    __syncthreads();
    // L1(t-1) on halo 2
    if (t >= 2) {
      double* Lcur = L1b + ((t - 1) & 1) * WN;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        qL[s][0] = qL[s][1]; qL[s][1] = qL[s][2];
        double l = 0.0;
        if (r2[s]) {
          l = ih2 * (lap_xy(Lin, qs[s]) + (qU[s][0] + qU[s][2] - 2.0 * qU[s][1]) +
                     0.0);
          Lcur[qs[s]] = l;
        }
        qL[s][2] = l;
      }
    }
    __syncthreads();
    // A(t-2) | bracket(t-2) on halo 1
    if (t >= 4) {
      const double* Lp = L1b + ((t - 2) & 1) * WN;
      double* Acur = AAb + ((t - 2) & 1) * WN;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        qA[s][0] = qA[s][1]; qA[s][1] = qA[s][2];
        double aval = 0.0;
        if (r1[s]) {
          double lapL = ih2 * (lap_xy(Lp, qs[s]) + (qL[s][0] + qL[s][2] - 2.0 * qL[s][1]));
          double a = qa[s][1], b = qb[s][1];   // plane t-2
          if (OP == OP_RESID) {
            double N = 0.25 * (a * a * a + a * a * b + a * b * b + b * b * b);
            aval = (1.0 - p.gamma) * qU[s][0] + 2.0 * qL[s][1] + lapL + N;
          } else {
            aval = (0.5 * (1.0 - p.gamma) + b) * a + qL[s][1] + 0.5 * lapL;
          }
          Acur[qs[s]] = aval;
        }
        qA[s][2] = aval;
      }
    }
    __syncthreads();
    // F(t-3) on halo 0
    if (t >= 6) {
      const double* Ap = AAb + ((t - 3) & 1) * WN;
      const int zo = z0 + (t - 6);   // output plane
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        if (r0[s]) {
          double lapA = ih2 * (lap_xy(Ap, qs[s]) + (qA[s][0] + qA[s][2] - 2.0 * qA[s][1]));
          double o;
          if (OP == OP_RESID) o = (qa[s][0] - qb[s][0]) * p.idt - lapA;
          else o = qa[s][0] * p.idt - lapA;
          p.out[gofs[s] + plane * zo] = o;
          nrm += o * o;
        }
      }
    }
  }
  if (p.partials) {
    double sblk = block_sum(nrm, red);
    if (tid == 0) p.partials[blockIdx.y * gridDim.x + blockIdx.x] = sblk;
  }
}

constexpr int SMEM_BYTES = (2 * RING + 6) * WN * (int)sizeof(double) + 128;

template <int OP>
cudaError_t launch3d(pfc_ctx* ctx, const double* a, const double* b, double dt, double* out,
                     double* partials, int* nparts) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(stencil3d_kernel<OP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int nx = ctx->cfg.n[0], ny = ctx->cfg.n[1], nz = ctx->cfg.n[2];
  const int ntiles = ((nx + TX - 1) / TX) * ((ny + TY - 1) / TY);
  // z chunk: about 4 waves of 148 CTAs, 8..64 planes per chunk
  int want = (ntiles * nz) / (148 * 4);
  int zc = want < 8 ? 8 : (want > 64 ? 64 : want);
  if (zc > nz) zc = nz;
  const int nzc = (nz + zc - 1) / zc;
  S3Args p{a, b, out, partials, nx, ny, nz, zc, 1.0 / dt, ctx->cfg.gamma, ctx->ih2, 0};
  CUtensorMap ma, mb;
  memset(&ma, 0, sizeof(ma));
  memset(&mb, 0, sizeof(mb));
  const int box[3] = {WX, WY, 1};
  if (nx % 2 == 0 && nx >= WX && ny >= WY && tma_usable(a) && tma_usable(b) &&
      tma_encode(&ma, a, 3, ctx->cfg.n, box) && tma_encode(&mb, b, 3, ctx->cfg.n, box))
    p.use_tma = 1;
  dim3 grid(ntiles, nzc);
  if (nparts) *nparts = grid.x * grid.y;
  stencil3d_kernel<OP><<<grid, NT, SMEM_BYTES, ctx->stream>>>(ma, mb, p);
  ctx->launches++;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_residual_3d(pfc_ctx* ctx, const double* phi_new, const double* phi_old,
                               double dt, double* F, double* partials, int* nparts) {
  return launch3d<OP_RESID>(ctx, phi_new, phi_old, dt, F, partials, nparts);
}

cudaError_t launch_jv_3d(pfc_ctx* ctx, const double* v, const double* c, double dt,
                         double* out) {
  return launch3d<OP_JV>(ctx, v, c, dt, out, nullptr, nullptr);
}
