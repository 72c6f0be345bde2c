// stencil3d.cu -- fused 3D DVD residual (K1) and Jacobian-vector product (K2), sm_100a.
//
// Same operators as stencil2d.cu (Eq. NSOP, Eq. discretedG, Eq. Jacobi
// P:351-356), the 7-point Delta_d composed three times: a radius-3, 63-point stencil.
//
// 2.5D z-march.  A CTA (1024 threads, one per SM) owns a TX x TY column of outputs and a chunk
// of ZC z-planes.  Input planes z0-3 .. z0+ZC+2 stream through an 8-slot ring per field filled
// by TMA (cp.async.bulk.tensor.3d, one (TX+8) x (TY+6) x 1 box per field and plane, 4 planes in
// flight, one mbarrier per slot).  Every thread owns ONE fixed position of the 40 x 22 plane
// window for all stages and keeps its z-neighbours in registers; at streamed plane t it computes
//     u(t) [halo 3]  ->  L1(t-1) [halo 2]  ->  A(t-2) [halo 1]  ->  F(t-3) [halo 0]
// taking xy-neighbours from one shared-memory plane per stage (double-buffered).  Two
// barriers per plane.  Periodic x/y wrap: TMA zero-fills out-of-range cells and edge tiles
// reload exactly those cells with wrapped loads; z wraps incrementally.  Optional fused
// ||F||^2 partial per CTA.
#include "pfc_device.cuh"
#include "pfc_internal.h"

namespace {

constexpr int TX = 32, TY = 16;
constexpr int HX = 4, HY = 3;
constexpr int WX = TX + 2 * HX;   // 40
constexpr int WY = TY + 2 * HY;   // 22
constexpr int WN = WX * WY;       // 880
constexpr int NT = 1024;
constexpr int RING = 8;           // power of two
constexpr int PREFETCH = 4;

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
  double* L1b = ringB + RING * WN;         // 2 planes
  double* AAb = L1b + 2 * WN;              // 2 planes
  double* Ub = AAb + 2 * WN;               // 2 planes (resid only)
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

  // this thread's window position and its stage memberships
  const int q = tid < WN ? tid : 0;
  const bool valid = tid < WN;
  const int qx = q % WX, qy = q / WX;
  auto inr = [&](int r) {
    return valid && qx >= HX - r && qx < HX + TX + r && qy >= HY - r && qy < HY + TY + r;
  };
  const bool r3 = inr(3) && OP == OP_RESID, r2 = inr(2), r1 = inr(1);
  const int gx = gx0 + qx, gy = gy0 + qy;
  const bool r0 = inr(0) && gx < nx && gy < ny;                 // ragged tiles: no output
  const bool reload = valid && (!p.use_tma || (edge && (gx < 0 || gx >= nx || gy < 0 || gy >= ny)));
  const size_t gofs = (size_t)wrapi(gx, nx) + (size_t)nx * wrapi(gy, ny);

  const int zfirst = wrapi(z0 - 3, nz);
  if (p.use_tma) {
    if (tid == 0) {
      for (int i = 0; i < RING; ++i) mbar_init(&bars[i], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
      int zi = zfirst;
      for (int t = 0; t < PREFETCH && t < T; ++t) {
        const int slot = t & (RING - 1);
        mbar_expect_tx(&bars[slot], 2u * WN * sizeof(double));
        tma_load_3d(ringA + slot * WN, &ma, &bars[slot], gx0, gy0, zi);
        tma_load_3d(ringB + slot * WN, &mb, &bars[slot], gx0, gy0, zi);
        zi = (zi + 1 == nz) ? 0 : zi + 1;
      }
    }
  }
  int zpre = wrapi(z0 - 3 + PREFETCH, nz);   // plane of the next TMA issue
  int zcur = zfirst;                          // plane t

  // register z-queues of this thread's position: [0] oldest
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;      // input A (Phi | v) planes t-3..t
  double b0 = 0, b1 = 0, b2 = 0, b3 = 0;      // input B (psi | c) planes t-3..t
  double u0 = 0, u1 = 0, u2 = 0;              // u planes t-2..t (resid)
  double l0 = 0, l1 = 0, l2 = 0;              // L1 planes t-3..t-1
  double A0 = 0, A1 = 0, A2 = 0;              // A planes t-4..t-2
  double nrm = 0.0;
  double* outp = p.out + gofs + plane * (size_t)z0;

#pragma unroll 2
  for (int t = 0; t < T; ++t) {
    const int slot = t & (RING - 1);
    double* pa = ringA + slot * WN;
    double* pb = ringB + slot * WN;
    if (p.use_tma) {
      if (tid == 0 && t + PREFETCH < T) {
        const int ps = (t + PREFETCH) & (RING - 1);
        mbar_expect_tx(&bars[ps], 2u * WN * sizeof(double));
        tma_load_3d(ringA + ps * WN, &ma, &bars[ps], gx0, gy0, zpre);
        tma_load_3d(ringB + ps * WN, &mb, &bars[ps], gx0, gy0, zpre);
      }
      zpre = (zpre + 1 == nz) ? 0 : zpre + 1;
      mbar_wait(&bars[slot], (t / RING) & 1);
    }
    // own inputs of plane t
    double va = 0.0, vb = 0.0;
    if (valid) {
      if (reload) {
        const size_t g = gofs + plane * zcur;
        va = p.a[g];
        vb = p.b[g];
        pa[q] = va;
        pb[q] = vb;
        if (p.use_tma) fence_proxy_async();   // generic write before a later TMA overwrite
      } else {
        va = pa[q];
        vb = pb[q];
      }
    }
    zcur = (zcur + 1 == nz) ? 0 : zcur + 1;
    a0 = a1; a1 = a2; a2 = a3; a3 = va;
    b0 = b1; b1 = b2; b2 = b3; b3 = vb;
    const double* Lin;                         // plane whose xy-Laplacian feeds L1(t-1)
    if (OP == OP_RESID) {
      u0 = u1; u1 = u2; u2 = 0.5 * (va + vb);
      if (r3) Ub[(t & 1) * WN + q] = u2;
      Lin = Ub + ((t - 1) & 1) * WN;
    } else {
      u0 = a1; u1 = a2; u2 = a3;              // v planes t-2, t-1, t
      Lin = ringA + ((t - 1) & (RING - 1)) * WN;
    }
    // L1(t-1) on halo 2: xy-neighbours of plane t-1 were completed before the previous
    // iteration's barriers
    if (t >= 2) {
      l0 = l1; l1 = l2;
      double l = 0.0;
      if (r2) {
        l = ih2 * (lap_xy(Lin, q) + (u0 + u2 - 2.0 * u1));
        L1b[((t - 1) & 1) * WN + q] = l;
      }
      l2 = l;
    }
    __syncthreads();
    // A(t-2) | bracket(t-2) on halo 1
    if (t >= 4) {
      A0 = A1; A1 = A2;
      double av = 0.0;
      if (r1) {
        const double lapL = ih2 * (lap_xy(L1b + ((t - 2) & 1) * WN, q) + (l0 + l2 - 2.0 * l1));
        const double a = a1, b = b1;           // plane t-2
        if (OP == OP_RESID) {
          const double N = 0.25 * (a * a * a + a * a * b + a * b * b + b * b * b);
          av = (1.0 - p.gamma) * u0 + 2.0 * l1 + lapL + N;
        } else {
          av = (0.5 * (1.0 - p.gamma) + b) * a + l1 + 0.5 * lapL;
        }
        AAb[((t - 2) & 1) * WN + q] = av;
      }
      A2 = av;
    }
    __syncthreads();
    // F(t-3) on halo 0
    if (t >= 6 && r0) {
      const double lapA = ih2 * (lap_xy(AAb + ((t - 3) & 1) * WN, q) + (A0 + A2 - 2.0 * A1));
      double o;
      if (OP == OP_RESID) o = (a0 - b0) * p.idt - lapA;
      else o = a0 * p.idt - lapA;
      *outp = o;
      outp += plane;
      nrm += o * o;
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
  pfc_account(ctx, OP == OP_RESID ? PFC_K_RESIDUAL : PFC_K_JV, 24.0 * ctx->N,
              (OP == OP_RESID ? 42.0 : 31.0) * ctx->N);
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
