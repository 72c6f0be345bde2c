// stencil2d.cu -- fused 2D DVD residual (K1) and Jacobian-vector product (K2), sm_100a.
//
// Residual, Eq. (NSOP) P:257-263 with M = 1, and A from Eq. (discretedG) P:250-255:
//   F = (Phi - psi)/dt - Delta_d[(1-gamma)u + 2 Delta_d u + Delta_d^2 u + N(Phi,psi)],
//   u = (Phi+psi)/2, N = (Phi^3 + Phi^2 psi + Phi psi^2 + psi^3)/4.
// Jacobian (Eq. Jacobi):
//   Jv = v/dt - Delta_d[(1/2)(1-gamma)v + c v + Delta_d v + (1/2) Delta_d^2 v].
// Delta_d (1+Delta_d)^2 is a radius-3 stencil ("3 is the stencil width"), applied
// here by composing three 5-point Laplacians inside shared memory.
//
// One CTA computes a TX x TY output tile.  Its (TX+8) x (TY+6) input window (halo 3, plus
// one slack column per side so rows are 16-byte multiples) is staged into shared memory by
// one TMA tile load per field (cp.async.bulk.tensor.2d, mbarrier completion).  TMA has no
// periodic mode: out-of-range cells arrive zero-filled and edge tiles overwrite exactly those
// cells with wrapped loads.  Then three in-SMEM stages shrink the halo 3 -> 2 -> 1 -> 0.
// Optional fused ||F||^2 partial per tile (deterministic, finalized in fixed order).
#include "pfc_device.cuh"
#include "pfc_internal.h"

namespace {

constexpr int TX = 32, TY = 16;          // output tile
constexpr int HX = 4, HY = 3;            // loaded halo (x: 3 + 1 slack for 16-B rows)
constexpr int WX = TX + 2 * HX;          // 40
constexpr int WY = TY + 2 * HY;          // 22
constexpr int WN = WX * WY;
constexpr int NT = 256;

enum { OP_RESID = 0, OP_JV = 1 };

struct S2Args {
  const double* a;   // Phi (resid) | v (jv)
  const double* b;   // psi (resid) | c (jv)
  double* out;
  double* partials;  // per-tile ||out||^2 or nullptr
  int nx, ny;
  double idt, gamma, ih2;
  int use_tma;
  const int* gate;   // device-resident FGMRES: skip the launch when *gate != 0 (f1)
};

__device__ __forceinline__ double lap5(const double* f, int q, double ih2) {
  return ih2 * ((f[q - 1] + f[q + 1]) + (f[q - WX] + f[q + WX]) - 4.0 * f[q]);
}

template <int OP>
__global__ void __launch_bounds__(NT) stencil2d_kernel(const __grid_constant__ CUtensorMap ma,
                                                       const __grid_constant__ CUtensorMap mb,
                                                       S2Args p) {
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
    if (OP == OP_RESID) o = (A0[f] - B0[f]) * p.idt - lap5(AA, f, ih2);
    else o = A0[f] * p.idt - lap5(AA, f, ih2);
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
cudaError_t launch2d(pfc_ctx* ctx, const double* a, const double* b, double dt, double* out,
                     double* partials, int* nparts) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(stencil2d_kernel<OP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int nx = ctx->cfg.n[0], ny = ctx->cfg.n[1];
  S2Args p{a, b, out, partials, nx, ny, 1.0 / dt, ctx->cfg.gamma, ctx->ih2, 0,
           OP == OP_JV ? ctx->gate : nullptr};
  CUtensorMap ma, mb;
  memset(&ma, 0, sizeof(ma));
  memset(&mb, 0, sizeof(mb));
  const int box[2] = {WX, WY};
  if (nx % 2 == 0 && nx >= WX && ny >= WY && tma_usable(a) && tma_usable(b) &&
      tma_encode(&ma, a, 2, ctx->cfg.n, box) && tma_encode(&mb, b, 2, ctx->cfg.n, box))
    p.use_tma = 1;
  dim3 grid((nx + TX - 1) / TX, (ny + TY - 1) / TY);
  if (nparts) *nparts = grid.x * grid.y;
  stencil2d_kernel<OP><<<grid, NT, SMEM_BYTES, ctx->stream>>>(ma, mb, p);
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
