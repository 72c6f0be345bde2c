// energy.cu -- discrete free energy and mass (K8), sm_100a.
//
// G_d = (1-gamma)/2 phi^2 + phi^4/4 + (Delta_d phi)^2/2 - sum_axis ((D+phi)^2 + (D-phi)^2)/2
// (Eq. relations), F_d = h^d sum G_d (Eq. freeenergy), M = h^d sum phi
// (P:276-277).  Radius-1 stencil read straight from global memory (L1/L2 serve the 5/7
// neighbour re-reads); a fixed grid with a fixed per-thread index set, then a fixed-order
// two-stage reduction, so the scalars are bitwise reproducible.  8 B/pt algorithmic.
// Periodic neighbours, or mirror ghosts (bc = PFC_BC_MIRROR, reading R23: node -1 is node 0,
// node n is node n-1, so D+ / D- vanish across the boundary faces).
#include "pfc_device.cuh"
#include "pfc_internal.h"

namespace {
constexpr int NT = 256;

template <int ND>
__global__ void __launch_bounds__(NT) k_energy_mass(const double* __restrict__ f, int nx, int ny,
                                                    int nz, double gamma, double ih, int mirror,
                                                    double* __restrict__ partials) {
  __shared__ double red[64];
  __shared__ double outv[2];
  const size_t N = (size_t)nx * ny * nz;
  double acc[2] = {0.0, 0.0};
  for (size_t q = blockIdx.x * (size_t)NT + threadIdx.x; q < N; q += (size_t)gridDim.x * NT) {
    int i = (int)(q % nx);
    size_t r = q / nx;
    int j = (int)(r % ny);
    int k = (int)(r / ny);
    double p = f[q];
    size_t rowb = q - i;
    double xm = f[rowb + (i == 0 ? (mirror ? 0 : nx - 1) : i - 1)];
    double xp = f[rowb + (i == nx - 1 ? (mirror ? nx - 1 : 0) : i + 1)];
    size_t pl = (size_t)k * nx * ny;
    double ym = f[pl + (size_t)(j == 0 ? (mirror ? 0 : ny - 1) : j - 1) * nx + i];
    double yp = f[pl + (size_t)(j == ny - 1 ? (mirror ? ny - 1 : 0) : j + 1) * nx + i];
    double lap = (xp - 2.0 * p + xm) + (yp - 2.0 * p + ym);
    double dxp = (xp - p) * ih, dxm = (p - xm) * ih, dyp = (yp - p) * ih, dym = (p - ym) * ih;
    double grad = 0.5 * (dxp * dxp + dxm * dxm) + 0.5 * (dyp * dyp + dym * dym);
    if (ND == 3) {
      size_t col = (size_t)j * nx + i, pls = (size_t)nx * ny;
      double zm = f[(size_t)(k == 0 ? (mirror ? 0 : nz - 1) : k - 1) * pls + col];
      double zp = f[(size_t)(k == nz - 1 ? (mirror ? nz - 1 : 0) : k + 1) * pls + col];
      lap += zp - 2.0 * p + zm;
      double dzp = (zp - p) * ih, dzm = (p - zm) * ih;
      grad += 0.5 * (dzp * dzp + dzm * dzm);
    }
    lap *= ih * ih;
    acc[0] += 0.5 * (1.0 - gamma) * p * p + 0.25 * p * p * p * p + 0.5 * lap * lap - grad;
    acc[1] += p;
  }
  block_sum_multi<2>(acc, red, outv);
  if (threadIdx.x < 2) partials[blockIdx.x * 2 + threadIdx.x] = outv[threadIdx.x];
}
}  // namespace

cudaError_t launch_energy_mass(pfc_ctx* ctx, const double* phi, double* partials, int* nparts) {
  const int nb = blas_nblocks(ctx->N);
  const int* n = ctx->cfg.n;
  const double ih = 1.0 / ctx->cfg.h;
  const int mir = ctx->cfg.bc == PFC_BC_MIRROR;
  if (ctx->cfg.ndim == 2)
    k_energy_mass<2><<<nb, NT, 0, ctx->stream>>>(phi, n[0], n[1], 1, ctx->cfg.gamma, ih, mir,
                                                 partials);
  else
    k_energy_mass<3><<<nb, NT, 0, ctx->stream>>>(phi, n[0], n[1], n[2], ctx->cfg.gamma, ih, mir,
                                                 partials);
  ctx->launches++;
  pfc_account(ctx, PFC_K_ENERGY, 8.0 * ctx->N, 25.0 * ctx->N);
  *nparts = nb;
  return cudaGetLastError();
}
