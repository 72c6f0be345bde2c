// mobility.cu -- variable-mobility residual and Jacobian-vector product, 2D/3D (NEXT row f3).
//
// Eq. (NSOP) P:257-263 with M_d = M((Phi+psi)/2), M(phi) = 1 - phi^2 (Test B
// variants) and (grad . M grad)_d of P:208-212 (edge midpoint value = average of
// the two end nodes):
//   F    = (Phi - psi)/dt - (grad . M grad)_d A,   A of Eq. (discretedG)
//   J v  = v/dt - (grad . M grad)_d (dA v) - (grad . (dM v) grad)_d A,
//          dA v = (1/2)[(1-gamma) + 2 Delta_d + Delta_d^2] v + c v,  dM v = -u v,
//          u = (Phi+psi)/2, c = (3Phi^2 + 2Phi psi + psi^2)/4.
// Each operator is a chain of three radius-1 kernels over global memory (neighbours through
// L1/L2): Laplacian, Laplacian + pointwise combine, divergence form.  This is the
// correctness-first path of the row (DESIGN.md §6 gives its measured rate); the periodic M = 1
// configurations run the fused single-pass stencils of stencil2d.cu / stencil3d.cu.  The same
// chain serves the Neumann-type mirror BCs (row f3, reading R23; with M = 1 too): every
// radius-1 neighbour reflects across the boundary face, which composes to the even extension.
#include "pfc_device.cuh"
#include "pfc_internal.h"

#include <algorithm>

namespace {

constexpr int NT = 256;

// bc: periodic or mirror ghosts (R23); mob: M = 1 - u^2 (else M = 1, the mirror-BC M = 1 path)
struct Grid { int nx, ny, nz, nd, mirror, mob; };

// the node q and its 2*nd neighbours (x-, x+, y-, y+, z-, z+): periodic, or mirrored across
// the boundary faces (node -1 is node 0, node n is node n-1)
struct Nb {
  size_t c, m[3], p[3];
};
__device__ __forceinline__ Nb nbrs(size_t q, const Grid& G) {
  const size_t nxy = (size_t)G.nx * G.ny;
  const int i = (int)(q % G.nx), j = (int)((q / G.nx) % G.ny), k = (int)(q / nxy);
  const int im = i == 0 ? (G.mirror ? 0 : G.nx - 1) : i - 1;
  const int ip = i + 1 == G.nx ? (G.mirror ? i : 0) : i + 1;
  const int jm = j == 0 ? (G.mirror ? 0 : G.ny - 1) : j - 1;
  const int jp = j + 1 == G.ny ? (G.mirror ? j : 0) : j + 1;
  const int km = k == 0 ? (G.mirror ? 0 : G.nz - 1) : k - 1;
  const int kp = k + 1 == G.nz ? (G.mirror ? k : 0) : k + 1;
  const size_t row = (size_t)G.nx * j + nxy * k;
  Nb n;
  n.c = q;
  n.m[0] = row + im; n.p[0] = row + ip;
  n.m[1] = (size_t)G.nx * jm + nxy * k + i; n.p[1] = (size_t)G.nx * jp + nxy * k + i;
  n.m[2] = (size_t)G.nx * j + nxy * km + i; n.p[2] = (size_t)G.nx * j + nxy * kp + i;
  return n;
}
template <class F>
__device__ __forceinline__ double lapf(const F& f, const Nb& n, int nd, double ih2) {
  double s = 0.0;
  for (int d = 0; d < nd; ++d) s += f(n.m[d]) + f(n.p[d]);
  return ih2 * (s - 2.0 * nd * f(n.c));
}

// L = Delta_d f, where f = (a + b) * s (a 2-field average when b != nullptr, s = 1/2)
__global__ void k_lap(const double* __restrict__ a, const double* __restrict__ b, double s,
                      double* __restrict__ L, Grid G, double ih2) {
  const size_t N = (size_t)G.nx * G.ny * G.nz;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < N;
       q += (size_t)gridDim.x * blockDim.x) {
    const Nb n = nbrs(q, G);
    auto f = [&](size_t k) { return b ? (a[k] + b[k]) * s : a[k]; };
    L[q] = lapf(f, n, G.nd, ih2);
  }
}

// residual / state: A = (1-gamma) u + 2 L1 + Delta L1 + (Phi^3 + Phi^2 psi + Phi psi^2 + psi^3)/4
// J v:              dA = (1/2)[(1-gamma) v + 2 L1 + Delta L1] + c v
template <bool JV>
__global__ void k_combine(const double* __restrict__ a, const double* __restrict__ b,
                          const double* __restrict__ L1, double* __restrict__ out, Grid G,
                          double ih2, double gamma) {
  const size_t N = (size_t)G.nx * G.ny * G.nz;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < N;
       q += (size_t)gridDim.x * blockDim.x) {
    const Nb n = nbrs(q, G);
    const size_t c = q;
    const double LL = lapf([&](size_t k) { return L1[k]; }, n, G.nd, ih2);
    if (JV) {            // a = v, b = c
      out[c] = 0.5 * ((1.0 - gamma) * a[c] + 2.0 * L1[c] + LL) + b[c] * a[c];
    } else {             // a = Phi, b = psi
      const double p = a[c], s = b[c];
      out[c] = (1.0 - gamma) * 0.5 * (p + s) + 2.0 * L1[c] + LL +
               0.25 * (p * p * p + p * p * s + p * s * s + s * s * s);
    }
  }
}

// (grad . M grad)_d g at node n.c, M given by the function m(k)
template <class MF>
__device__ __forceinline__ double div_mgrad(const MF& m, const double* __restrict__ g, const Nb& n,
                                            int nd, double ih2) {
  const double mc = m(n.c), gc = g[n.c];
  double s = 0.0;
  for (int d = 0; d < nd; ++d)
    s += 0.5 * (mc + m(n.p[d])) * (g[n.p[d]] - gc) - 0.5 * (mc + m(n.m[d])) * (gc - g[n.m[d]]);
  return ih2 * s;
}

// residual: F = (Phi - psi)/dt - (grad . M grad) A, M = 1 - u^2; fixed-grid per-block ||F||^2
__global__ void k_resid_out(const double* __restrict__ phi, const double* __restrict__ psi,
                            const double* __restrict__ A, double* __restrict__ F,
                            double* __restrict__ partials, Grid G, double ih2, double idt_h,
                            const double* dtp) {
  __shared__ double red[64];
  const double idt = dt_inv(dtp, idt_h);
  const size_t N = (size_t)G.nx * G.ny * G.nz;
  auto m = [&](size_t k) {
    const double u = 0.5 * (phi[k] + psi[k]);
    return G.mob ? 1.0 - u * u : 1.0;
  };
  double nrm = 0.0;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < N;
       q += (size_t)gridDim.x * blockDim.x) {
    const Nb n = nbrs(q, G);
    const double o = (phi[q] - psi[q]) * idt - div_mgrad(m, A, n, G.nd, ih2);
    F[q] = o;
    nrm += o * o;
  }
  if (partials) {
    const double s = block_sum(nrm, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
  }
}

// J v = v/dt - (grad . M grad) dA - (grad . (-u v) grad) A
__global__ void k_jv_out(const double* __restrict__ v, const double* __restrict__ dA,
                         const double* __restrict__ phi, const double* __restrict__ psi,
                         const double* __restrict__ A, double* __restrict__ out, Grid G,
                         double ih2, double idt_h, const int* gate, const double* dtp) {
  if (gate && *gate) return;
  const double idt = dt_inv(dtp, idt_h);
  const size_t N = (size_t)G.nx * G.ny * G.nz;
  auto m = [&](size_t k) {
    const double u = 0.5 * (phi[k] + psi[k]);
    return G.mob ? 1.0 - u * u : 1.0;
  };
  auto dm = [&](size_t k) { return -0.5 * (phi[k] + psi[k]) * v[k]; };
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < N;
       q += (size_t)gridDim.x * blockDim.x) {
    const Nb n = nbrs(q, G);
    double o = v[q] * idt - div_mgrad(m, dA, n, G.nd, ih2);
    if (G.mob) o -= div_mgrad(dm, A, n, G.nd, ih2);   // M = 1: no mobility-derivative term
    out[q] = o;
  }
}

int grid_for(size_t N) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0, v = 0;
    nsm = (cudaGetDevice(&dev) == cudaSuccess &&
           cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
              ? v : 148;
  }
  const size_t want = (N + NT - 1) / NT;
  return (int)std::min<size_t>(want, (size_t)nsm * 8);   // fixed for a given N: deterministic
}

// A(Phi, psi) into `A` through the work field t0
Grid grid_of(const pfc_ctx* ctx) {
  const pfc_config& c = ctx->cfg;
  return Grid{c.n[0], c.n[1], c.ndim == 3 ? c.n[2] : 1, c.ndim, c.bc == PFC_BC_MIRROR,
              c.mobility == PFC_MOBILITY_QUADRATIC};
}

cudaError_t a_field(pfc_ctx* ctx, const double* phi, const double* psi, double* A, double* t0) {
  const Grid G = grid_of(ctx);
  const int g = grid_for(ctx->N);
  k_lap<<<g, NT, 0, ctx->stream>>>(phi, psi, 0.5, t0, G, ctx->ih2);
  k_combine<false><<<g, NT, 0, ctx->stream>>>(phi, psi, t0, A, G, ctx->ih2, ctx->cfg.gamma);
  ctx->launches += 2;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_mob_state(pfc_ctx* ctx, const double* phi, const double* psi) {
  ctx->mob_phi = phi;
  ctx->mob_psi = psi;
  cudaError_t e = a_field(ctx, phi, psi, ctx->mob_A, ctx->mob_t[0]);
  pfc_account(ctx, PFC_K_COEF, 48.0 * ctx->N, 30.0 * ctx->N);
  return e;
}

cudaError_t launch_residual_mob(pfc_ctx* ctx, const double* phi, const double* psi, double dt,
                                double* F, double* partials, int* nparts) {
  const Grid G = grid_of(ctx);
  cudaError_t e = a_field(ctx, phi, psi, ctx->mob_t[1], ctx->mob_t[0]);
  if (e != cudaSuccess) return e;
  const int g = grid_for(ctx->N);
  k_resid_out<<<g, NT, 0, ctx->stream>>>(phi, psi, ctx->mob_t[1], F, partials, G, ctx->ih2,
                                          1.0 / dt, ctx->dtdev);
  ctx->launches++;
  if (nparts) *nparts = g;
  // algorithmic: Phi, psi in, F out (the two intermediate fields are work of this path)
  pfc_account(ctx, PFC_K_RESIDUAL, 24.0 * ctx->N, 50.0 * ctx->N);
  return cudaGetLastError();
}

cudaError_t launch_jv_mob(pfc_ctx* ctx, const double* v, const double* c, double dt,
                          double* out) {
  const Grid G = grid_of(ctx);
  const int g = grid_for(ctx->N);
  // device-resident FGMRES (f1): only the final write is gated; the two producer kernels
  // run unconditionally into work fields nobody reads when the gate is set
  k_lap<<<g, NT, 0, ctx->stream>>>(v, nullptr, 1.0, ctx->mob_t[0], G, ctx->ih2);
  k_combine<true><<<g, NT, 0, ctx->stream>>>(v, c, ctx->mob_t[0], ctx->mob_t[1], G, ctx->ih2,
                                             ctx->cfg.gamma);
  k_jv_out<<<g, NT, 0, ctx->stream>>>(v, ctx->mob_t[1], ctx->mob_phi, ctx->mob_psi, ctx->mob_A,
                                       out, G, ctx->ih2, 1.0 / dt, ctx->gate, ctx->dtdev);
  ctx->launches += 3;
  pfc_account(ctx, PFC_K_JV, 24.0 * ctx->N, 45.0 * ctx->N);
  return cudaGetLastError();
}
