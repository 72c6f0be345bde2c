// krylov.cu -- HBM-bound pointwise and Krylov kernels (K3, K5-K7, K9), sm_100a.
//
// Classical Gram-Schmidt applied twice (CGS2) for the FGMRES Arnoldi step:
//   pass 1: h1 = V^T w                                    (k_multidot)
//   fused : w <- w - V h1 ; h2 = V^T w                     (k_axpy_dot: V read once for both)
//   fused : w <- w - V h2 ; |w|^2                          (k_axpy_norm)
// Reductions are deterministic: a FIXED grid (blas_nblocks(N)) with grid-stride loops, a
// per-block shuffle + shared-memory tree in fixed order, then the last block to finish sums the
// per-block partials in fixed order (finalize_last_block; k_finalize for the stencil partials).
// Results are bitwise reproducible run to run.
#include "pfc_device.cuh"
#include "pfc_internal.h"
#include "gmres_close.cuh"

namespace {

constexpr int NT = 256;

// Fused fixed-order finalisation: after every block has written its NV partials, the LAST block
// to finish (atomic ticket; it decides only WHO sums, not the order) adds the partials of all
// blocks in the same order k_finalize uses (thread-strided over blocks, then the block tree),
// so the result is bitwise identical to a separate k_finalize launch, without the launch.
template <int NV>
__device__ __forceinline__ bool finalize_last_block(const double* partials, double* out,
                                                    unsigned int* ticket, double* red,
                                                    double* outv) {
  __shared__ unsigned int last;
  __threadfence();                       // this block's partials before the ticket
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += NT) {
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] += __ldcg(partials + (size_t)b * NV + k);
  }
  block_sum_multi<NV>(acc, red, outv);
  if (threadIdx.x < NV) out[threadIdx.x] = outv[threadIdx.x];
  if (threadIdx.x == 0) *ticket = 0u;    // ready for the next reduction on this stream
  return true;
}

__device__ __forceinline__ double2 ld2g(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}

struct Coef {
  double c[PFC_MAX_RESTART];
};

__global__ void k_coef(const double* __restrict__ phi, const double* __restrict__ psi,
                       double* __restrict__ c, size_t N) {
  // J coefficient dN/dPhi = (3 Phi^2 + 2 Phi psi + psi^2)/4 (derivative of Eq. discretedG)
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x) {
    double a = phi[i], b = psi[i];
    c[i] = 0.25 * (3.0 * a * a + 2.0 * a * b + b * b);
  }
}

__global__ void k_axpby(double a, const double* x, double b, const double* y, double* out,
                        size_t N) {   // out may alias x or y (elementwise)
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x) {
    double yi = y ? y[i] : 0.0;
    out[i] = a * x[i] + b * yi;
  }
}

template <int NV>
__global__ void __launch_bounds__(NT) k_multidot(const double* __restrict__ V, size_t ldv,
                                                 const double* __restrict__ w, size_t N,
                                                 double* __restrict__ partials,
                                                 double* __restrict__ out,
                                                 unsigned int* __restrict__ ticket,
                                                 const int* __restrict__ gate) {
  if (gate && *gate) return;
  __shared__ double red[32 * NV];
  __shared__ double outv[NV];
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  if ((N & 1) == 0) {   // 16-byte pairs (N even: every column of V starts 16-byte aligned)
    const size_t N2 = N >> 1;
    for (size_t q = blockIdx.x * (size_t)NT + threadIdx.x; q < N2; q += (size_t)gridDim.x * NT) {
      const double2 wi = ld2g(w + 2 * q);
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const double2 v = ld2g(V + k * ldv + 2 * q);
        acc[k] = fma(v.y, wi.y, fma(v.x, wi.x, acc[k]));
      }
    }
  } else {
    for (size_t i = blockIdx.x * (size_t)NT + threadIdx.x; i < N; i += (size_t)gridDim.x * NT) {
      double wi = w[i];
#pragma unroll
      for (int k = 0; k < NV; ++k) acc[k] += V[k * ldv + i] * wi;
    }
  }
  block_sum_multi<NV>(acc, red, outv);
  if (threadIdx.x < NV) partials[blockIdx.x * NV + threadIdx.x] = outv[threadIdx.x];
  finalize_last_block<NV>(partials, out, ticket, red, outv);
}

template <int NV>
__global__ void __launch_bounds__(NT) k_axpy_dot(const double* __restrict__ V, size_t ldv,
                                                 const double* __restrict__ h,
                                                 double* __restrict__ w, size_t N,
                                                 double* __restrict__ partials,
                                                 double* __restrict__ out,
                                                 unsigned int* __restrict__ ticket,
                                                 const int* __restrict__ gate) {
  if (gate && *gate) return;
  __shared__ double red[32 * NV];
  __shared__ double outv[NV];
  double hk[NV], acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) { hk[k] = h[k]; acc[k] = 0.0; }
  if ((N & 1) == 0) {
    const size_t N2 = N >> 1;
    for (size_t q = blockIdx.x * (size_t)NT + threadIdx.x; q < N2; q += (size_t)gridDim.x * NT) {
      double2 v[NV];
      double2 wi = ld2g(w + 2 * q);
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        v[k] = ld2g(V + k * ldv + 2 * q);
        wi.x -= hk[k] * v[k].x;
        wi.y -= hk[k] * v[k].y;
      }
      *reinterpret_cast<double2*>(w + 2 * q) = wi;
#pragma unroll
      for (int k = 0; k < NV; ++k) acc[k] = fma(v[k].y, wi.y, fma(v[k].x, wi.x, acc[k]));
    }
  } else {
    for (size_t i = blockIdx.x * (size_t)NT + threadIdx.x; i < N; i += (size_t)gridDim.x * NT) {
      double v[NV];
      double wi = w[i];
#pragma unroll
      for (int k = 0; k < NV; ++k) { v[k] = V[k * ldv + i]; wi -= hk[k] * v[k]; }
      w[i] = wi;
#pragma unroll
      for (int k = 0; k < NV; ++k) acc[k] += v[k] * wi;
    }
  }
  block_sum_multi<NV>(acc, red, outv);
  if (threadIdx.x < NV) partials[blockIdx.x * NV + threadIdx.x] = outv[threadIdx.x];
  finalize_last_block<NV>(partials, out, ticket, red, outv);
}

template <int NV>
__global__ void __launch_bounds__(NT) k_axpy_norm(const double* __restrict__ V, size_t ldv,
                                                  const double* __restrict__ h,
                                                  double* __restrict__ w, size_t N,
                                                  double* __restrict__ partials,
                                                  double* __restrict__ out,
                                                  unsigned int* __restrict__ ticket,
                                                  pfc_gmres_dev* __restrict__ gm,
                                                  const double* __restrict__ h1) {
  if (gm && gm->stop) return;
  __shared__ double red[32];
  __shared__ double outv[1];
  double hk[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) hk[k] = h[k];
  double acc[1] = {0.0};
  if ((N & 1) == 0) {
    const size_t N2 = N >> 1;
    for (size_t q = blockIdx.x * (size_t)NT + threadIdx.x; q < N2; q += (size_t)gridDim.x * NT) {
      double2 wi = ld2g(w + 2 * q);
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const double2 v = ld2g(V + k * ldv + 2 * q);
        wi.x -= hk[k] * v.x;
        wi.y -= hk[k] * v.y;
      }
      *reinterpret_cast<double2*>(w + 2 * q) = wi;
      acc[0] = fma(wi.y, wi.y, fma(wi.x, wi.x, acc[0]));
    }
  } else {
    for (size_t i = blockIdx.x * (size_t)NT + threadIdx.x; i < N; i += (size_t)gridDim.x * NT) {
      double wi = w[i];
#pragma unroll
      for (int k = 0; k < NV; ++k) wi -= hk[k] * V[k * ldv + i];
      w[i] = wi;
      acc[0] += wi * wi;
    }
  }
  block_sum_multi<1>(acc, red, outv);
  if (threadIdx.x == 0) partials[blockIdx.x] = outv[0];
  const bool last = finalize_last_block<1>(partials, out, ticket, red, outv);
  if (gm && last && threadIdx.x == 0) arnoldi_close(gm, NV - 1, h1, h, outv[0]);
}

__global__ void __launch_bounds__(NT) k_norm2(const double* __restrict__ x, size_t N,
                                              double* __restrict__ partials,
                                              double* __restrict__ out,
                                              unsigned int* __restrict__ ticket) {
  __shared__ double red[32];
  __shared__ double outv[1];
  double acc[1] = {0.0};
  for (size_t i = blockIdx.x * (size_t)NT + threadIdx.x; i < N; i += (size_t)gridDim.x * NT)
    acc[0] += x[i] * x[i];
  block_sum_multi<1>(acc, red, outv);
  if (threadIdx.x == 0) partials[blockIdx.x] = outv[0];
  finalize_last_block<1>(partials, out, ticket, red, outv);
}

// out[v] = sum_b partials[b*nval + v], fixed order; one CTA per value
__global__ void __launch_bounds__(NT) k_finalize(const double* __restrict__ partials, int nblk,
                                                 int nval, double* __restrict__ out) {
  __shared__ double red[32];
  __shared__ double outv[1];
  const int v = blockIdx.x;
  double acc[1] = {0.0};
  for (int b = threadIdx.x; b < nblk; b += NT) acc[0] += partials[(size_t)b * nval + v];
  block_sum_multi<1>(acc, red, outv);
  if (threadIdx.x == 0) out[v] = outv[0];
}

template <int NV>
__global__ void __launch_bounds__(NT) k_lincomb(double* __restrict__ x,
                                                const double* __restrict__ Z, size_t ldz,
                                                Coef coef, size_t N) {
  for (size_t i = blockIdx.x * (size_t)NT + threadIdx.x; i < N; i += (size_t)gridDim.x * NT) {
    double s = x[i];
#pragma unroll
    for (int k = 0; k < NV; ++k) s += coef.c[k] * Z[k * ldz + i];
    x[i] = s;
  }
}

// V_{j+1} = w / h_{j+1,j} (skipped when the cycle stopped at step j)
__global__ void k_scale_next(const pfc_gmres_dev* __restrict__ gm, const double* __restrict__ w,
                             double* __restrict__ vnext, size_t N) {
  if (gm->stop) return;
  const double ihn = gm->ihn;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x)
    vnext[i] = ihn * w[i];
}

__global__ void k_cycle_init(pfc_gmres_dev* gm, double beta, double tol, int m, int maxit,
                             int its_done) {
  gm->beta = beta;
  gm->tol = tol;
  gm->m = m;
  gm->maxit = maxit;
  gm->its = its_done;
  gm->jm = 0;
  gm->reason = PFC_GM_RUNNING;
  gm->stop = 0;
  gm->graph = 0;
  for (int i = 0; i <= m; ++i) gm->g[i] = 0.0;
  gm->g[0] = beta;
}

// y = R^{-1} g (back substitution, the host loop's order and roundings) by one thread ...
__global__ void k_backsolve(pfc_gmres_dev* gm) {
  const int jm = gm->jm, ld = gm->m + 1;
  for (int i = jm - 1; i >= 0; --i) {
    double s = gm->g[i];
    for (int l = i + 1; l < jm; ++l) s = __dsub_rn(s, __dmul_rn(gm->H[i + ld * l], gm->y[l]));
    gm->y[i] = s / gm->H[i + ld * i];
  }
}

// ... then x += Z y over the jm columns of the cycle (FGMRES: solution from Z)
__global__ void __launch_bounds__(NT) k_lincomb_dev(double* __restrict__ x,
                                                    const double* __restrict__ Z, size_t ldz,
                                                    const pfc_gmres_dev* __restrict__ gm,
                                                    size_t N) {
  __shared__ double yk[PFC_MAX_RESTART];
  const int jm = gm->jm;
  if (threadIdx.x < jm) yk[threadIdx.x] = gm->y[threadIdx.x];
  __syncthreads();
  for (size_t i = blockIdx.x * (size_t)NT + threadIdx.x; i < N; i += (size_t)gridDim.x * NT) {
    double s = x[i];
    for (int k = 0; k < jm; ++k) s += yk[k] * Z[k * ldz + i];
    x[i] = s;
  }
}

#define PFC_NV_CASES(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) \
  X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) X(31) X(32)

}  // namespace

int blas_nblocks(size_t N) {
  size_t b = (N + 4 * NT - 1) / (4 * NT);   // >= 4 elements per thread
  if (b > 148 * 8) b = 148 * 8;
  if (b < 1) b = 1;
  return (int)b;
}

static int grid_pointwise(size_t N) {
  size_t b = (N + NT - 1) / NT;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

cudaError_t launch_coef(pfc_ctx* ctx, const double* phi, const double* psi, double* c) {
  k_coef<<<grid_pointwise(ctx->N), NT, 0, ctx->stream>>>(phi, psi, c, ctx->N);
  ctx->launches++;
  pfc_account(ctx, PFC_K_COEF, 24.0 * ctx->N, 5.0 * ctx->N);
  return cudaGetLastError();
}

cudaError_t launch_axpby(pfc_ctx* ctx, double a, const double* x, double b, const double* y,
                         double* out) {
  k_axpby<<<grid_pointwise(ctx->N), NT, 0, ctx->stream>>>(a, x, b, y, out, ctx->N);
  ctx->launches++;
  pfc_account(ctx, PFC_K_VECTOR, (y ? 24.0 : 16.0) * ctx->N, (y ? 3.0 : 1.0) * ctx->N);
  return cudaGetLastError();
}

cudaError_t launch_multidot(pfc_ctx* ctx, const double* V, int nv, const double* w,
                            double* partials, double* out) {
  const int nb = blas_nblocks(ctx->N);
  switch (nv) {
#define X(K)                                                                        \
  case K:                                                                           \
    k_multidot<K><<<nb, NT, 0, ctx->stream>>>(V, ctx->N, w, ctx->N, partials, out,  \
                                              ctx->ticket, ctx->gate);              \
    break;
    PFC_NV_CASES(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
  ctx->launches++;
  pfc_account(ctx, PFC_K_ORTH, 8.0 * (nv + 1) * ctx->N, 2.0 * nv * ctx->N);
  return cudaGetLastError();
}

cudaError_t launch_axpy_dot(pfc_ctx* ctx, const double* V, int nv, const double* h, double* w,
                            double* partials, double* out) {
  const int nb = blas_nblocks(ctx->N);
  switch (nv) {
#define X(K)                                                                          \
  case K:                                                                             \
    k_axpy_dot<K><<<nb, NT, 0, ctx->stream>>>(V, ctx->N, h, w, ctx->N, partials, out, \
                                              ctx->ticket, ctx->gate);                \
    break;
    PFC_NV_CASES(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
  ctx->launches++;
  pfc_account(ctx, PFC_K_ORTH, 8.0 * (nv + 2) * ctx->N, 4.0 * nv * ctx->N);
  return cudaGetLastError();
}

static cudaError_t axpy_norm_impl(pfc_ctx* ctx, const double* V, int nv, const double* h1,
                                  const double* h, double* w, double* partials, double* out,
                                  pfc_gmres_dev* gm) {
  const int nb = blas_nblocks(ctx->N);
  switch (nv) {
#define X(K)                                                                           \
  case K:                                                                              \
    k_axpy_norm<K><<<nb, NT, 0, ctx->stream>>>(V, ctx->N, h, w, ctx->N, partials, out, \
                                               ctx->ticket, gm, h1);                   \
    break;
    PFC_NV_CASES(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
  ctx->launches++;
  pfc_account(ctx, PFC_K_ORTH, 8.0 * (nv + 2) * ctx->N, (2.0 * nv + 2.0) * ctx->N);
  return cudaGetLastError();
}

cudaError_t launch_axpy_norm(pfc_ctx* ctx, const double* V, int nv, const double* h, double* w,
                             double* partials, double* out) {
  return axpy_norm_impl(ctx, V, nv, nullptr, h, w, partials, out, nullptr);
}

cudaError_t launch_axpy_norm_close(pfc_ctx* ctx, const double* V, int nv, const double* h1,
                                   const double* h2, double* w, double* partials, double* out) {
  return axpy_norm_impl(ctx, V, nv, h1, h2, w, partials, out, ctx->gm);
}

cudaError_t launch_scale_next(pfc_ctx* ctx, const double* w, double* vnext) {
  k_scale_next<<<grid_pointwise(ctx->N), NT, 0, ctx->stream>>>(ctx->gm, w, vnext, ctx->N);
  ctx->launches++;
  pfc_account(ctx, PFC_K_VECTOR, 16.0 * ctx->N, 1.0 * ctx->N);
  return cudaGetLastError();
}

cudaError_t launch_cycle_init(pfc_ctx* ctx, double beta, double tol, int its_done) {
  k_cycle_init<<<1, 1, 0, ctx->stream>>>(ctx->gm, beta, tol, ctx->cfg.gmres_restart,
                                         ctx->cfg.gmres_maxit, its_done);
  ctx->launches++;
  return cudaGetLastError();
}

cudaError_t launch_backsolve_lincomb(pfc_ctx* ctx, double* x, const double* Z, int jm) {
  k_backsolve<<<1, 1, 0, ctx->stream>>>(ctx->gm);
  ctx->launches++;
  k_lincomb_dev<<<blas_nblocks(ctx->N), NT, 0, ctx->stream>>>(x, Z, ctx->N, ctx->gm, ctx->N);
  ctx->launches++;
  pfc_account(ctx, PFC_K_VECTOR, 8.0 * (jm + 2) * ctx->N, 2.0 * jm * ctx->N);
  return cudaGetLastError();
}

cudaError_t launch_lincomb_dev(pfc_ctx* ctx, double* x, const double* Z) {
  k_lincomb_dev<<<blas_nblocks(ctx->N), NT, 0, ctx->stream>>>(x, Z, ctx->N, ctx->gm, ctx->N);
  ctx->launches++;
  return cudaGetLastError();
}

cudaError_t launch_norm2(pfc_ctx* ctx, const double* x, double* partials, double* out) {
  k_norm2<<<blas_nblocks(ctx->N), NT, 0, ctx->stream>>>(x, ctx->N, partials, out, ctx->ticket);
  ctx->launches++;
  pfc_account(ctx, PFC_K_VECTOR, 8.0 * ctx->N, 2.0 * ctx->N);
  return cudaGetLastError();
}

cudaError_t launch_finalize(pfc_ctx* ctx, const double* partials, int nblk, int nval,
                            double* out) {
  k_finalize<<<nval, NT, 0, ctx->stream>>>(partials, nblk, nval, out);
  ctx->launches++;
  pfc_account(ctx, PFC_K_FINALIZE, 8.0 * nblk * nval, 1.0 * nblk * nval);
  return cudaGetLastError();
}

cudaError_t launch_lincomb(pfc_ctx* ctx, double* x, const double* Z, int nv, const double* coef) {
  if (nv <= 0) return cudaSuccess;
  Coef cf;
  for (int k = 0; k < PFC_MAX_RESTART; ++k) cf.c[k] = k < nv ? coef[k] : 0.0;
  const int nb = blas_nblocks(ctx->N);
  // chunks of <= 32 vectors (gmres_restart <= 64)
  int done = 0;
  while (done < nv) {
    int k = nv - done > 32 ? 32 : nv - done;
    Coef cc;
    for (int i = 0; i < PFC_MAX_RESTART; ++i) cc.c[i] = i < k ? cf.c[done + i] : 0.0;
    const double* Zk = Z + (size_t)done * ctx->N;
    switch (k) {
#define X(K)                                                                    \
  case K:                                                                       \
    k_lincomb<K><<<nb, NT, 0, ctx->stream>>>(x, Zk, ctx->N, cc, ctx->N);        \
    break;
      PFC_NV_CASES(X)
#undef X
    }
    ctx->launches++;
    pfc_account(ctx, PFC_K_VECTOR, 8.0 * (k + 2) * ctx->N, 2.0 * k * ctx->N);
    done += k;
  }
  return cudaGetLastError();
}
