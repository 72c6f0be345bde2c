// pfc.cu -- host solver (inexact Newton + FGMRES + left-RAS, adaptive dt) and the C ABI of
// include/pfc.h.  Every arithmetic step runs in this library's kernels; the host only holds
// the (m+1) x m Hessenberg matrix, the Givens rotations and the stopping tests, as in
// Algorithm P:344-380.  There is no CPU fallback: without a usable CUDA device every entry
// point fails with PFC_ECUDA.
#include <math.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include <cudaTypedefs.h>

#include <algorithm>
#include <vector>

#include "pfc_internal.h"

// ------------------------------------------------------------------ error helpers

pfc_status pfc_fail(pfc_ctx* ctx, pfc_status st, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return st;
}

pfc_status pfc_check_cuda(pfc_ctx* ctx, cudaError_t e, const char* where) {
  if (e == cudaSuccess) return PFC_OK;
  char buf[512];
  snprintf(buf, sizeof buf, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
  return pfc_fail(ctx, e == cudaErrorMemoryAllocation ? PFC_ENOMEM : PFC_ECUDA, buf);
}

#define CK(expr, where)                                          \
  do {                                                           \
    pfc_status _s = pfc_check_cuda(ctx, (expr), where);          \
    if (_s != PFC_OK) return _s;                                 \
  } while (0)

// ------------------------------------------------------------------ profiling

static cudaEvent_t ev_get(pfc_ctx* ctx) {
  if (!ctx->ev_pool.empty()) {
    cudaEvent_t e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

static void prof_begin(pfc_ctx* ctx) {
  if (!ctx->prof) return;
  ctx->ev_open = ev_get(ctx);
  cudaEventRecord(ctx->ev_open, ctx->stream);
}

static void prof_end(pfc_ctx* ctx, int cls) {
  if (!ctx->prof || !ctx->ev_open) return;
  cudaEvent_t b = ev_get(ctx);
  cudaEventRecord(b, ctx->stream);
  ctx->pending.push_back({cls, ctx->ev_open, b});
  ctx->ev_open = nullptr;
}

static void prof_drain(pfc_ctx* ctx) {
  if (ctx->pending.empty()) return;
  cudaStreamSynchronize(ctx->stream);
  for (auto& p : ctx->pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    ctx->prof_count[p.cls]++;
    ctx->prof_ms[p.cls] += ms;
    ctx->ev_pool.push_back(p.a);
    ctx->ev_pool.push_back(p.b);
  }
  ctx->pending.clear();
}

// launch with optional per-class event bracketing
#define KL(cls, expr, where)                        \
  do {                                              \
    prof_begin(ctx);                                \
    cudaError_t _e = (expr);                        \
    prof_end(ctx, cls);                             \
    CK(_e, where);                                  \
  } while (0)

// ------------------------------------------------------------------ TMA descriptors

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool tma_encode(CUtensorMap* map, const double* ptr, int ndim, const int* n, const int* box) {
  if (!g_encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return false;
    }
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[3], strides[2];
  cuuint32_t bx[3], es[3] = {1, 1, 1};
  for (int d = 0; d < ndim; ++d) {
    dims[d] = (cuuint64_t)n[d];
    bx[d] = (cuuint32_t)box[d];
  }
  strides[0] = (cuuint64_t)n[0] * sizeof(double);
  if (ndim == 3) strides[1] = (cuuint64_t)n[0] * n[1] * sizeof(double);
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, ndim, const_cast<double*>(ptr), dims,
                        strides, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool tma_usable(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

// ------------------------------------------------------------------ dispatch

cudaError_t launch_residual(pfc_ctx* ctx, const double* a, const double* b, double dt, double* F,
                            double* partials, int* nparts) {
  if (generic_path(ctx->cfg)) return launch_residual_mob(ctx, a, b, dt, F, partials, nparts);
  return ctx->cfg.ndim == 2 ? launch_residual_2d(ctx, a, b, dt, F, partials, nparts)
                            : launch_residual_3d(ctx, a, b, dt, F, partials, nparts);
}

cudaError_t launch_jv(pfc_ctx* ctx, const double* v, const double* c, double dt, double* out) {
  if (generic_path(ctx->cfg)) return launch_jv_mob(ctx, v, c, dt, out);
  return ctx->cfg.ndim == 2 ? launch_jv_2d(ctx, v, c, dt, out) : launch_jv_3d(ctx, v, c, dt, out);
}

cudaError_t launch_jac_state(pfc_ctx* ctx, const double* phi_new, const double* phi_old) {
  cudaError_t e = launch_coef(ctx, phi_new, phi_old, ctx->c);
  if (e != cudaSuccess || !generic_path(ctx->cfg)) return e;
  return launch_mob_state(ctx, phi_new, phi_old);
}

int ras_plan(pfc_ctx* ctx) { return ctx->cfg.ndim == 2 ? ras2d_plan(ctx) : ras3d_plan(ctx); }

cudaError_t launch_ras(pfc_ctx* ctx, const double* v, const double* c, double dt, double* z) {
  if (ctx->cfg.ras_local_solver != PFC_LOCAL_GMRES) return launch_ras_ilu(ctx, v, z);
  if (ctx->cfg.ndim == 2) return launch_ras_2d(ctx, v, c, dt, z);
  if (ctx->ras3_col == 2) return launch_ras_3d_cl2(ctx, v, c, dt, z, ctx->ras_scratch);
  return ctx->ras3_col ? launch_ras_3d_col(ctx, v, c, dt, z, ctx->ras_scratch)
                       : launch_ras_3d(ctx, v, c, dt, z, ctx->ras_scratch);
}

// ------------------------------------------------------------------ scalars


static pfc_status fetch(pfc_ctx* ctx, int off, int count) {
  CK(cudaMemcpyAsync(ctx->hscal + off, ctx->dscal + off, count * sizeof(double),
                     cudaMemcpyDeviceToHost, ctx->stream),
     "D2H scalars");
  CK(cudaStreamSynchronize(ctx->stream), "stream sync");
  return PFC_OK;
}

// ||F(phi_new; psi)|| with F written to `F`
static pfc_status residual_norm(pfc_ctx* ctx, const double* phi_new, double dt, double* F,
                                double* nrm) {
  int np = 0;
  KL(PFC_K_RESIDUAL, launch_residual(ctx, phi_new, ctx->psi, dt, F, ctx->partials, &np), "residual");
  KL(PFC_K_FINALIZE, launch_finalize(ctx, ctx->partials, np, 1, ctx->dscal + SC_NRM), "finalize");
  pfc_status s = fetch(ctx, SC_NRM, 1);
  if (s) return s;
  *nrm = sqrt(ctx->hscal[SC_NRM]);
  return PFC_OK;
}

static pfc_status energy_mass(pfc_ctx* ctx, const double* phi, double* F_d, double* M) {
  int np = 0;
  KL(PFC_K_ENERGY, launch_energy_mass(ctx, phi, ctx->partials, &np), "energy");
  KL(PFC_K_FINALIZE, launch_finalize(ctx, ctx->partials, np, 2, ctx->dscal + SC_EN), "finalize");
  pfc_status s = fetch(ctx, SC_EN, 2);
  if (s) return s;
  if (F_d) *F_d = ctx->hscal[SC_EN] * ctx->hd;
  if (M) *M = ctx->hscal[SC_EN + 1] * ctx->hd;
  return PFC_OK;
}

// ------------------------------------------------------------------ FGMRES

// Solve J S = -F approximately: right-preconditioned flexible GMRES(m), CGS2 Arnoldi, Givens,
// x0 = 0, stop at ||r|| <= max(xi_r ||F||, xi_a) or gmres_maxit iterations.  Host-driven
// loop (one D2H round trip per Arnoldi step): the default (see fgmres() below for why).
static pfc_status fgmres_host(pfc_ctx* ctx, double dt, double Fnorm, int* its_out) {
  const pfc_config& c = ctx->cfg;
  const int m = c.gmres_restart;
  const size_t N = ctx->N;
  const double tol = std::max(c.gmres_rtol * Fnorm, c.gmres_atol);
  std::vector<double> H((m + 1) * m), cs(m), sn(m), g(m + 1), y(m);
  int its = 0;
  CK(cudaMemsetAsync(ctx->S, 0, N * sizeof(double), ctx->stream), "memset S");
  if (Fnorm <= tol || Fnorm == 0.0) { *its_out = 0; return PFC_OK; }
  // r0 = -F, V0 = r0/beta
  double beta = Fnorm;
  KL(PFC_K_VECTOR, launch_axpby(ctx, -1.0 / beta, ctx->F, 0.0, nullptr, ctx->V), "axpby");
  for (;;) {
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int jm = 0;
    bool stop = false;
    for (int j = 0; j < m; ++j) {
      double* Vj = ctx->V + (size_t)j * N;
      double* Zj = ctx->Z + (size_t)j * N;
      KL(PFC_K_RAS, launch_ras(ctx, Vj, ctx->c, dt, Zj), "ras");
      if (ctx->tail) {   // w = J z_j, CGS2 and v_{j+1} = w/|w| in one cooperative kernel
        KL(PFC_K_ORTH, launch_arnoldi_tail(ctx, ctx->V, Zj, ctx->c, dt, j, ctx->V + (size_t)(j + 1) * N, ctx->dscal), "arnoldi tail");
      } else {
        KL(PFC_K_JV, launch_jv(ctx, Zj, ctx->c, dt, ctx->w), "jv");
        KL(PFC_K_ORTH, launch_multidot(ctx, ctx->V, j + 1, ctx->w, ctx->partials, ctx->dscal + SC_H1), "multidot");
        KL(PFC_K_ORTH, launch_axpy_dot(ctx, ctx->V, j + 1, ctx->dscal + SC_H1, ctx->w, ctx->partials, ctx->dscal + SC_H2), "cgs2");
        KL(PFC_K_ORTH, launch_axpy_norm(ctx, ctx->V, j + 1, ctx->dscal + SC_H2, ctx->w, ctx->partials, ctx->dscal + SC_NRM), "cgs2");
      }
      pfc_status s = fetch(ctx, 0, SC_NRM + 1);
      if (s) return s;
      const double* h1 = ctx->hscal + SC_H1;
      const double* h2 = ctx->hscal + SC_H2;
      const double hn = sqrt(ctx->hscal[SC_NRM]);
      for (int i = 0; i <= j; ++i) H[i + (m + 1) * j] = h1[i] + h2[i];
      H[j + 1 + (m + 1) * j] = hn;
      for (int i = 0; i < j; ++i) {
        double a = H[i + (m + 1) * j], b = H[i + 1 + (m + 1) * j];
        H[i + (m + 1) * j] = cs[i] * a + sn[i] * b;
        H[i + 1 + (m + 1) * j] = -sn[i] * a + cs[i] * b;
      }
      double a = H[j + (m + 1) * j], b = H[j + 1 + (m + 1) * j];
      double r = sqrt(a * a + b * b);
      cs[j] = r == 0.0 ? 1.0 : a / r;
      sn[j] = r == 0.0 ? 0.0 : b / r;
      H[j + (m + 1) * j] = cs[j] * a + sn[j] * b;
      H[j + 1 + (m + 1) * j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++its;
      jm = j + 1;
      const double res = fabs(g[j + 1]);
      if (!isfinite(res)) return pfc_fail(ctx, PFC_EBREAKDOWN, "FGMRES: non-finite residual");
      if (hn <= 1e-14 * beta) { stop = true; break; }           // happy breakdown
      if (!ctx->tail)   // (the fused tail has written v_{j+1} already)
        KL(PFC_K_VECTOR, launch_axpby(ctx, 1.0 / hn, ctx->w, 0.0, nullptr, ctx->V + (size_t)(j + 1) * N), "scale");
      if (res <= tol || its >= c.gmres_maxit) { stop = true; break; }
    }
    for (int i = jm - 1; i >= 0; --i) {
      double s = g[i];
      for (int l = i + 1; l < jm; ++l) s -= H[i + (m + 1) * l] * y[l];
      y[i] = s / H[i + (m + 1) * i];
    }
    KL(PFC_K_VECTOR, launch_lincomb(ctx, ctx->S, ctx->Z, jm, y.data()), "lincomb");   // S += Z y
    if (stop) break;
    // restart: r = -F - J S (true residual), V0 = r/|r|
    KL(PFC_K_JV, launch_jv(ctx, ctx->S, ctx->c, dt, ctx->w), "jv");
    KL(PFC_K_VECTOR, launch_axpby(ctx, -1.0, ctx->F, -1.0, ctx->w, ctx->w), "axpby");
    KL(PFC_K_VECTOR, launch_norm2(ctx, ctx->w, ctx->partials, ctx->dscal + SC_NRM), "norm");
    pfc_status s = fetch(ctx, SC_NRM, 1);
    if (s) return s;
    beta = sqrt(ctx->hscal[SC_NRM]);
    if (beta <= tol) break;
    KL(PFC_K_VECTOR, launch_axpby(ctx, 1.0 / beta, ctx->w, 0.0, nullptr, ctx->V), "scale");
  }
  *its_out = its;
  return PFC_OK;
}

// Device-resident FGMRES (NEXT row f1): same mathematics and stopping rule as fgmres_host, but
// the Givens update and the stop decision of every Arnoldi step run on the device (in the
// last block of k_axpy_norm).  The host launches step j+1 before it knows whether step j
// stopped the cycle and only then waits for step j-1's flags, so the GPU never idles for a
// host round trip inside a cycle; kernels of a step launched after the stop exit at once
// (gate = &gm->stop).  Back substitution and S += Z y run on the device too.  The host syncs
// once per cycle (restart / exit) instead of once per Arnoldi step.
static pfc_status fgmres_device(pfc_ctx* ctx, double dt, double Fnorm, int* its_out) {
  const pfc_config& c = ctx->cfg;
  const int m = c.gmres_restart;
  const size_t N = ctx->N;
  const double tol = std::max(c.gmres_rtol * Fnorm, c.gmres_atol);
  int its = 0;
  CK(cudaMemsetAsync(ctx->S, 0, N * sizeof(double), ctx->stream), "memset S");
  if (Fnorm <= tol || Fnorm == 0.0) { *its_out = 0; return PFC_OK; }
  double beta = Fnorm;
  KL(PFC_K_VECTOR, launch_axpby(ctx, -1.0 / beta, ctx->F, 0.0, nullptr, ctx->V), "axpby");
  for (;;) {
    KL(PFC_K_VECTOR, launch_cycle_init(ctx, beta, tol, its), "cycle init");
    ctx->gate = &ctx->gm->stop;
    int* fl = nullptr;            // flags of the step that stopped the cycle
    int launched = 0;
    for (int j = 0; j < m && !fl; ++j) {
      double* Vj = ctx->V + (size_t)j * N;
      double* Zj = ctx->Z + (size_t)j * N;
      KL(PFC_K_RAS, launch_ras(ctx, Vj, ctx->c, dt, Zj), "ras");
      if (ctx->tail) {   // J z, CGS2, v_{j+1} and the device Givens / stop test in one kernel
        KL(PFC_K_ORTH, launch_arnoldi_tail(ctx, ctx->V, Zj, ctx->c, dt, j, ctx->V + (size_t)(j + 1) * N, ctx->dscal, ctx->gm), "arnoldi tail");
      } else {
        KL(PFC_K_JV, launch_jv(ctx, Zj, ctx->c, dt, ctx->w), "jv");
        KL(PFC_K_ORTH, launch_multidot(ctx, ctx->V, j + 1, ctx->w, ctx->partials, ctx->dscal + SC_H1), "multidot");
        KL(PFC_K_ORTH, launch_axpy_dot(ctx, ctx->V, j + 1, ctx->dscal + SC_H1, ctx->w, ctx->partials, ctx->dscal + SC_H2), "cgs2");
        KL(PFC_K_ORTH, launch_axpy_norm_close(ctx, ctx->V, j + 1, ctx->dscal + SC_H1, ctx->dscal + SC_H2, ctx->w, ctx->partials, ctx->dscal + SC_NRM), "cgs2");
        if (j + 1 < m)
          KL(PFC_K_VECTOR, launch_scale_next(ctx, ctx->w, ctx->V + (size_t)(j + 1) * N), "scale");
      }
      CK(cudaMemcpyAsync(ctx->hflags + 4 * j, &ctx->gm->stop, 4 * sizeof(int),
                         cudaMemcpyDeviceToHost, ctx->stream), "D2H flags");
      CK(cudaEventRecord(ctx->step_ev[j], ctx->stream), "event");
      launched = j + 1;
      if (j >= 1) {   // step j is queued behind step j-1: now look at step j-1
        CK(cudaEventSynchronize(ctx->step_ev[j - 1]), "event sync");
        if (ctx->hflags[4 * (j - 1)]) fl = ctx->hflags + 4 * (j - 1);
      }
    }
    if (!fl) {        // the last launched step decides (the cycle always stops by step m-1)
      CK(cudaEventSynchronize(ctx->step_ev[launched - 1]), "event sync");
      fl = ctx->hflags + 4 * (launched - 1);
    }
    ctx->gate = nullptr;
    const int jm = fl[1], reason = fl[3];
    its = fl[2];
    if (reason == PFC_GM_NONFINITE)
      return pfc_fail(ctx, PFC_EBREAKDOWN, "FGMRES: non-finite residual");
    KL(PFC_K_VECTOR, launch_backsolve_lincomb(ctx, ctx->S, ctx->Z, jm), "lincomb");   // S += Z y
    if (reason != PFC_GM_RESTART) break;
    // restart: r = -F - J S (true residual), V0 = r/|r|
    KL(PFC_K_JV, launch_jv(ctx, ctx->S, ctx->c, dt, ctx->w), "jv");
    KL(PFC_K_VECTOR, launch_axpby(ctx, -1.0, ctx->F, -1.0, ctx->w, ctx->w), "axpby");
    KL(PFC_K_VECTOR, launch_norm2(ctx, ctx->w, ctx->partials, ctx->dscal + SC_NRM), "norm");
    pfc_status s = fetch(ctx, SC_NRM, 1);
    if (s) return s;
    beta = sqrt(ctx->hscal[SC_NRM]);
    if (beta <= tol) break;
    KL(PFC_K_VECTOR, launch_axpby(ctx, 1.0 / beta, ctx->w, 0.0, nullptr, ctx->V), "scale");
  }
  *its_out = its;
  return PFC_OK;
}

// Default: the host-driven loop.  Measured on B200 (round 1, bench.py, 197 / 20 steps): the
// device-resident cycle was 2-5% SLOWER on cfg1, cfg2 and equal on cfg4 -- the cycles are short
// (2-3 Arnoldi steps per Newton iteration at the configs' dt), so the early-exit kernels of the
// one speculative step per cycle cost more than the ~5 us host round trips they remove.
// PFC_DEVICE_ARNOLDI=1 selects fgmres_device (same results to rounding; parity-tested).
// With the fused Arnoldi tail (2D grids of configs 1-3) an Arnoldi step is two kernels; the
// device-resident cycle then measured 479 vs 473 steps/s on cfg1 and 418 vs 430 on cfg2
// (round 2, bench.py): still not worth its speculative launches, so it stays opt-in
// (PFC_DEVICE_ARNOLDI=1; it uses the fused tail where the host loop does).
static pfc_status fgmres(pfc_ctx* ctx, double dt, double Fnorm, int* its_out) {
  const char* e = getenv("PFC_DEVICE_ARNOLDI");
  const bool dev = e && e[0] != '0';
  return dev ? fgmres_device(ctx, dt, Fnorm, its_out) : fgmres_host(ctx, dt, Fnorm, its_out);
}

// ------------------------------------------------------------------ Newton

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static pfc_status newton(pfc_ctx* ctx, double dt, pfc_step_info* inf) {
  const pfc_config& c = ctx->cfg;
  const size_t bytes = ctx->N * sizeof(double);
  CK(cudaMemcpyAsync(ctx->phi, ctx->psi, bytes, cudaMemcpyDeviceToDevice, ctx->stream),
     "Phi_0 = psi");
  double nrm = 0.0;
  pfc_status s = residual_norm(ctx, ctx->phi, dt, ctx->F, &nrm);
  if (s) return s;
  const double n0 = nrm;
  const double stop = std::max(c.newton_rtol * n0, c.newton_atol);
  inf->res0 = n0;
  while (!(nrm <= stop)) {
    if (!isfinite(nrm)) {
      inf->res_final = nrm;
      return pfc_fail(ctx, PFC_EBREAKDOWN, "Newton: non-finite residual norm");
    }
    if (inf->newton_its >= c.newton_maxit) {
      inf->res_final = nrm;
      return pfc_fail(ctx, PFC_ENOCONV, "Newton: newton_maxit reached");
    }
    KL(PFC_K_COEF, launch_jac_state(ctx, ctx->phi, ctx->psi), "coef");
    if (c.ras_local_solver != PFC_LOCAL_GMRES && (!c.ras_ilu_reuse || inf->newton_its == 0))
      KL(PFC_K_RAS, launch_ilu_factor(ctx, ctx->c, dt), "ilu factor");
    int its = 0;
    s = fgmres(ctx, dt, nrm, &its);
    if (s) return s;
    inf->gmres_its += its;
    double lambda = 1.0;
    bool accepted = false;
    for (int t = 0; t <= 40 && lambda >= c.ls_min_lambda; ++t) {
      KL(PFC_K_VECTOR, launch_axpby(ctx, 1.0, ctx->phi, lambda, ctx->S, ctx->trial), "trial");
      double nt = 0.0;
      s = residual_norm(ctx, ctx->trial, dt, ctx->Ft, &nt);
      if (s) return s;
      if (nt <= (1.0 - c.ls_c1 * lambda) * nrm) {
        accepted = true;
        nrm = nt;
        break;
      }
      lambda *= 0.5;
      inf->ls_backtracks++;
    }
    if (!accepted) {
      inf->res_final = nrm;
      return pfc_fail(ctx, PFC_ENOCONV, "Newton: line search reached ls_min_lambda");
    }
    std::swap(ctx->phi, ctx->trial);
    std::swap(ctx->F, ctx->Ft);
    inf->newton_its++;
  }
  inf->res_final = nrm;
  inf->converged = 1;
  return PFC_OK;
}

// ------------------------------------------------------------------ C ABI

extern "C" {

void pfc_config_default(pfc_config* c) {
  if (!c) return;
  memset(c, 0, sizeof *c);
  c->ndim = 2;
  c->n[0] = c->n[1] = 64;
  c->n[2] = 1;
  c->h = M_PI / 4.0;
  c->gamma = 0.25;
  c->adaptive = 0;
  c->dt_min = 0.01;
  c->dt_max = 10.0;
  c->eta = 5000.0;
  c->newton_rtol = 1e-10;
  c->newton_atol = 1e-10;
  c->newton_maxit = 50;
  c->ls_c1 = 1e-4;
  c->ls_min_lambda = 1e-12;
  c->gmres_restart = 30;
  c->gmres_maxit = 300;
  c->gmres_rtol = 1e-3;
  c->gmres_atol = 1e-11;
  c->ras_box[0] = c->ras_box[1] = c->ras_box[2] = 16;
  c->ras_overlap = 2;
  c->ras_local_k = 10;
  c->ras_variant = PFC_RAS_LEFT;
  c->mobility = PFC_MOBILITY_ONE;
  c->ras_local_solver = PFC_LOCAL_GMRES;
  c->ras_ilu_level = 0;
  c->ras_ilu_reuse = 0;
  c->bc = PFC_BC_PERIODIC;
}

static pfc_status validate(const pfc_config& c, std::string* why) {
  char b[256];
  auto bad = [&](const char* m) { *why = m; return PFC_EINVAL; };
  if (c.ndim != 2 && c.ndim != 3) return bad("ndim must be 2 or 3");
  for (int d = 0; d < c.ndim; ++d) {
    if (c.n[d] < 4) return bad("every n_d must be >= 4");
    if (c.ras_box[d] < 1 || c.n[d] % c.ras_box[d] != 0) return bad("ras_box_d must divide n_d");
    if (c.ras_overlap < 0 || c.ras_overlap >= c.ras_box[d])
      return bad("need 0 <= ras_overlap < ras_box_d");
    if (c.ras_box[d] + 2 * c.ras_overlap + 6 > c.n[d]) {
      snprintf(b, sizeof b, "ext box + zero ring (%d) exceeds n[%d]=%d (P:429-437 ring would wrap)",
               c.ras_box[d] + 2 * c.ras_overlap + 6, d, c.n[d]);
      *why = b;
      return PFC_EINVAL;
    }
  }
  if ((double)c.n[0] * c.n[1] * (c.ndim == 3 ? c.n[2] : 1) > 2147483647.0)
    return bad("grid too large (N must fit int32 indexing of planes)");
  if (!(c.h > 0)) return bad("h must be > 0");
  if (!(c.gamma > 0)) return bad("gamma must be > 0");
  if (c.adaptive && !(c.dt_min > 0 && c.dt_min <= c.dt_max)) return bad("need 0 < dt_min <= dt_max");
  if (c.adaptive && !(c.eta >= 0)) return bad("eta must be >= 0");
  if (c.ras_local_k < 1 || c.ras_local_k > PFC_MAX_LOCAL_K) return bad("ras_local_k in [1,15]");
  if (c.ras_variant != PFC_RAS_LEFT && c.ras_variant != PFC_RAS_AS && c.ras_variant != PFC_RAS_RIGHT)
    return bad("ras_variant must be PFC_RAS_LEFT, PFC_RAS_AS or PFC_RAS_RIGHT");
  if (c.mobility != PFC_MOBILITY_ONE && c.mobility != PFC_MOBILITY_QUADRATIC)
    return bad("mobility must be PFC_MOBILITY_ONE or PFC_MOBILITY_QUADRATIC");
  if (c.ras_local_solver != PFC_LOCAL_GMRES && c.ras_local_solver != PFC_LOCAL_ILU &&
      c.ras_local_solver != PFC_LOCAL_LU)
    return bad("ras_local_solver must be PFC_LOCAL_GMRES, PFC_LOCAL_ILU or PFC_LOCAL_LU");
  if (c.ras_local_solver == PFC_LOCAL_ILU && (c.ras_ilu_level < 0 || c.ras_ilu_level > 4))
    return bad("ras_ilu_level in [0,4]");
  if (c.ras_local_solver != PFC_LOCAL_GMRES && c.mobility != PFC_MOBILITY_ONE)
    return bad("PFC_LOCAL_ILU / PFC_LOCAL_LU are built for PFC_MOBILITY_ONE");
  if (c.bc != PFC_BC_PERIODIC && c.bc != PFC_BC_MIRROR)
    return bad("bc must be PFC_BC_PERIODIC or PFC_BC_MIRROR");
  if (c.bc == PFC_BC_MIRROR &&
      (c.ras_box[0] < 3 || c.ras_box[1] < 3 || (c.ndim == 3 && c.ras_box[2] < 3)))
    return bad("PFC_BC_MIRROR needs ras_box >= 3 (mirror partners inside the boundary box)");
  if (c.gmres_restart < 1 || c.gmres_restart > PFC_MAX_RESTART) return bad("gmres_restart in [1,32]");
  if (c.gmres_maxit < 1 || c.newton_maxit < 0) return bad("iteration limits must be positive");
  if (!(c.newton_rtol >= 0 && c.newton_atol >= 0 && c.gmres_rtol >= 0 && c.gmres_atol >= 0))
    return bad("tolerances must be >= 0");
  return PFC_OK;
}

pfc_status pfc_create(const pfc_config* cfg, void* stream, pfc_ctx** out) {
  if (!cfg || !out) return PFC_EINVAL;
  *out = nullptr;
  pfc_ctx* ctx = new pfc_ctx();
  ctx->cfg = *cfg;
  if (ctx->cfg.ndim == 2) {
    ctx->cfg.n[2] = 1;
    ctx->cfg.ras_box[2] = 1;
  }
  std::string why;
  pfc_status st = validate(ctx->cfg, &why);
  auto fail = [&](pfc_status s) {
    *out = ctx;   // let the caller read pfc_last_error, then pfc_destroy
    return s;
  };
  if (st) { ctx->err = why; return fail(st); }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    ctx->err = "no CUDA device: libpfc has no CPU fallback";
    return fail(PFC_ECUDA);
  }
  cudaGetDevice(&ctx->device);
  ctx->stream = (cudaStream_t)stream;
  const pfc_config& c = ctx->cfg;
  ctx->N = (size_t)c.n[0] * c.n[1] * c.n[2];
  ctx->ih2 = 1.0 / (c.h * c.h);
  ctx->hd = pow(c.h, c.ndim);
  if (!ras_plan(ctx)) {
    ctx->err = "RAS extended box too large for the subdomain kernel's shared-memory plan";
    return fail(PFC_EINVAL);
  }
  const size_t bytes = ctx->N * sizeof(double);
  const int m = c.gmres_restart;
  double** fields[] = {&ctx->phi, &ctx->psi, &ctx->F, &ctx->Ft, &ctx->trial,
                       &ctx->S,   &ctx->c,   &ctx->w, &ctx->stage};
  for (double** f : fields)
    if (pfc_check_cuda(ctx, cudaMalloc(f, bytes), "cudaMalloc field")) return fail(PFC_ENOMEM);
  if (generic_path(c)) {
    double** mf[] = {&ctx->mob_A, &ctx->mob_t[0], &ctx->mob_t[1], &ctx->mob_t[2]};
    for (double** f : mf)
      if (pfc_check_cuda(ctx, cudaMalloc(f, bytes), "cudaMalloc mobility field")) return fail(PFC_ENOMEM);
  }
  if (pfc_check_cuda(ctx, cudaMalloc(&ctx->V, bytes * (m + 1)), "cudaMalloc V") ||
      pfc_check_cuda(ctx, cudaMalloc(&ctx->Z, bytes * m), "cudaMalloc Z"))
    return fail(PFC_ENOMEM);
  // reduction scratch: max(per-tile partials, blas blocks * 32, energy blocks * 2)
  size_t tiles = 0;
  if (c.ndim == 2) tiles = (size_t)((c.n[0] + 31) / 32) * ((c.n[1] + 15) / 16);
  else tiles = (size_t)((c.n[0] + 31) / 32) * ((c.n[1] + 15) / 16) * (size_t)c.n[2];
  ctx->npartials = std::max<size_t>(std::max<size_t>(tiles, (size_t)blas_nblocks(ctx->N) * 32),
                                    (size_t)4096 * 40) + 64;   // (fused tail: blocks x 40)
  if (pfc_check_cuda(ctx, cudaMalloc(&ctx->partials, ctx->npartials * sizeof(double)), "partials") ||
      pfc_check_cuda(ctx, cudaMalloc(&ctx->dscal, SC_TOTAL * sizeof(double)), "dscal") ||
      pfc_check_cuda(ctx, cudaMalloc(&ctx->ticket, sizeof(unsigned int)), "ticket") ||
      pfc_check_cuda(ctx, cudaMemset(ctx->ticket, 0, sizeof(unsigned int)), "ticket") ||
      pfc_check_cuda(ctx, cudaMalloc(&ctx->gm, sizeof(pfc_gmres_dev)), "gmres state") ||
      pfc_check_cuda(ctx, cudaMemset(ctx->gm, 0, sizeof(pfc_gmres_dev)), "gmres state") ||
      pfc_check_cuda(ctx, cudaMallocHost(&ctx->hflags, 4 * PFC_MAX_RESTART * sizeof(int)), "flags") ||
      pfc_check_cuda(ctx, cudaMallocHost(&ctx->hscal, SC_TOTAL * sizeof(double)), "hscal") ||
      pfc_check_cuda(ctx, cudaMalloc(&ctx->d_jcnt, 4 * sizeof(unsigned long long)), "jcnt") ||
      pfc_check_cuda(ctx, cudaMemset(ctx->d_jcnt, 0, 4 * sizeof(unsigned long long)), "jcnt"))
    return fail(PFC_ENOMEM);
  if (c.ndim == 3) {
    // subdomain kernel: the 2-CTA cluster kernel (basis on chip) where instantiated, else the
    // single-CTA column kernel, else the global-scratch kernel; PFC_RAS3D=col|v1 forces one
    int grid = 0;
    size_t d = 0;
    const char* force = getenv("PFC_RAS3D");
    const bool v1 = getenv("PFC_RAS3D_V1") != nullptr || (force && !strcmp(force, "v1"));
    ctx->ras3_col = 0;
    // (variable mobility and mirror walls run the global-scratch kernel)
    const bool plain = !c.mobility && c.bc == PFC_BC_PERIODIC;
    if (!v1 && plain && !(force && !strcmp(force, "col")) && ras3d_cl2_plan(ctx, &grid, &d))
      ctx->ras3_col = 2;
    else if (!v1 && plain && ras3d_col_plan(ctx, &d, &grid))
      ctx->ras3_col = 1;
    else
      d = ras3d_scratch_doubles(ctx, &grid);
    if (pfc_check_cuda(ctx, cudaMalloc(&ctx->ras_scratch, d * sizeof(double)), "ras scratch") ||
        pfc_check_cuda(ctx, cudaMemset(ctx->ras_scratch, 0, d * sizeof(double)), "ras scratch"))
      return fail(PFC_ENOMEM);
  }
  ctx->tail = tail_enabled(ctx);
  {  // the device-resident graph step (f1) unless the speculative-launch cycle is asked for
    const char* da = getenv("PFC_DEVICE_ARNOLDI");
    ctx->use_graph = graph_enabled(ctx) && !(da && da[0] != '0');
  }
  ctx->step_ev.resize(PFC_MAX_RESTART);
  for (auto& e : ctx->step_ev)
    if (pfc_check_cuda(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "events"))
      return fail(PFC_ECUDA);
  if (c.ras_variant != PFC_RAS_LEFT &&
      pfc_check_cuda(ctx, cudaMalloc(&ctx->ras_y, ras_ext_doubles(ctx) * sizeof(double)),
                     "ras ext-box solutions"))
    return fail(PFC_ENOMEM);
  if (c.ras_local_solver != PFC_LOCAL_GMRES) {
    pfc_status si = ilu_setup(ctx);
    if (si) return fail(si);
  }
  *out = ctx;
  return PFC_OK;
}

void pfc_destroy(pfc_ctx* ctx) {
  if (!ctx) return;
  double* fs[] = {ctx->phi, ctx->psi,   ctx->F,        ctx->Ft,       ctx->trial, ctx->S,
                  ctx->c,   ctx->w,     ctx->stage,    ctx->V,        ctx->Z,     ctx->partials,
                  ctx->dscal, ctx->ras_scratch, ctx->ras_y, ctx->mob_A, ctx->mob_t[0],
                  ctx->mob_t[1], ctx->mob_t[2]};
  for (double* f : fs)
    if (f) cudaFree(f);
  if (ctx->ticket) cudaFree(ctx->ticket);
  if (ctx->d_jcnt) cudaFree(ctx->d_jcnt);
  if (ctx->gm) cudaFree(ctx->gm);
  if (ctx->hflags) cudaFreeHost(ctx->hflags);
  for (cudaEvent_t e : ctx->step_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->hscal) cudaFreeHost(ctx->hscal);
  ilu_free(ctx);
  graph_free(ctx);
  prof_drain(ctx);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  delete ctx;
}

const char* pfc_last_error(const pfc_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

long long pfc_kernel_launches(const pfc_ctx* ctx) { return ctx ? ctx->launches : 0; }

pfc_status pfc_profile_enable(pfc_ctx* ctx, int on) {
  if (!ctx) return PFC_EINVAL;
  prof_drain(ctx);
  ctx->prof = on != 0;
  for (int i = 0; i < PFC_K_NCLASSES; ++i) {
    ctx->prof_count[i] = 0;
    ctx->prof_ms[i] = 0.0;
    ctx->prof_bytes[i] = 0.0;
    ctx->prof_flops[i] = 0.0;
  }
  ctx->ras_model_next = ctx->ras_model_cs = ctx->ras_model_nout = 0.0;
  CK(cudaMemsetAsync(ctx->d_jcnt, 0, 4 * sizeof(unsigned long long), ctx->stream), "jcnt reset");
  CK(cudaStreamSynchronize(ctx->stream), "jcnt reset");
  return PFC_OK;
}

pfc_status pfc_profile_query(pfc_ctx* ctx, int cls, long long* count, double* total_ms,
                             double* bytes, double* flops) {
  if (!ctx || cls < 0 || cls >= PFC_K_NCLASSES) return PFC_EINVAL;
  prof_drain(ctx);
  if (count) *count = ctx->prof_count[cls];
  if (total_ms) *total_ms = ctx->prof_ms[cls];
  if (bytes) *bytes = ctx->prof_bytes[cls];
  if (flops) {
    *flops = ctx->prof_flops[cls];
    if (cls == PFC_K_RAS && ctx->ras_model_next > 0.0) {   // counted Arnoldi steps
      unsigned long long j[3] = {0, 0, 0};
      CK(cudaMemcpy(j, ctx->d_jcnt, sizeof j, cudaMemcpyDeviceToHost), "jcnt read");
      const double s1 = (double)j[0], s2 = (double)j[1], nb = (double)j[2];
      *flops += ctx->ras_model_next * (ctx->ras_model_cs * s1 + 4.0 * (s2 + s1) + 3.0 * s1 +
                                       3.0 * nb) + 2.0 * s1 * ctx->ras_model_nout;
    }
  }
  return PFC_OK;
}

static pfc_status check_fields(pfc_ctx* ctx, double dt, std::initializer_list<const void*> in,
                               const void* out) {
  if (!ctx) return PFC_EINVAL;
  ctx->err.clear();
  if (!(dt > 0) || !isfinite(dt)) return pfc_fail(ctx, PFC_EINVAL, "dt must be finite and > 0");
  for (const void* p : in) {
    if (!p) return pfc_fail(ctx, PFC_EINVAL, "null field pointer");
    if (p == out) return pfc_fail(ctx, PFC_EINVAL, "output aliases an input");
    if (!is_device_ptr(p)) return pfc_fail(ctx, PFC_EINVAL, "operator fields must be device pointers");
  }
  if (!out || !is_device_ptr(out)) return pfc_fail(ctx, PFC_EINVAL, "output must be a device pointer");
  return PFC_OK;
}

pfc_status pfc_residual(pfc_ctx* ctx, const double* phi_new, const double* phi_old, double dt,
                        double* F) {
  pfc_status s = check_fields(ctx, dt, {phi_new, phi_old}, F);
  if (s) return s;
  KL(PFC_K_RESIDUAL, launch_residual(ctx, phi_new, phi_old, dt, F, nullptr, nullptr), "pfc_residual");
  return PFC_OK;
}

pfc_status pfc_jacobian_apply(pfc_ctx* ctx, const double* phi_new, const double* phi_old,
                              double dt, const double* v, double* Jv) {
  pfc_status s = check_fields(ctx, dt, {phi_new, phi_old, v}, Jv);
  if (s) return s;
  KL(PFC_K_COEF, launch_jac_state(ctx, phi_new, phi_old), "pfc_jacobian_apply coef");
  KL(PFC_K_JV, launch_jv(ctx, v, ctx->c, dt, Jv), "pfc_jacobian_apply");
  return PFC_OK;
}

pfc_status pfc_ras_apply(pfc_ctx* ctx, const double* phi_new, const double* phi_old, double dt,
                         const double* v, double* z) {
  pfc_status s = check_fields(ctx, dt, {phi_new, phi_old, v}, z);
  if (s) return s;
  KL(PFC_K_COEF, launch_jac_state(ctx, phi_new, phi_old), "pfc_ras_apply coef");
  if (ctx->cfg.ras_local_solver != PFC_LOCAL_GMRES)
    KL(PFC_K_RAS, launch_ilu_factor(ctx, ctx->c, dt), "pfc_ras_apply ilu factor");
  KL(PFC_K_RAS, launch_ras(ctx, v, ctx->c, dt, z), "pfc_ras_apply");
  return PFC_OK;
}

static pfc_status stage_in(pfc_ctx* ctx, const double* phi, const double** dev) {
  if (is_device_ptr(phi)) {
    *dev = phi;
    return PFC_OK;
  }
  CK(cudaMemcpyAsync(ctx->stage, phi, ctx->N * sizeof(double), cudaMemcpyHostToDevice, ctx->stream),
     "H2D");
  *dev = ctx->stage;
  return PFC_OK;
}

pfc_status pfc_energy(pfc_ctx* ctx, const double* phi, double* F_d) {
  if (!ctx || !phi || !F_d) return ctx ? pfc_fail(ctx, PFC_EINVAL, "null argument") : PFC_EINVAL;
  ctx->err.clear();
  const double* d = nullptr;
  pfc_status s = stage_in(ctx, phi, &d);
  if (s) return s;
  return energy_mass(ctx, d, F_d, nullptr);
}

pfc_status pfc_mass(pfc_ctx* ctx, const double* phi, double* M) {
  if (!ctx || !phi || !M) return ctx ? pfc_fail(ctx, PFC_EINVAL, "null argument") : PFC_EINVAL;
  ctx->err.clear();
  const double* d = nullptr;
  pfc_status s = stage_in(ctx, phi, &d);
  if (s) return s;
  return energy_mass(ctx, d, nullptr, M);
}

pfc_status pfc_step(pfc_ctx* ctx, double* phi, double* dt, pfc_step_info* info) {
  if (!ctx || !phi || !dt) return ctx ? pfc_fail(ctx, PFC_EINVAL, "null argument") : PFC_EINVAL;
  ctx->err.clear();
  if (!(*dt > 0) || !isfinite(*dt)) return pfc_fail(ctx, PFC_EINVAL, "dt must be finite and > 0");
  const pfc_config& c = ctx->cfg;
  const long long l0 = ctx->launches;
  pfc_step_info inf;
  memset(&inf, 0, sizeof inf);
  inf.dt_used = *dt;
  const bool dev = is_device_ptr(phi);
  const size_t bytes = ctx->N * sizeof(double);
  CK(cudaMemcpyAsync(ctx->psi, phi, bytes, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     ctx->stream),
     "load phi^n");
  pfc_status s;
  // f1: energies + Newton + FGMRES as one CUDA graph (newton_graph.cu); the profiling pass
  // (per-launch events per kernel class) runs the host loop
  if (ctx->use_graph && !ctx->prof) {
    s = newton_graph(ctx, *dt, &inf);
  } else {
    s = energy_mass(ctx, ctx->psi, &inf.energy_old, nullptr);
    if (!s) s = newton(ctx, *dt, &inf);
    if (!s) s = energy_mass(ctx, ctx->phi, &inf.energy, &inf.mass);
  }
  if (!s) {
    CK(cudaMemcpyAsync(phi, ctx->phi, bytes, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       ctx->stream),
       "store phi^{n+1}");
    CK(cudaStreamSynchronize(ctx->stream), "stream sync");
    // Eq. (sencondt) P:325-327 for the next step
    double next = *dt;
    if (c.adaptive) {
      double Fp = fabs((inf.energy - inf.energy_old) / *dt);
      next = std::max(c.dt_min, c.dt_max / sqrt(1.0 + c.eta * Fp * Fp));
    }
    inf.dt_next = next;
    *dt = next;
  }
  inf.kernel_launches = ctx->launches - l0;
  if (info) *info = inf;
  return s;
}

}  // extern "C"
