// newton_graph.cu -- the device-resident time step (NEXT row f1): the inexact Newton loop with
// its line search, the restarted FGMRES(m) inside it and the energy
// before and after, captured ONCE per context as a CUDA graph with conditional nodes and
// replayed by every pfc_step (dt is a device scalar that every dt-dependent kernel reads).  The
// host writes dt, launches one graph per step and reads one small state block back; no host
// round trip happens inside the step.
//
// Structure (WHILE / IF / SWITCH are conditional nodes; their handles are set by the host
// loop's decisions -- pfc.cu newton() / fgmres_host(), statement for statement, in the same
// floating-point operations -- run by one thread at the end of the kernel that produces their
// input, so no kernel exists only to decide):
//
//   energy(psi) -> e_old ; Phi = psi ; F(Phi) ; |F| + Newton stop        (k_fin_ctl<INIT>)
//   WHILE newton:
//     c = c(Phi, psi) ; S = 0, V_0 = -F/|F|, tol, first cycle             (k_fgm_start)
//     WHILE cycle:
//       WHILE arnoldi:
//         SWITCH j:   body j = the host loop's Arnoldi step j with j a constant:
//                     z_j = M^-1 v_j ; w = J z_j ; CGS2 ; v_{j+1} = w / h_{j+1,j} ;
//                     Givens + stop test + next j (arnoldi_close, gmres_close.cuh)
//       y = R^-1 g, stop / restart (k_backsolve_ctl) ; S += Z y
//       IF restart:  w = -F - J S ; |w| ; beta, next cycle (k_restart_ctl) ; V_0 = w / beta
//     trial = Phi + S ; F(trial) ; Armijo, and on acceptance the Newton count / stop
//     (k_fin_ctl<LS>) ; WHILE backtracking: the same with lambda halved
//     Phi = trial, F = Ft
//   energy(Phi) -> e_new
//
// The Arnoldi-step kernels are exactly the host loop's (same templates, same j), and the
// scalar decisions use the same IEEE operations (no contraction: __dmul_rn etc. where the host
// rounds a product before a sum), so the graph step is bitwise identical to the host loop.
// The accepted trial is copied into Phi / F instead of the host loop's pointer swap (the graph
// captures fixed pointers): 32 B per node per Newton iteration.
#include <chrono>
#include <cstdio>

#include "pfc_device.cuh"
#include "pfc_internal.h"

namespace {

constexpr int NT = 256;

struct NwtParams {   // the solver settings the control code needs (pfc_config)
  double newton_rtol, newton_atol, gmres_rtol, gmres_atol, ls_c1, ls_min_lambda;
  int newton_maxit, gmres_restart, gmres_maxit;
};

// kernel counts of the graph's sections (nd->kc), added to nd->launches where they run
enum { KC_PRE = 0, KC_HEAD, KC_CTAIL, KC_RESTART, KC_LS, KC_N };

// host: std::max(a, b) = (a < b) ? b : a
__device__ __forceinline__ double hmax(double a, double b) { return (a < b) ? b : a; }

// ---- the host loop's decisions (pfc.cu newton() / fgmres_host()), run by one thread at the
// end of the kernel that produces their input

// `while (!(nrm <= stop))` head of the Newton loop with its two failure exits
__device__ bool newton_continue(pfc_newton_dev* nd, int maxit) {
  if (nd->nrm <= nd->stop) return false;
  if (!isfinite(nd->nrm)) {
    nd->status = PFC_EBREAKDOWN;
    nd->why = PFC_GW_NEWTON_NONFINITE;
    return false;
  }
  if (nd->newton_its >= maxit) {
    nd->status = PFC_ENOCONV;
    nd->why = PFC_GW_NEWTON_MAXIT;
    return false;
  }
  return true;
}

// a new FGMRES cycle: g = beta e_1, j = 0
__device__ void cycle_init(pfc_gmres_dev* gm) {
  const int m = gm->m;
  for (int i = 0; i <= m; ++i) gm->g[i] = 0.0;
  gm->g[0] = gm->beta;
  gm->jm = 0;
  gm->reason = PFC_GM_RUNNING;
  gm->stop = 0;
  cudaGraphSetConditional(gm->hSW, 0u);
  cudaGraphSetConditional(gm->hA, 1u);
}

// FGMRES finished (or failed): start the line search, or leave the Newton loop on failure
__device__ void fgmres_done(pfc_newton_dev* nd, pfc_gmres_dev* gm) {
  cudaGraphSetConditional(nd->hR, 0u);
  nd->launches += gm->klaunch;   // the Arnoldi-step kernels counted by arnoldi_close
  gm->klaunch = 0;
  if (nd->status != PFC_OK) {
    cudaGraphSetConditional(nd->hLS, 0u);
    cudaGraphSetConditional(nd->hN, 0u);
    return;
  }
  nd->gmres_its += gm->its;
  nd->lambda = 1.0;
  nd->ls_t = 0;
  nd->accepted = 0;
  cudaGraphSetConditional(nd->hLS, 0u);   // the first trial's check decides on more
}

// Phi_0 = psi: |F(Phi_0)|, the Newton stopping threshold
__device__ void ctl_init(pfc_newton_dev* nd, pfc_gmres_dev* gm, const NwtParams& q, double sum) {
  const double nrm = sqrt(sum);
  nd->nrm = nrm;
  nd->n0 = nrm;
  nd->stop = hmax(__dmul_rn(q.newton_rtol, nrm), q.newton_atol);
  nd->newton_its = nd->gmres_its = nd->ls_backtracks = 0;
  nd->status = PFC_OK;
  nd->why = PFC_GW_NONE;
  nd->launches = nd->kc[KC_PRE];
  gm->klaunch = 0;
  cudaGraphSetConditional(nd->hN, newton_continue(nd, q.newton_maxit) ? 1u : 0u);
}

// Armijo test of the trial (R16): |F(Phi + lambda S)| <= (1 - c1 lambda) |F(Phi)|; at the end
// of the line search the Newton iteration's accept / count / stop (the host loop's tail)
__device__ void ctl_ls(pfc_newton_dev* nd, const NwtParams& q, double sum) {
  nd->launches += nd->kc[KC_LS];
  if (nd->status != PFC_OK) return;   // FGMRES failed: the first trial ran on garbage
  const double nt = sqrt(sum);
  const double lambda = nd->lambda;
  if (nt <= __dmul_rn(__dsub_rn(1.0, __dmul_rn(q.ls_c1, lambda)), nd->nrm)) {
    nd->accepted = 1;
    nd->nrm = nt;
    cudaGraphSetConditional(nd->hLS, 0u);
    nd->newton_its++;
    cudaGraphSetConditional(nd->hN, newton_continue(nd, q.newton_maxit) ? 1u : 0u);
    return;
  }
  nd->lambda = lambda * 0.5;
  nd->ls_backtracks++;
  nd->ls_t++;
  if (nd->ls_t <= 40 && nd->lambda >= q.ls_min_lambda) {   // next trial
    cudaGraphSetConditional(nd->hLS, 1u);
    return;
  }
  cudaGraphSetConditional(nd->hLS, 0u);
  nd->status = PFC_ENOCONV;
  nd->why = PFC_GW_LINESEARCH;
  cudaGraphSetConditional(nd->hN, 0u);
}

// fixed-order sum of one value over nblk partials (k_finalize's order, so the sums are
// bitwise those of the host loop), then the control step `mode` on thread 0
enum { CTL_INIT = 0, CTL_LS = 1 };
template <int MODE>
__global__ void __launch_bounds__(NT) k_fin_ctl(const double* __restrict__ partials, int nblk,
                                                double* __restrict__ out, pfc_newton_dev* nd,
                                                pfc_gmres_dev* gm, NwtParams q) {
  __shared__ double red[32];
  __shared__ double outv[1];
  double acc[1] = {0.0};
  for (int b = threadIdx.x; b < nblk; b += NT) acc[0] += partials[b];
  block_sum_multi<1>(acc, red, outv);
  if (threadIdx.x != 0) return;
  out[0] = outv[0];
  if (MODE == CTL_INIT) ctl_init(nd, gm, q, outv[0]);
  else ctl_ls(nd, q, outv[0]);
}

// Newton iteration head (fgmres_host's start): S = 0, V_0 = -F / |F| on the whole grid; block 0
// decides tol, the x0 = 0 exit and starts the first cycle
__global__ void k_fgm_start(pfc_newton_dev* nd, pfc_gmres_dev* gm, NwtParams q,
                            const double* __restrict__ F, double* __restrict__ V0,
                            double* __restrict__ S, size_t N) {
  const double Fnorm = nd->nrm;
  const double a = -1.0 / Fnorm, b = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x) {
    S[i] = 0.0;
    const double yi = 0.0;
    V0[i] = a * F[i] + b * yi;   // the host loop's k_axpby(-1/beta, F, 0, null)
  }
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  nd->launches += nd->kc[KC_HEAD];
  const double tol = hmax(__dmul_rn(q.gmres_rtol, Fnorm), q.gmres_atol);
  gm->tol = tol;
  gm->m = q.gmres_restart;
  gm->maxit = q.gmres_maxit;
  gm->its = 0;
  gm->graph = 1;
  if (Fnorm <= tol || Fnorm == 0.0) {
    fgmres_done(nd, gm);
    return;
  }
  gm->beta = Fnorm;
  cudaGraphSetConditional(nd->hR, 1u);
  cycle_init(gm);
}

// end of a cycle: y = R^-1 g (the host loop's back substitution), then stop / fail / restart
__global__ void k_backsolve_ctl(pfc_gmres_dev* gm, pfc_newton_dev* nd) {
  nd->launches += nd->kc[KC_CTAIL];
  const int jm = gm->jm, ld = gm->m + 1;
  for (int i = jm - 1; i >= 0; --i) {
    double s = gm->g[i];
    for (int l = i + 1; l < jm; ++l) s = __dsub_rn(s, __dmul_rn(gm->H[i + ld * l], gm->y[l]));
    gm->y[i] = s / gm->H[i + ld * i];
  }
  const int reason = gm->reason;
  if (reason == PFC_GM_NONFINITE) {
    nd->status = PFC_EBREAKDOWN;
    nd->why = PFC_GW_FGMRES_NONFINITE;
  }
  const bool restart = reason == PFC_GM_RESTART;
  cudaGraphSetConditional(nd->hRS, restart ? 1u : 0u);
  if (!restart) fgmres_done(nd, gm);
}

// restart: beta = |r| of the true residual r = -F - J S; stop if beta <= tol, else a new cycle
__global__ void k_restart_ctl(pfc_gmres_dev* gm, const double* dscal, pfc_newton_dev* nd) {
  nd->launches += nd->kc[KC_RESTART];
  const double beta = sqrt(dscal[SC_NRM]);
  if (beta <= gm->tol) {
    fgmres_done(nd, gm);
    return;
  }
  gm->beta = beta;
  gm->scal = 1.0 / beta;
  cycle_init(gm);
}

// out = a x (+ b y) with device-resident scales (the host loop's k_axpby expression)
__global__ void k_axpby_ds(const double* pa, const double* x, double a0, double b0,
                           const double* pb, const double* y, double* out, size_t N) {
  const double a = pa ? *pa : a0, b = pb ? *pb : b0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x) {
    double yi = y ? y[i] : 0.0;
    out[i] = a * x[i] + b * yi;
  }
}

// Phi = trial, F = Ft (the host loop swaps the pointers)
__global__ void k_copy2(double* __restrict__ a, const double* __restrict__ a_src,
                        double* __restrict__ b, const double* __restrict__ b_src, size_t N) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x) {
    a[i] = a_src[i];
    b[i] = b_src[i];
  }
}

int grid_pw(size_t N) {
  size_t b = (N + NT - 1) / NT;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

// ---- capture helpers: a stack of streams, one per nesting level of conditional bodies
struct Cap {
  pfc_ctx* ctx;
  cudaStream_t s[8];
  int lvl = 0;
  cudaError_t err = cudaSuccess;
  cudaStream_t cur() const { return s[lvl]; }
  void ok(cudaError_t e) {
    if (err == cudaSuccess && e != cudaSuccess) err = e;
  }
  // a handle on the top-level graph (settable from any body, as the WHILE pattern needs)
  cudaGraphConditionalHandle handle(cudaGraph_t g) {
    cudaGraphConditionalHandle h = 0;
    if (err == cudaSuccess) ok(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
    return h;
  }
  cudaGraph_t graph() {
    cudaStreamCaptureStatus cs;
    cudaGraph_t g = nullptr;
    ok(cudaStreamGetCaptureInfo(cur(), &cs, nullptr, &g, nullptr, nullptr));
    return g;
  }
  // add a conditional node behind the current level's frontier; returns its body graphs
  cudaGraph_t* node(cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type, int size) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    ok(cudaStreamGetCaptureInfo(cur(), &cs, nullptr, &g, &deps, &nd));
    if (err != cudaSuccess) return nullptr;
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = type;
    p.conditional.size = size;
    cudaGraphNode_t n;
    ok(cudaGraphAddNode(&n, g, deps, nd, &p));
    if (err != cudaSuccess) return nullptr;
    ok(cudaStreamUpdateCaptureDependencies(cur(), &n, 1, cudaStreamSetCaptureDependencies));
    return p.conditional.phGraph_out;
  }
  void open(cudaGraph_t body) {   // capture the next level into `body`
    if (err != cudaSuccess) return;
    ++lvl;
    ok(cudaStreamBeginCaptureToGraph(s[lvl], body, nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    ctx->stream = cur();
  }
  void close() {
    cudaGraph_t b = nullptr;
    ok(cudaStreamEndCapture(s[lvl], &b));
    --lvl;
    ctx->stream = cur();
  }
};

}  // namespace

// Default: the graph for the local-GMRES subdomain solves (all configurations).  A conditional
// body costs ~3 us on the device (tools/graph_cond_test.cu: a WHILE iteration of a 1-kernel
// body 4.2 us, a kernel node 1.0 us), about what a host-loop round trip costs, so the graph
// pays most where the kernels are short (cfg1 64^2: 476 -> 567 steps/s).  dt is read from the
// device state by every dt-dependent kernel, so one capture serves every dt of an adaptive run.
// PFC_GRAPH=1 / 0 forces it on / off.
int graph_enabled(pfc_ctx* ctx) {
  // the factor-based local solves decide per Newton iteration on the host (reuse)
  if (ctx->cfg.ras_local_solver != PFC_LOCAL_GMRES) return 0;
  const char* e = getenv("PFC_GRAPH");
  if (e && e[0]) return e[0] != '0';
  return 1;
}

void graph_free(pfc_ctx* ctx) {
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  ctx->gexec = nullptr;
  if (ctx->nd) cudaFree(ctx->nd);
  if (ctx->hnd) cudaFreeHost(ctx->hnd);
  ctx->nd = nullptr;
  ctx->hnd = nullptr;
}

// record the whole step (every pointer of the launches is fixed; dt is read from nd->dt, the
// launchers' host dt only fills the unused host-value fields)
static cudaError_t capture(pfc_ctx* ctx, double dt, cudaGraph_t* out) {
  const pfc_config& c = ctx->cfg;
  const size_t N = ctx->N;
  const int m = c.gmres_restart;
  NwtParams q{c.newton_rtol, c.newton_atol, c.gmres_rtol, c.gmres_atol, c.ls_c1,
              c.ls_min_lambda, c.newton_maxit, m, c.gmres_maxit};
  pfc_newton_dev* nd = ctx->nd;
  pfc_gmres_dev* gm = ctx->gm;
  double* dscal = ctx->dscal;
  Cap cp;
  cp.ctx = ctx;
  cudaStream_t user = ctx->stream;
  for (int i = 0; i < 8; ++i) cp.s[i] = nullptr;
  for (int i = 0; i < 8; ++i) cp.ok(cudaStreamCreateWithFlags(&cp.s[i], cudaStreamNonBlocking));
  const long long l_start = ctx->launches;
  long long mark = ctx->launches;
  auto since = [&]() {   // kernels captured since the last call
    const long long k = ctx->launches - mark;
    mark = ctx->launches;
    return (int)k;
  };
  int kc[KC_N] = {0};
  int kstep[PFC_MAX_RESTART] = {0};
  pfc_newton_dev hh;   // handles, written to the device with the section counts
  cudaGraphConditionalHandle hA = 0, hSW = 0;
  const bool prof = ctx->prof;
  ctx->prof = false;   // no per-launch event bracketing or accounting inside a capture
  ctx->dtdev = nd->dt;   // every dt-dependent kernel reads its dt scalars from the device state
  if (cp.err == cudaSuccess) {
    ctx->stream = cp.s[0];
    cp.ok(cudaStreamBeginCapture(cp.s[0], cudaStreamCaptureModeThreadLocal));
  }
  int np = 0;
  if (cp.err == cudaSuccess) {
    cudaGraph_t top = cp.graph();
    hh.hN = cp.handle(top);
    hh.hR = cp.handle(top);
    hh.hRS = cp.handle(top);
    hh.hLS = cp.handle(top);
    hA = cp.handle(top);
    hSW = cp.handle(top);
    // ---- energy of phi^n, Phi_0 = psi, F(Phi_0), Newton stop
    cp.ok(launch_energy_mass(ctx, ctx->psi, ctx->partials, &np));
    cp.ok(launch_finalize(ctx, ctx->partials, np, 2, nd->e_old));
    cp.ok(cudaMemcpyAsync(ctx->phi, ctx->psi, N * sizeof(double), cudaMemcpyDeviceToDevice,
                          cp.cur()));
    cp.ok(launch_residual(ctx, ctx->phi, ctx->psi, dt, ctx->F, ctx->partials, &np));
    k_fin_ctl<CTL_INIT><<<1, NT, 0, cp.cur()>>>(ctx->partials, np, dscal + SC_NRM, nd, gm, q);
    ctx->launches++;
    kc[KC_PRE] = since();
    cudaGraph_t* bN = cp.node(hh.hN, cudaGraphCondTypeWhile, 1);
    if (bN) {
      cp.open(bN[0]);   // ======== Newton iteration
      cp.ok(launch_jac_state(ctx, ctx->phi, ctx->psi));
      k_fgm_start<<<grid_pw(N), NT, 0, cp.cur()>>>(nd, gm, q, ctx->F, ctx->V, ctx->S, N);
      ctx->launches++;
      kc[KC_HEAD] = since();
      cudaGraph_t* bR = cp.node(hh.hR, cudaGraphCondTypeWhile, 1);
      if (bR) {
        cp.open(bR[0]);   // ======== FGMRES cycle
        cudaGraph_t* bA = cp.node(hA, cudaGraphCondTypeWhile, 1);
        if (bA) {
          cp.open(bA[0]);   // ======== Arnoldi step
          cudaGraph_t* bSW = cp.node(hSW, cudaGraphCondTypeSwitch, m);
          if (bSW) {
            for (int j = 0; j < m && cp.err == cudaSuccess; ++j) {
              cp.open(bSW[j]);   // ---- step j: the host loop's kernels; arnoldi_close
              double* Vj = ctx->V + (size_t)j * N;   // sets the handles (gmres_close.cuh)
              double* Zj = ctx->Z + (size_t)j * N;
              double* Vn = ctx->V + (size_t)(j + 1) * N;
              cp.ok(launch_ras(ctx, Vj, ctx->c, dt, Zj));
              if (ctx->tail) {
                cp.ok(launch_arnoldi_tail(ctx, ctx->V, Zj, ctx->c, dt, j, Vn, dscal, gm));
              } else {
                cp.ok(launch_jv(ctx, Zj, ctx->c, dt, ctx->w));
                cp.ok(launch_multidot(ctx, ctx->V, j + 1, ctx->w, ctx->partials, dscal + SC_H1));
                cp.ok(launch_axpy_dot(ctx, ctx->V, j + 1, dscal + SC_H1, ctx->w, ctx->partials,
                                      dscal + SC_H2));
                cp.ok(launch_axpy_norm_close(ctx, ctx->V, j + 1, dscal + SC_H1, dscal + SC_H2,
                                             ctx->w, ctx->partials, dscal + SC_NRM));
                if (j + 1 < m) cp.ok(launch_scale_next(ctx, ctx->w, Vn));
              }
              kstep[j] = since();
              cp.close();
            }
          }
          cp.close();
        }
        k_backsolve_ctl<<<1, 1, 0, cp.cur()>>>(gm, nd);
        ctx->launches++;
        cp.ok(launch_lincomb_dev(ctx, ctx->S, ctx->Z));   // S += Z y
        kc[KC_CTAIL] = since();
        cudaGraph_t* bRS = cp.node(hh.hRS, cudaGraphCondTypeIf, 1);
        if (bRS) {
          cp.open(bRS[0]);   // ======== restart: r = -F - J S, V_0 = r / |r|
          cp.ok(launch_jv(ctx, ctx->S, ctx->c, dt, ctx->w));
          cp.ok(launch_axpby(ctx, -1.0, ctx->F, -1.0, ctx->w, ctx->w));
          cp.ok(launch_norm2(ctx, ctx->w, ctx->partials, dscal + SC_NRM));
          k_restart_ctl<<<1, 1, 0, cp.cur()>>>(gm, dscal, nd);
          k_axpby_ds<<<grid_pw(N), NT, 0, cp.cur()>>>(&gm->scal, ctx->w, 0.0, 0.0, nullptr,
                                                       nullptr, ctx->V, N);
          ctx->launches += 2;
          kc[KC_RESTART] = since();
          cp.close();
        }
        cp.close();
      }
      // line search: the first trial (lambda = 1) outside the WHILE node, whose body then
      // runs only for backtracking trials
      auto trial = [&]() {
        k_axpby_ds<<<grid_pw(N), NT, 0, cp.cur()>>>(nullptr, ctx->phi, 1.0, 0.0, &nd->lambda,
                                                     ctx->S, ctx->trial, N);
        ctx->launches++;
        cp.ok(launch_residual(ctx, ctx->trial, ctx->psi, dt, ctx->Ft, ctx->partials, &np));
        k_fin_ctl<CTL_LS><<<1, NT, 0, cp.cur()>>>(ctx->partials, np, dscal + SC_NRM, nd, gm, q);
        ctx->launches++;
        kc[KC_LS] = since();
      };
      trial();
      cudaGraph_t* bLS = cp.node(hh.hLS, cudaGraphCondTypeWhile, 1);
      if (bLS) {
        cp.open(bLS[0]);   // ======== backtracking trial
        trial();
        cp.close();
      }
      k_copy2<<<grid_pw(N), NT, 0, cp.cur()>>>(ctx->phi, ctx->trial, ctx->F, ctx->Ft, N);
      ctx->launches++;
      kc[KC_HEAD] += since();   // (runs once per Newton iteration, like the head)
      cp.close();
    }
    // ---- energy and mass of phi^{n+1}
    cp.ok(launch_energy_mass(ctx, ctx->phi, ctx->partials, &np));
    cp.ok(launch_finalize(ctx, ctx->partials, np, 2, nd->e_new));
    ctx->g_post_launches = since();
    cudaGraph_t g = nullptr;
    cp.ok(cudaStreamEndCapture(cp.s[0], &g));
    *out = g;
  }
  cp.ok(cudaGetLastError());
  ctx->stream = user;
  ctx->prof = prof;
  ctx->dtdev = nullptr;
  ctx->launches = l_start;   // captured, not executed
  for (int i = 0; i < 8; ++i)
    if (cp.s[i]) cudaStreamDestroy(cp.s[i]);
  if (cp.err == cudaSuccess) {   // handles and section counts into the device state
    for (int i = 0; i < KC_N; ++i) hh.kc[i] = kc[i];
    cp.ok(cudaMemcpy(&nd->hN, &hh.hN, offsetof(pfc_newton_dev, kc) + sizeof(hh.kc) -
                                          offsetof(pfc_newton_dev, hN), cudaMemcpyHostToDevice));
    cp.ok(cudaMemcpy(&gm->hA, &hA, sizeof hA, cudaMemcpyHostToDevice));
    cp.ok(cudaMemcpy(&gm->hSW, &hSW, sizeof hSW, cudaMemcpyHostToDevice));
    cp.ok(cudaMemcpy(gm->kstep, kstep, sizeof kstep, cudaMemcpyHostToDevice));
  }
  return cp.err;
}

pfc_status newton_graph(pfc_ctx* ctx, double dt, pfc_step_info* inf) {
  if (!ctx->nd) {
    if (pfc_check_cuda(ctx, cudaMalloc(&ctx->nd, sizeof(pfc_newton_dev)), "newton state") ||
        pfc_check_cuda(ctx, cudaMallocHost(&ctx->hnd, 2 * sizeof(pfc_newton_dev)), "newton state"))
      return PFC_ENOMEM;
  }
  const double* ptrs[4] = {ctx->phi, ctx->F, ctx->trial, ctx->Ft};
  bool same = ctx->gexec != nullptr;
  for (int i = 0; i < 4; ++i) same = same && ctx->g_ptrs[i] == ptrs[i];
  if (!same) {
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
    cudaGraph_t g = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = capture(ctx, dt, &g);
    const auto t1 = std::chrono::steady_clock::now();
    if (e == cudaSuccess) e = cudaGraphInstantiate(&ctx->gexec, g, 0);
    const auto t2 = std::chrono::steady_clock::now();
    if (getenv("PFC_GRAPH_VERBOSE"))
      fprintf(stderr, "pfc graph: capture %.1f us, instantiate %.1f us\n",
              std::chrono::duration<double, std::micro>(t1 - t0).count(),
              std::chrono::duration<double, std::micro>(t2 - t1).count());
    if (g) cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      ctx->gexec = nullptr;
      return pfc_check_cuda(ctx, e, "newton graph capture");
    }
    for (int i = 0; i < 4; ++i) ctx->g_ptrs[i] = ptrs[i];
  }
  // dt of this step into the device state (hnd[1] is the pinned H2D source: hnd[0] receives the
  // state at the end of the previous step's launch)
  {  // the launchers' expressions (stencil2d/3d, tail2d, ras2d, ras3d*: 1/dt and W0)
    const double ih2 = ctx->ih2, ih4 = ih2 * ih2, ih6 = ih4 * ih2;
    const double al = 0.5 * (1.0 - ctx->cfg.gamma);
    double* t = ctx->hnd[1].dt;
    t[0] = dt;
    t[1] = 1.0 / dt;
    t[2] = 1.0 / dt + 4.0 * al * ih2 - 20.0 * ih4 + 56.0 * ih6;
    t[3] = 1.0 / dt + 6.0 * al * ih2 - 42.0 * ih4 + 162.0 * ih6;
  }
  pfc_status s = pfc_check_cuda(ctx, cudaMemcpyAsync(ctx->nd->dt, ctx->hnd[1].dt, 4 * sizeof(double),
                                                     cudaMemcpyHostToDevice, ctx->stream), "H2D dt");
  if (s) return s;
  s = pfc_check_cuda(ctx, cudaGraphLaunch(ctx->gexec, ctx->stream), "graph launch");
  if (s) return s;
  s = pfc_check_cuda(ctx, cudaMemcpyAsync(ctx->hnd, ctx->nd, sizeof(pfc_newton_dev),
                                          cudaMemcpyDeviceToHost, ctx->stream), "D2H state");
  if (s) return s;
  s = pfc_check_cuda(ctx, cudaStreamSynchronize(ctx->stream), "graph sync");
  if (s) return s;
  const pfc_newton_dev& h = *ctx->hnd;
  ctx->launches += h.launches + ctx->g_post_launches;
  inf->res0 = h.n0;
  inf->res_final = h.nrm;
  inf->newton_its = h.newton_its;
  inf->gmres_its = h.gmres_its;
  inf->ls_backtracks = h.ls_backtracks;
  inf->energy_old = h.e_old[0] * ctx->hd;
  inf->energy = h.e_new[0] * ctx->hd;
  inf->mass = h.e_new[1] * ctx->hd;
  switch (h.why) {
    case PFC_GW_NEWTON_NONFINITE:
      return pfc_fail(ctx, PFC_EBREAKDOWN, "Newton: non-finite residual norm");
    case PFC_GW_NEWTON_MAXIT: return pfc_fail(ctx, PFC_ENOCONV, "Newton: newton_maxit reached");
    case PFC_GW_LINESEARCH:
      return pfc_fail(ctx, PFC_ENOCONV, "Newton: line search reached ls_min_lambda");
    case PFC_GW_FGMRES_NONFINITE:
      return pfc_fail(ctx, PFC_EBREAKDOWN, "FGMRES: non-finite residual");
    default: break;
  }
  inf->converged = 1;
  return PFC_OK;
}
