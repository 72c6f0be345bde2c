// pfc_internal.h -- context layout and kernel launchers of libpfc.so (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/pfc.h"

#define PFC_MAX_RESTART 32
#define PFC_MAX_LOCAL_K 15

// Device-resident state of one FGMRES cycle (NEXT row f1): the Givens QR of the Hessenberg
// matrix is updated on the device at the end of every Arnoldi step, which also decides
// whether the cycle stops; `stop` gates every kernel of the following (speculatively
// launched) steps, so the host never waits between Arnoldi steps.
struct pfc_gmres_dev {
  double H[(PFC_MAX_RESTART + 1) * PFC_MAX_RESTART];   // H[i + (m+1) j], reduced to R
  double cs[PFC_MAX_RESTART], sn[PFC_MAX_RESTART];
  double g[PFC_MAX_RESTART + 1], y[PFC_MAX_RESTART];
  double beta, tol, ihn, res;
  double scal;   // graph path (f1): the scale of the next V_0 (-1/beta, then 1/|r| at a restart)
  // graph path (f1): arnoldi_close also sets the WHILE (continue the cycle) and SWITCH (next j)
  // handles and counts the kernels of step j (kstep[j]) into klaunch
  cudaGraphConditionalHandle hA, hSW;
  long long klaunch;
  int kstep[PFC_MAX_RESTART];
  int graph;
  int m, maxit;
  // read back by the host after every step (contiguous): stop flag, columns, total its, why
  int stop, jm, its, reason;
};
enum { PFC_GM_RUNNING = 0, PFC_GM_CONVERGED = 1, PFC_GM_HAPPY = 2, PFC_GM_MAXIT = 3,
       PFC_GM_RESTART = 4, PFC_GM_NONFINITE = 5 };

// Device-resident Newton state of the graph path (NEXT row f1, newton_graph.cu): the scalars
// of the inexact Newton loop with its line search, read back once per time step.
struct pfc_newton_dev {
  double nrm, n0, stop, lambda;
  double e_old[2], e_new[2];   // raw sums of G_d and phi before / after the step (x h^d on host)
  long long launches;          // kernels of this library executed by the graph
  int newton_its, gmres_its, ls_backtracks, ls_t, accepted, status, why;
  double dt[4];                // {dt, 1/dt, W0 2D, W0 3D} of the step (host-written per launch)
  // conditional-node handles (Newton, FGMRES cycle, restart section, line search) and the
  // kernel counts of the graph's sections, written by the host after the capture
  cudaGraphConditionalHandle hN, hR, hRS, hLS;
  int kc[8];
};
enum { PFC_GW_NONE = 0, PFC_GW_NEWTON_NONFINITE = 1, PFC_GW_NEWTON_MAXIT = 2,
       PFC_GW_LINESEARCH = 3, PFC_GW_FGMRES_NONFINITE = 4 };

// device-scalar slots of ctx->dscal
enum { SC_H1 = 0, SC_H2 = 32, SC_NRM = 64, SC_EN = 66, SC_TOTAL = 128 };

struct pfc_ilu;   // ILU(k) subdomain-solve structures (ilu.cu, row f2)

struct pfc_ctx {
  pfc_config cfg;
  cudaStream_t stream = nullptr;
  int device = 0;
  size_t N = 0;
  double ih2 = 0.0;        // 1/h^2
  double hd = 0.0;         // h^d (cell volume)

  // device workspace (N doubles each unless noted)
  double* phi = nullptr;   // Phi_m (Newton iterate)
  double* psi = nullptr;   // phi^n
  double* F = nullptr;     // residual at Phi_m
  double* Ft = nullptr;    // residual at a line-search trial
  double* trial = nullptr; // Phi_m + lambda S
  double* S = nullptr;     // Newton direction
  double* c = nullptr;     // Jacobian coefficient (3Phi^2 + 2Phi psi + psi^2)/4
  double* w = nullptr;     // Arnoldi work vector
  double* V = nullptr;     // (m+1) N  Krylov basis
  double* Z = nullptr;     // m N      preconditioned basis (flexible GMRES)
  double* ras_scratch = nullptr;  // 3D subdomain-solve scratch (L2-resident)
  double* ras_y = nullptr;        // AS / right-RAS: ext-box solutions [box][ext node]
  double* stage = nullptr;     // staging field for host-pointer calls
  // variable mobility (row f3): the Jacobian state A(Phi, psi) and the iterate it belongs to,
  // plus three work fields for the composed stencils
  double* mob_A = nullptr;
  double* mob_t[3] = {nullptr, nullptr, nullptr};
  const double* mob_phi = nullptr;
  const double* mob_psi = nullptr;
  pfc_ilu* ilu = nullptr;          // PFC_LOCAL_ILU: pattern, schedules and per-box factors
  double ilu_dt = 0.0;             // dt the current factors were built with
  double* partials = nullptr;  // reduction scratch
  size_t npartials = 0;
  double* dscal = nullptr;     // device scalars: [0,64) h1, [64,128) h2, [128] |w|^2, ...
  double* hscal = nullptr;     // pinned host mirror of dscal
  unsigned int* ticket = nullptr;  // last-block ticket of the fused reductions (device, 0)
  pfc_gmres_dev* gm = nullptr;     // device FGMRES cycle state (f1)
  int* hflags = nullptr;           // pinned: per-step snapshots of gm->{stop, jm, its, reason}
  std::vector<cudaEvent_t> step_ev;   // one event per Arnoldi step of a cycle
  const int* gate = nullptr;       // &gm->stop while a device-resident cycle is being launched

  // device-resident time step as one CUDA graph with conditional nodes (f1, newton_graph.cu):
  // the executable graph, the dt and field pointers it was captured with, and its state
  pfc_newton_dev* nd = nullptr;
  pfc_newton_dev* hnd = nullptr;   // pinned: [0] host mirror of *nd, [1].dt the H2D dt source
  cudaGraphExec_t gexec = nullptr;
  const double* g_ptrs[4] = {nullptr, nullptr, nullptr, nullptr};
  long long g_post_launches = 0;   // kernels after the Newton loop (counted on the host)
  // while capturing the graph: the device copy of dt every dt-dependent kernel reads
  const double* dtdev = nullptr;
  int use_graph = 0;

  // RAS launch plan
  int ras_smem = 0;
  int ras_threads = 0;
  int ras_cluster = 1;
  int ras_rows = 0;
  int ras_tmem = 0;        // 2D: the two-boxes-per-SM kernel with the basis in tensor memory
  int tail = 0;            // 2D small grids: fused J v + CGS2 + next vector (tail2d.cu)
  int tail_rs = 0;         //   its tiled form: rows per thread (0: the gather form)
  int tail_blocks = 0;     //   and co-resident tiles
  int ras3_col = 0;        // 3D: 2 = 2-CTA cluster kernel (ras3d_cl2.cu), 1 = column kernel
                           // (ras3d_col.cu), 0 = global-scratch kernel (ras3d.cu)

  long long launches = 0;
  std::string err;

  // profiling (pfc_profile_enable): event pairs per launch, accumulated per kernel class
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  struct Pending { int cls; cudaEvent_t a, b; };
  std::vector<Pending> pending;
  cudaEvent_t ev_open = nullptr;
  long long prof_count[PFC_K_NCLASSES] = {0};
  double prof_ms[PFC_K_NCLASSES] = {0};
  double prof_bytes[PFC_K_NCLASSES] = {0};   // algorithmic bytes of the launched kernels
  double prof_flops[PFC_K_NCLASSES] = {0};   // algorithmic flops
  // local-GMRES subdomain solves: flops come from the Arnoldi steps the boxes actually took
  // (device counters d_jcnt = {sum jm, sum jm^2, boxes} over the profiled launches) and the
  // per-box model of the launch (ext nodes, stencil flops per node and step, output nodes)
  unsigned long long* d_jcnt = nullptr;
  double ras_model_next = 0.0, ras_model_cs = 0.0, ras_model_nout = 0.0;
};

// record the per-box flop model of a local-GMRES subdomain-solve launch (profiling only):
// flops of a box = next (Cs jm + 4 jm (jm+1) + 3 jm + 3) + 2 jm nout
inline void ras_flop_model(pfc_ctx* ctx, double next_box, double cs, double nout_box) {
  if (ctx->prof) {
    ctx->ras_model_next = next_box;
    ctx->ras_model_cs = cs;
    ctx->ras_model_nout = nout_box;
  }
}

// algorithmic bytes/flops of a launch (counted only while profiling)
inline void pfc_account(pfc_ctx* ctx, int cls, double bytes, double flops) {
  if (ctx->prof) {
    ctx->prof_bytes[cls] += bytes;
    ctx->prof_flops[cls] += flops;
  }
}

// set ctx->err and return the status
pfc_status pfc_fail(pfc_ctx* ctx, pfc_status st, const std::string& msg);
pfc_status pfc_check_cuda(pfc_ctx* ctx, cudaError_t e, const char* where);

// ---------------------------------------------------------------- launchers (return cudaError)
// stencils (2D/3D dispatched on ctx->cfg.ndim)
cudaError_t launch_residual(pfc_ctx* ctx, const double* phi_new, const double* phi_old, double dt,
                            double* F, double* norm_partials, int* nparts);
cudaError_t launch_jv(pfc_ctx* ctx, const double* v, const double* c, double dt, double* out);
// Jacobian state of (phi_new, phi_old): c (k_coef) and, with variable mobility, A and the
// iterate pointers used by the mobility J v and the subdomain solves
cudaError_t launch_jac_state(pfc_ctx* ctx, const double* phi_new, const double* phi_old);
// variable-mobility operators (mobility.cu, 2D)
cudaError_t launch_residual_mob(pfc_ctx*, const double* phi_new, const double* phi_old, double dt,
                                double* F, double* partials, int* nparts);
cudaError_t launch_jv_mob(pfc_ctx*, const double* v, const double* c, double dt, double* out);
// the global-memory operator chain of mobility.cu serves variable mobility and mirror BCs
inline bool generic_path(const pfc_config& c) {
  return c.mobility != PFC_MOBILITY_ONE || c.bc != PFC_BC_PERIODIC;
}
cudaError_t launch_mob_state(pfc_ctx*, const double* phi_new, const double* phi_old);
// ILU(k) subdomain solves (ilu.cu)
pfc_status ilu_setup(pfc_ctx* ctx);
void ilu_free(pfc_ctx* ctx);
cudaError_t launch_ilu_factor(pfc_ctx* ctx, const double* c, double dt);
cudaError_t launch_ras_ilu(pfc_ctx* ctx, const double* v, double* z);
cudaError_t launch_energy_mass(pfc_ctx* ctx, const double* phi, double* partials, int* nparts);
cudaError_t launch_ras(pfc_ctx* ctx, const double* v, const double* c, double dt, double* z);
int ras_plan(pfc_ctx* ctx);   // fills ras_smem/threads/cluster; returns 0 if infeasible
// (R_k^delta)^T overlap-add of ctx->ras_y into z (AS, right-RAS); scratch size in doubles
cudaError_t launch_ras_extend(pfc_ctx* ctx, double* z);
size_t ras_ext_doubles(const pfc_ctx* ctx);

// per-dimension kernels
cudaError_t launch_residual_2d(pfc_ctx*, const double*, const double*, double, double*, double*,
                               int*);
cudaError_t launch_residual_3d(pfc_ctx*, const double*, const double*, double, double*, double*,
                               int*);
cudaError_t launch_jv_2d(pfc_ctx*, const double*, const double*, double, double*);
cudaError_t launch_jv_3d(pfc_ctx*, const double*, const double*, double, double*);
int ras2d_plan(pfc_ctx* ctx);
int ras3d_plan(pfc_ctx* ctx);
size_t ras3d_scratch_doubles(pfc_ctx* ctx, int* grid);
cudaError_t launch_ras_2d(pfc_ctx*, const double* v, const double* c, double dt, double* z);
cudaError_t launch_ras_3d(pfc_ctx*, const double* v, const double* c, double dt, double* z,
                          double* scratch);
int ras3d_col_plan(pfc_ctx* ctx, size_t* scratch_doubles, int* grid);
int ras3d_cl2_plan(pfc_ctx* ctx, int* clusters, size_t* scratch_doubles);
cudaError_t launch_ras_3d_cl2(pfc_ctx*, const double* v, const double* c, double dt, double* z,
                              double* scratch);
cudaError_t launch_ras_3d_col(pfc_ctx*, const double* v, const double* c, double dt, double* z,
                              double* scratch);

// fused Arnoldi tail (tail2d.cu): w = J z, CGS2, v_{j+1} = w/|w| in one cooperative kernel
int tail_enabled(pfc_ctx* ctx);
cudaError_t launch_arnoldi_tail(pfc_ctx* ctx, const double* V, const double* z, const double* c,
                                double dt, int j, double* vnext, double* out,
                                pfc_gmres_dev* gm = nullptr);

// Krylov / pointwise (krylov.cu)
int blas_nblocks(size_t N);
cudaError_t launch_coef(pfc_ctx* ctx, const double* phi, const double* psi, double* c);
cudaError_t launch_axpby(pfc_ctx* ctx, double a, const double* x, double b, const double* y,
                         double* out);
// the reductions below finish in their own last block: `out` receives the nv final sums
cudaError_t launch_multidot(pfc_ctx* ctx, const double* V, int nv, const double* w,
                            double* partials, double* out);
cudaError_t launch_axpy_dot(pfc_ctx* ctx, const double* V, int nv, const double* h, double* w,
                            double* partials, double* out);
cudaError_t launch_axpy_norm(pfc_ctx* ctx, const double* V, int nv, const double* h, double* w,
                             double* partials, double* out);
// device-resident FGMRES cycle (f1): axpy_norm + Givens update of column nv-1 in its last
// block; V_{j+1} = w / h_{j+1,j}; cycle init; back substitution + S += Z y on the device
cudaError_t launch_axpy_norm_close(pfc_ctx* ctx, const double* V, int nv, const double* h1,
                                   const double* h2, double* w, double* partials, double* out);
cudaError_t launch_scale_next(pfc_ctx* ctx, const double* w, double* vnext);
cudaError_t launch_cycle_init(pfc_ctx* ctx, double beta, double tol, int its_done);
cudaError_t launch_backsolve_lincomb(pfc_ctx* ctx, double* x, const double* Z, int jm);
// x += Z y with y, jm from the device FGMRES state (graph path)
cudaError_t launch_lincomb_dev(pfc_ctx* ctx, double* x, const double* Z);
cudaError_t launch_norm2(pfc_ctx* ctx, const double* x, double* partials, double* out);
cudaError_t launch_finalize(pfc_ctx* ctx, const double* partials, int nblk, int nval,
                            double* out);
cudaError_t launch_lincomb(pfc_ctx* ctx, double* x, const double* Z, int nv, const double* coef);

// device-resident time step (newton_graph.cu, row f1)
int graph_enabled(pfc_ctx* ctx);
pfc_status newton_graph(pfc_ctx* ctx, double dt, pfc_step_info* inf);
void graph_free(pfc_ctx* ctx);
cudaError_t launch_energy_mass_into(pfc_ctx* ctx, const double* phi, double* out2);

// TMA descriptor encoding through the driver entry point (no libcuda link dependency)
bool tma_encode(CUtensorMap* map, const double* ptr, int ndim, const int* n, const int* box);
bool tma_usable(const void* ptr);
