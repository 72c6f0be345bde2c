/*
 * pfc.h -- C ABI of libpfc.so: the per-time-step Newton-Krylov-Schwarz solve of the
 * DVD phase-field-crystal scheme of Wei, Yang & Huang, arXiv 1703.01202, on one B200.
 *
 * Citations: "P:n" = line n of the paper's text; equations by their LaTeX label.
 *
 * Conventions (all entry points)
 *  - Fields are fp64, contiguous, x-fastest: idx = i + n[0]*(j + n[1]*k), N = n[0]*n[1]*n[2]
 *    (n[2] = 1 in 2D).  Nodes are cell-centred x_i = (i + 1/2) h; the grid is
 *    periodic in every axis unless pfc_config.bc selects the mirror walls (ABI 5), and the
 *    mobility is M = 1 (grad_d.M_d grad_d = Delta_d) unless pfc_config.mobility
 *    selects M(phi) = 1 - phi^2 (ABI 3); the enums below define both.
 *  - Field arguments of the operator calls (pfc_residual, pfc_jacobian_apply, pfc_ras_apply)
 *    are DEVICE pointers on the context's device.  pfc_step, pfc_energy and pfc_mass accept
 *    device OR host pointers (host buffers are staged through context-owned device memory;
 *    pinned host memory makes the copies asynchronous).  16-byte alignment is recommended:
 *    it enables the TMA tile loads; unaligned pointers take a plain-load path.
 *  - Ownership: the caller owns every pointer it passes; none is retained after a call
 *    returns.  The context owns its device workspace until pfc_destroy.
 *  - Streams: all work is enqueued on the stream given to pfc_create (NULL = legacy default
 *    stream).  Operator calls are asynchronous; pfc_step, pfc_energy, pfc_mass synchronize
 *    the stream because they return host scalars.
 *  - Errors: every call returns a pfc_status; on failure nothing is partially committed
 *    except where stated, and pfc_last_error() returns a message.  A context is not
 *    reentrant: one host thread per context.
 *  - No CPU fallback: every arithmetic step runs in this library's CUDA kernels (sm_100a).
 */
#ifndef PFC_H
#define PFC_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFC_ABI_VERSION 5

typedef struct pfc_ctx pfc_ctx;
typedef int pfc_status;

enum {
  PFC_OK = 0,
  PFC_EINVAL = 1,      /* invalid argument or configuration */
  PFC_ENOMEM = 2,      /* device allocation failed */
  PFC_ECUDA = 3,       /* CUDA runtime/driver error (message in pfc_last_error) */
  PFC_ENOCONV = 4,     /* Newton hit newton_maxit or the line search hit ls_min_lambda */
  PFC_EBREAKDOWN = 5   /* non-finite residual */
};

/* Problem and solver configuration.  Defaults: pfc_config_default(). */
typedef struct pfc_config {
  int ndim;               /* 2 or 3 */
  int n[3];               /* nodes per axis (n[2] ignored and set to 1 when ndim == 2) */
  double h;               /* mesh spacing dx = dy (= dz) */
  double gamma;           /* quench depth gamma > 0 */
  int adaptive;           /* 1: adaptive dt, Eq. (sencondt); 0: fixed dt */
  double dt_min, dt_max;  /* bounds of the adaptive law */
  double eta;             /* adaptivity weight eta >= 0 */
  double newton_rtol;     /* eps_r, stop when ||F|| <= max(eps_r ||F_0||, eps_a) */
  double newton_atol;     /* eps_a */
  int newton_maxit;
  double ls_c1;           /* line search sufficient decrease ||F(Phi+lS)|| <= (1-c1 l)||F|| */
  double ls_min_lambda;   /* smallest step length before PFC_ENOCONV */
  int gmres_restart;      /* FGMRES restart length m (1..32) */
  int gmres_maxit;        /* total FGMRES iterations per Newton step */
  double gmres_rtol;      /* xi_r: ||r|| <= max(xi_r ||F||, xi_a) */
  double gmres_atol;      /* xi_a */
  int ras_box[3];         /* owned subdomain box Omega_k (nodes per axis); must divide n */
  int ras_overlap;        /* overlap o in MESH LAYERS (paper's delta = o/3) */
  int ras_local_k;        /* fixed number of local GMRES steps in each subdomain solve (1..15) */
  int ras_variant;        /* Schwarz preconditioner (enum below; default PFC_RAS_LEFT) */
  int mobility;           /* PFC_MOBILITY_ONE (M = 1, default) or PFC_MOBILITY_QUADRATIC */
  int ras_local_solver;   /* PFC_LOCAL_GMRES (default, reading R9), PFC_LOCAL_ILU, PFC_LOCAL_LU */
  int ras_ilu_level;      /* PFC_LOCAL_ILU: fill level k of ILU(k), 0..4 (Table 1) */
  int ras_ilu_reuse;      /* ILU / LU: 1 = factors of the step's first Newton iteration */
  int bc;                 /* PFC_BC_PERIODIC (default) or PFC_BC_MIRROR (enum below) */
} pfc_config;

/* Subdomain solve inv(A_k) of the Schwarz preconditioner:
 *   PFC_LOCAL_GMRES  exactly ras_local_k steps of GMRES (CGS2, Givens) on A_k, zero initial
 *                    guess (reading R9: robust at every dt of the configurations);
 *   PFC_LOCAL_ILU    the paper's ILU(k) of A_k in natural order (Table 1
 *                    P:872-909), U^{-1} L^{-1} per apply; with ras_ilu_reuse the factors of the
 *                    step's first Newton iteration (Phi_0 = phi^n) serve all its iterations
 *                    (P:910-915).  M = 1 only, either bc; usable at small dt for the configurations' h
 *                    (ILU(0) loses positive pivots near dt >= 0.5);
 *   PFC_LOCAL_LU     the paper's LU (Table 1): the same factor path with unlimited fill, i.e.
 *                    the exact factorisation of A_k in natural order (no pivoting: A_k of the
 *                    configurations keeps positive pivots, eigenvalues in [1.9, 914] at dt=0.5,
 *                    SURVEY App. A), reuse as above.  Band fill ~ 2 (3 E_x) per row: 2D ext
 *                    boxes up to the shared-memory plan (EINVAL beyond, e.g. every 3D box). */
enum { PFC_LOCAL_GMRES = 0, PFC_LOCAL_ILU = 1, PFC_LOCAL_LU = 2 };

/* Boundary conditions (row f3, reading R23):
 *   PFC_BC_PERIODIC  the paper's periodic domain, all five configurations;
 *   PFC_BC_MIRROR    the paper's "Neumann-type boundary conditions" (Test B cases c, d
 *                    P:620-621) as mirror ghosts on every axis: with the cell-centred nodes x_i = (i+1/2)h, ghost node -1-m is node m
 *                    and node n+m is node n-1-m, i.e. every operator acts on the even extension
 *                    (so D+ / D- vanish across the walls, mass is conserved and the energy
 *                    law of P:280-308 holds).  Subdomains are clipped at the walls: ext-box nodes
 *                    outside the domain are no unknowns of A_k = R_k J R_k^T.  Built for
 *                    ndim = 2 and 3 (3D since round 2), ras_box >= 3; PFC_LOCAL_GMRES with
 *                    either mobility, PFC_LOCAL_ILU / PFC_LOCAL_LU with M = 1 (identity rows
 *                    for the ext-box nodes outside the domain, one symbolic factorisation per
 *                    class of boxes by their position relative to the walls, ilu.cu).  Runs the global-memory operator chain (mobility.cu); the
 *                    subdomain solves run, in 2D for ras_local_k = 10 (any k with M = 1), the
 *                    column kernel with the basis in registers (ras2d.cu, MIR instantiation),
 *                    else the shared-memory-basis kernel, and in 3D the global-scratch kernel
 *                    (ras3d.cu) with per-box mirror ghosts; EINVAL otherwise. */
enum { PFC_BC_PERIODIC = 0, PFC_BC_MIRROR = 1 };

/* Mobility of Eq. (PFCeq) P:137-150 in the scheme's (grad . M_d grad)_d, P:208-212 (edge
 * midpoint value = average of the two end nodes), M_d = M((phi_new + phi_old)/2):
 *   PFC_MOBILITY_ONE        M = 1: (grad . M grad)_d = Delta_d (the five configurations);
 *   PFC_MOBILITY_QUADRATIC  M(phi) = 1 - phi^2 (Test B variants).  The
 *   Jacobian then carries the mobility derivative, J v = v/dt - (grad . M grad)(dA v)
 *   - (grad . (dM v) grad) A with dM v = -(phi_new+phi_old)/2 v, and the Schwarz subdomain
 *   matrix is A_k = R_k^delta J (R_k^delta)^T (Eq. Ak, reading R8b). */
enum { PFC_MOBILITY_ONE = 0, PFC_MOBILITY_QUADRATIC = 1 };

/* Schwarz preconditioner variants.  R_k^delta restricts to the extended box
 * Omega_k^delta, R_k^0 to the owned box Omega_k (zeros elsewhere on the extended box):
 *   PFC_RAS_LEFT   z = sum_k (R_k^0)^T     inv(A_k) R_k^delta v   Eq. (eq:ras) P:398-409
 *   PFC_RAS_AS     z = sum_k (R_k^delta)^T inv(A_k) R_k^delta v   Eq. (invM)
 *   PFC_RAS_RIGHT  z = sum_k (R_k^delta)^T inv(A_k) R_k^0 v       Eq. (eq:ash) P:410-419
 * The (R_k^delta)^T extension of AS / right-RAS is an overlap-add, done as a fixed-order
 * gather (deterministic); it needs one extra (#boxes x ext-box) fp64 work array. */
enum { PFC_RAS_LEFT = 0, PFC_RAS_AS = 1, PFC_RAS_RIGHT = 2 };

/* Per-step report of pfc_step. */
typedef struct pfc_step_info {
  int newton_its;         /* Newton iterations taken */
  int gmres_its;          /* total FGMRES iterations over the step */
  int ls_backtracks;      /* line-search halvings over the step */
  int converged;          /* 1 if the Newton stopping test was met */
  double dt_used;         /* Delta t_n of this step */
  double dt_next;         /* Delta t_{n+1} (adaptive law, or dt_used when fixed) */
  double res0;            /* ||F(Phi_0)||, Phi_0 = phi^n */
  double res_final;       /* ||F(Phi_final)|| */
  double energy_old;      /* F_d(phi^n), Eq. (freeenergy) */
  double energy;          /* F_d(phi^{n+1}) */
  double mass;            /* h^d sum phi^{n+1} */
  long long kernel_launches;  /* this library's kernel launches during the step */
} pfc_step_info;

/* Fill *cfg with defaults: 2D 64x64, h = pi/4, gamma = 0.25, fixed dt, eps_r = eps_a = 1e-10,
 * 50 Newton its, c1 = 1e-4, lambda_min = 1e-12, FGMRES(30) with 300 its, xi_r = 1e-3,
 * xi_a = 1e-11, RAS boxes 16^d, overlap 2, local k = 10. */
void pfc_config_default(pfc_config* cfg);

/* Create a context for `cfg` on the current CUDA device; `cuda_stream` is a cudaStream_t
 * (may be NULL).  Validates (PFC_EINVAL): ndim in {2,3}; every n_d >= 4; h > 0; gamma > 0;
 * 0 < dt_min <= dt_max when adaptive; n_d % ras_box_d == 0; 0 <= ras_overlap < ras_box_d and
 * ras_box_d + 2 ras_overlap + 6 <= n_d (the zero ring of P:429-437 must not wrap onto the box);
 * the ext box fits the subdomain kernel's shared-memory plan; 1 <= ras_local_k <= 15;
 * 1 <= gmres_restart <= 32; mobility is PFC_MOBILITY_ONE or PFC_MOBILITY_QUADRATIC (2D: the
 * ext box must fit the shared-memory subdomain kernel, at most 38^2 nodes).  Allocates the Krylov workspace (2m+1 fields
 * + 8 work fields; + 4 with PFC_MOBILITY_QUADRATIC). */
pfc_status pfc_create(const pfc_config* cfg, void* cuda_stream, pfc_ctx** out);
void pfc_destroy(pfc_ctx* ctx);

/* Residual of Eq. (NSOP) P:257-263 (with cfg.mobility; shown for M = 1):
 *   F = (phi_new - phi_old)/dt - Delta_d A(phi_new, phi_old),
 *   A = [(1-gamma) + 2 Delta_d + Delta_d^2](phi_new+phi_old)/2
 *       + (phi_new^3 + phi_new^2 phi_old + phi_new phi_old^2 + phi_old^3)/4   (Eq. discretedG)
 * Inputs/outputs: device fields of N doubles.  F must not alias an input.  dt > 0. */
pfc_status pfc_residual(pfc_ctx* ctx, const double* phi_new, const double* phi_old, double dt,
                        double* F);

/* Jacobian-vector product J v, J = dF/dphi_new (Eq. Jacobi):
 *   J v = v/dt - Delta_d[ (1/2)((1-gamma) + 2 Delta_d + Delta_d^2) v + c v ],
 *   c = (3 phi_new^2 + 2 phi_new phi_old + phi_old^2)/4.
 * Jv must not alias an input. */
pfc_status pfc_jacobian_apply(pfc_ctx* ctx, const double* phi_new, const double* phi_old,
                              double dt, const double* v, double* Jv);

/* Left restricted additive Schwarz preconditioner, Eq. (eq:ras) P:398-409:
 *   z = sum_k (R_k^0)^T inv(A_k) R_k^delta v
 * over the boxes Omega_k of cfg.ras_box (lexicographic, x fastest) extended by ras_overlap
 * mesh layers with periodic wrap.  A_k is the Jacobian at (phi_new, phi_old, dt) restricted
 * to the extended box with phi = 0 on the 3-layer ring outside it, which for
 * M = 1 equals R_k^delta J (R_k^delta)^T (Eq. Ak).  inv(A_k) is a fixed-work local solve:
 * exactly ras_local_k steps of GMRES (zero initial guess, CGS2, Givens), stopping early only
 * on exact breakdown.  Every node of z is written by exactly one box (its owner). */
pfc_status pfc_ras_apply(pfc_ctx* ctx, const double* phi_new, const double* phi_old, double dt,
                         const double* v, double* z);

/* One time step phi^n -> phi^{n+1} of Eq. (NSOP): inexact Newton from Phi_0 = phi^n
 * with backtracking line search, each Newton system J S = -F solved by
 * FGMRES(gmres_restart) right-preconditioned by pfc_ras_apply.
 *   phi : in phi^n, out phi^{n+1} (device or host pointer; in place)
 *   dt  : in Delta t_n; out Delta t_{n+1} = max(dt_min, dt_max/sqrt(1+eta F'^2)),
 *         F' = (F_d^{n+1} - F_d^n)/Delta t_n (Eq. sencondt) when adaptive, else unchanged.
 *   info: may be NULL.
 * On PFC_ENOCONV / PFC_EBREAKDOWN phi is left unchanged (phi^n) so the caller may retry with
 * a smaller dt; info still reports the failed attempt.
 * Execution: either the host-driven loop (one small D2H read per Arnoldi step and per residual
 * norm) or, with the default local GMRES solves, the whole step (both energies, Newton, line
 * search, FGMRES with restarts) as ONE CUDA graph with conditional nodes whose decisions run on
 * the device (captured once per context, dt passed as a device scalar; one D2H read per step).
 * Both give bitwise identical results and counts.  The graph is the default; environment
 * PFC_GRAPH=0 selects the host loop (so does the profiling mode, which times every launch). */
pfc_status pfc_step(pfc_ctx* ctx, double* phi, double* dt, pfc_step_info* info);

/* Discrete free energy F_d = h^d sum G_d, Eq. (relations)-(freeenergy) P:218-233:
 *   G_d = (1-gamma)/2 phi^2 + phi^4/4 + (Delta_d phi)^2/2 - sum_axis ((D+phi)^2 + (D-phi)^2)/2
 * phi: device or host; *F_d: host.  Deterministic (fixed-order two-stage reduction). */
pfc_status pfc_energy(pfc_ctx* ctx, const double* phi, double* F_d);

/* Mass M = h^d sum phi (conserved by the scheme).  phi: device or host. */
pfc_status pfc_mass(pfc_ctx* ctx, const double* phi, double* M);

/* Message of the last failed call on this context ("" if none).  Valid until the next call. */
const char* pfc_last_error(const pfc_ctx* ctx);

/* Number of this library's kernel launches on this context since creation. */
long long pfc_kernel_launches(const pfc_ctx* ctx);

/* Per-kernel-class device timing (tracing aid).  When enabled, every launch is bracketed by
 * CUDA events on the context stream (adds ~2 event records per launch); pfc_profile_query
 * synchronizes the stream and returns, for class `cls`, the number of launches, the summed
 * device time in milliseconds, and the summed ALGORITHMIC bytes and flops of those launches
 * (DESIGN.md §6 gives the per-node counts) since the last pfc_profile_enable(ctx, 1) (which
 * resets them).  Any output pointer may be NULL.
 * Classes: PFC_K_RESIDUAL, PFC_K_JV, PFC_K_RAS, PFC_K_COEF, PFC_K_ORTH (CGS2 multi-dot/axpy),
 * PFC_K_FINALIZE (reduction finalization), PFC_K_VECTOR (axpby/lincomb/norm), PFC_K_ENERGY. */
enum {
  PFC_K_RESIDUAL = 0, PFC_K_JV = 1, PFC_K_RAS = 2, PFC_K_COEF = 3, PFC_K_ORTH = 4,
  PFC_K_FINALIZE = 5, PFC_K_VECTOR = 6, PFC_K_ENERGY = 7, PFC_K_NCLASSES = 8
};
pfc_status pfc_profile_enable(pfc_ctx* ctx, int on);
pfc_status pfc_profile_query(pfc_ctx* ctx, int cls, long long* count, double* total_ms,
                             double* bytes, double* flops);

/* Host-only diagnostic (no GPU needed): the work plan of the 3D stencil kernels
 * for a grid of `ntiles` 32 x 32 xy-tiles and nz planes on nsm SMs.  plan[0] = n1, the number
 * of tiles streamed as whole z-columns (0 or a multiple of nsm); plan[1] = nzc, the number of
 * z-chunks of every other tile; plan[2] = zc, planes per chunk; plan[3] = the number of work
 * items n1 + (ntiles - n1) nzc; plan[4] = the plan's makespan in streamed planes under in-order
 * list scheduling (what the choice minimises).  two_phase = 0 restricts the choice to n1 = 0
 * (the residual kernel's plan).  Returns PFC_EINVAL for non-positive sizes or a NULL plan. */
pfc_status pfc_plan_stencil3d(int ntiles, int nz, int nsm, int two_phase, long long plan[5]);

#ifdef __cplusplus
}
#endif
#endif /* PFC_H */
