/*
 * pfc_oracle.h -- CPU ORACLE for the DVD phase-field-crystal Newton-Krylov-Schwarz step
 * of Wei, Yang & Huang, arXiv 1703.01202 ("P:n" = /root/reference/PAPER.md line n).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_1703_01202_b200/,
 * include/, libpfc.so) may include, link or call this.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs use it.
 * It shares no source with the CUDA path.
 *
 * Plain, slow, sequential, fp64 (-O2 -fno-fast-math).  Fields are x-fastest:
 * idx = i + nx*(j + ny*k); 2D grids have nd=2 and n[2]=1.
 */
#ifndef PFC_ORACLE_H
#define PFC_ORACLE_H
#include <stddef.h>

typedef struct {
  int nd;      /* 2 or 3 */
  int n[3];    /* nodes per axis, n[2]=1 in 2D */
  double h;    /* uniform spacing dx=dy(=dz) */
  int bc;      /* 0: periodic (the configurations); 1: Neumann-type mirror ghosts on every
                * axis (row f3, reading R23): node -1-m mirrors node m, node n+m mirrors n-1-m */
} or_grid;

typedef struct {
  double gamma;                 /* quench depth */
  double newton_rtol, newton_atol;   /* eps_r, eps_a */
  int newton_maxit;
  double ls_c1, ls_min_lambda;  /* line search (reading R16) */
  int gmres_restart, gmres_maxit;
  double gmres_rtol, gmres_atol;     /* xi_r, xi_a */
  int ras_box[3], ras_overlap, ras_local_k;  /* Schwarz boxes, local GMRES(k) (R9) */
  int ras_variant;  /* 0 left-RAS, 1 classical AS, 2 right-RAS */
  int mobility;     /* 0: M = 1 (the configs); 1: M(phi) = 1 - phi^2 */
  int ras_local_solver;  /* 0: fixed-work local GMRES (R9); 1: ILU(level); 2: LU (row f2) */
  int ras_ilu_level;     /* fill level k of ILU(k) (Table 1); >= n gives LU */
  int ras_ilu_reuse;     /* 1 (ILU / LU): factors of the step's first Newton iteration */
} or_params;

typedef struct {
  int newton_its, gmres_its, ls_backtracks, converged;
  double res0, res_final;
} or_newton_info;

/* difference operators and the scheme */
void or_laplacian(const or_grid* g, const double* f, double* out);
void or_dvd_derivative(const or_grid* g, double gamma, const double* phi_new,
                       const double* phi_old, double* A);
void or_residual(const or_grid* g, double gamma, double dt, const double* phi_new,
                 const double* phi_old, double* F);
void or_jacobian_apply(const or_grid* g, double gamma, double dt, const double* phi_new,
                       const double* phi_old, const double* v, double* Jv);
void or_local_energy(const or_grid* g, double gamma, const double* phi, double* G);
double or_free_energy(const or_grid* g, double gamma, const double* phi);
double or_mass(const or_grid* g, const double* phi);
double or_norm2(size_t n, const double* x);

/* variable mobility */
void or_div_mgrad(const or_grid* g, const double* M, const double* f, double* out);
void or_mobility(const or_grid* g, int mobility, const double* phi_new, const double* phi_old,
                 double* M);
void or_residual_p(const or_grid* g, const or_params* p, double dt, const double* phi_new,
                   const double* phi_old, double* F);
void or_jacobian_apply_p(const or_grid* g, const or_params* p, double dt, const double* phi_new,
                         const double* phi_old, const double* v, double* Jv);

/* Schwarz preconditioner */
int or_num_boxes(const or_grid* g, const or_params* p);
void or_local_jacobian_apply(const or_grid* g, const or_params* p, double dt,
                             const double* c_loc, const double* v_loc, double* w_loc);
void or_ras_apply(const or_grid* g, const or_params* p, double dt, const double* phi_new,
                  const double* phi_old, const double* v, double* z);  /* p->ras_variant */
void or_ras_apply_box(const or_grid* g, const or_params* p, double dt, const double* phi_new,
                      const double* phi_old, const double* v, int box, double* z_owned);

/* ILU(k) of a dense n x n matrix with the pattern of its nonzeros (tests of row f2): the
 * combined factors (unit-lower L below the diagonal, U on and above) written to LU. */
void or_ilu_dense(int n, const double* A, int level, double* LU);

/* Krylov, Newton and time step control */
int or_fgmres(const or_grid* g, const or_params* p, double dt, const double* phi_new,
              const double* phi_old, const double* b, double* x, int precondition,
              int* its_out);
int or_newton(const or_grid* g, const or_params* p, double dt, const double* phi_old,
              const double* source, double* phi_new, or_newton_info* info);
double or_next_dt(double dt_min, double dt_max, double eta, double F_n, double F_nm1,
                  double dt_nm1);

#endif
