/*
 * pfc_oracle.c -- CPU ORACLE (TEST INFRASTRUCTURE ONLY; see pfc_oracle.h).
 *
 * A plain, slow, obviously-correct transcription of arXiv 1703.01202's scheme and
 * solver, in the paper's order and notation.  Every function cites the passage it
 * follows ("P:n" = PAPER.md line n; "Rk" = a reading recorded in DESIGN.md §2).
 * No blocking, fusion or reordering beyond the definitions.
 *
 * Parity pins (tests/test_oracle_*.py): Fourier symbols, constant states, the DVD
 * identity, summation by parts, the mass and energy-balance identities, the exact
 * cubic Jv identity, dense-J brute force on 8^2 / 4^3, A_k = R J R^T, local GMRES
 * exactness, FGMRES vs dense solve, Crank-Nicolson amplification, second-order
 * convergence on a manufactured solution, energy decay at large dt.
 */
#include "pfc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- grid helpers */

static size_t npts(const or_grid* g) { return (size_t)g->n[0] * g->n[1] * g->n[2]; }

static int wrapi(int i, int n) {      /* periodic index, P:125 periodic BCs */
  int r = i % n;
  return r < 0 ? r + n : r;
}

/* mirror index (reading R23): the cell-centred nodes x_i = (i+1/2)h (R2) reflected across the
 * boundary faces x = 0 and x = L, i.e. the even extension; stencil offsets are <= 3 < n */
static int mirrori(int i, int n) {
  if (i < 0) return -1 - i;
  if (i >= n) return 2 * n - 1 - i;
  return i;
}

static int axisi(const or_grid* g, int i, int n) { return g->bc ? mirrori(i, n) : wrapi(i, n); }

static size_t gidx(const or_grid* g, int i, int j, int k) {
  return (size_t)axisi(g, i, g->n[0]) +
         (size_t)g->n[0] * ((size_t)axisi(g, j, g->n[1]) + (size_t)g->n[1] * axisi(g, k, g->n[2]));
}

/* with mirror BCs the subdomains are clipped at the physical boundary (R23): an ext-box node
 * outside the domain is no unknown of A_k */
static int in_domain(const or_grid* g, int i, int j, int k) {
  if (!g->bc) return 1;
  return i >= 0 && i < g->n[0] && j >= 0 && j < g->n[1] && k >= 0 && k < g->n[2];
}

static double* alloc0(size_t n) { return (double*)calloc(n ? n : 1, sizeof(double)); }

/* Compensated (Neumaier) summation: the scalar outputs F_d and mass are sums of up to
 * 1.3e8 terms; plain left-to-right summation would carry ~N eps relative error, above
 * the 1e-12 parity bar.  Compensation changes only rounding, not the sum's definition. */
static double sum_compensated(size_t n, const double* x) {
  double s = 0.0, c = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double t = s + x[i];
    if (fabs(s) >= fabs(x[i])) c += (s - t) + x[i];
    else c += (x[i] - t) + s;
    s = t;
  }
  return s + c;
}

double or_norm2(size_t n, const double* x) {          /* Euclidean norm, R6 */
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += x[i] * x[i];
  return sqrt(s);
}

/* -------------------------------------------------- difference operators P:199-207 */

/* Delta_d = sum over axes of D^<2>, D_x^<2> phi_i = (phi_{i+1} - 2 phi_i + phi_{i-1})/dx^2
 * (P:201), periodic or mirror ghosts (g->bc, R23). */
void or_laplacian(const or_grid* g, const double* f, double* out) {
  const double ih2 = 1.0 / (g->h * g->h);
  for (int k = 0; k < g->n[2]; ++k)
    for (int j = 0; j < g->n[1]; ++j)
      for (int i = 0; i < g->n[0]; ++i) {
        double c = f[gidx(g, i, j, k)];
        double s = (f[gidx(g, i + 1, j, k)] - 2.0 * c + f[gidx(g, i - 1, j, k)]) * ih2;
        s += (f[gidx(g, i, j + 1, k)] - 2.0 * c + f[gidx(g, i, j - 1, k)]) * ih2;
        if (g->nd == 3)
          s += (f[gidx(g, i, j, k + 1)] - 2.0 * c + f[gidx(g, i, j, k - 1)]) * ih2;
        out[gidx(g, i, j, k)] = s;
      }
}

/* ------------------------------------------------------ the DVD scheme P:218-263 */

/* Discrete variational derivative, Eq. (discretedG) P:250-255:
 *   A = [(1-gamma) + 2 Delta_d + Delta_d^2] ((phi_new+phi_old)/2)
 *       + (phi_new^3 + phi_new^2 phi_old + phi_new phi_old^2 + phi_old^3)/4 */
void or_dvd_derivative(const or_grid* g, double gamma, const double* pn, const double* po,
                       double* A) {
  size_t N = npts(g);
  double* u = alloc0(N);
  double* L1 = alloc0(N);
  double* L2 = alloc0(N);
  for (size_t q = 0; q < N; ++q) u[q] = 0.5 * (pn[q] + po[q]);
  or_laplacian(g, u, L1);     /* Delta_d u */
  or_laplacian(g, L1, L2);    /* Delta_d^2 u */
  for (size_t q = 0; q < N; ++q) {
    double a = pn[q], b = po[q];
    A[q] = (1.0 - gamma) * u[q] + 2.0 * L1[q] + L2[q] +
           (a * a * a + a * a * b + a * b * b + b * b * b) / 4.0;
  }
  free(u); free(L1); free(L2);
}

/* Residual of the semi-implicit scheme, Eq. (NSOP) P:257-263 with M = 1, where
 * grad_d . M_d grad_d = Delta_d (P:208-212 with M=1, R3):
 *   F(Phi) = (Phi - psi)/dt - Delta_d A(Phi, psi)            (R5: no extra scaling) */
void or_residual(const or_grid* g, double gamma, double dt, const double* pn,
                 const double* po, double* F) {
  size_t N = npts(g);
  double* A = alloc0(N);
  double* LA = alloc0(N);
  or_dvd_derivative(g, gamma, pn, po, A);
  or_laplacian(g, A, LA);
  for (size_t q = 0; q < N; ++q) F[q] = (pn[q] - po[q]) / dt - LA[q];
  free(A); free(LA);
}

/* Jacobian-vector product, J = dF/dPhi (Eq. Jacobi), differentiating
 * Eq. (discretedG) in phi_new:
 *   dA/dPhi v = (1/2)[(1-gamma) + 2 Delta_d + Delta_d^2] v + (3Phi^2 + 2 Phi psi + psi^2)/4 v
 *   J v = v/dt - Delta_d (dA/dPhi v) */
void or_jacobian_apply(const or_grid* g, double gamma, double dt, const double* pn,
                       const double* po, const double* v, double* Jv) {
  size_t N = npts(g);
  double* L1 = alloc0(N);
  double* L2 = alloc0(N);
  double* dA = alloc0(N);
  double* LdA = alloc0(N);
  or_laplacian(g, v, L1);
  or_laplacian(g, L1, L2);
  for (size_t q = 0; q < N; ++q) {
    double a = pn[q], b = po[q];
    double c = (3.0 * a * a + 2.0 * a * b + b * b) / 4.0;
    dA[q] = 0.5 * ((1.0 - gamma) * v[q] + 2.0 * L1[q] + L2[q]) + c * v[q];
  }
  or_laplacian(g, dA, LdA);
  for (size_t q = 0; q < N; ++q) Jv[q] = v[q] / dt - LdA[q];
  free(L1); free(L2); free(dA); free(LdA);
}

/* Discrete local energy, Eq. (relations) P:218-226:
 *   G_d = (1-gamma)/2 phi^2 + phi^4/4 + (Delta_d phi)^2/2
 *         - sum_axis ((D^+ phi)^2 + (D^- phi)^2)/2 */
void or_local_energy(const or_grid* g, double gamma, const double* f, double* G) {
  size_t N = npts(g);
  double* L = alloc0(N);
  or_laplacian(g, f, L);
  const double ih = 1.0 / g->h;
  for (int k = 0; k < g->n[2]; ++k)
    for (int j = 0; j < g->n[1]; ++j)
      for (int i = 0; i < g->n[0]; ++i) {
        size_t q = gidx(g, i, j, k);
        double p = f[q];
        double grad = 0.0;
        double dp = (f[gidx(g, i + 1, j, k)] - p) * ih, dm = (p - f[gidx(g, i - 1, j, k)]) * ih;
        grad += (dp * dp + dm * dm) / 2.0;
        dp = (f[gidx(g, i, j + 1, k)] - p) * ih; dm = (p - f[gidx(g, i, j - 1, k)]) * ih;
        grad += (dp * dp + dm * dm) / 2.0;
        if (g->nd == 3) {
          dp = (f[gidx(g, i, j, k + 1)] - p) * ih; dm = (p - f[gidx(g, i, j, k - 1)]) * ih;
          grad += (dp * dp + dm * dm) / 2.0;
        }
        G[q] = (1.0 - gamma) / 2.0 * p * p + p * p * p * p / 4.0 + 0.5 * L[q] * L[q] - grad;
      }
  free(L);
}

/* Discrete free energy, Eq. (freeenergy): F_d = sum G_d dx dy (dz). */
double or_free_energy(const or_grid* g, double gamma, const double* f) {
  size_t N = npts(g);
  double* G = alloc0(N);
  or_local_energy(g, gamma, f, G);
  double s = sum_compensated(N, G);
  free(G);
  return s * pow(g->h, g->nd);
}

/* Mass h^d sum phi (conserved by the scheme). */
double or_mass(const or_grid* g, const double* f) {
  return sum_compensated(npts(g), f) * pow(g->h, g->nd);
}

/* ------------------------------------------ variable mobility P:208-212 */

/* (grad . M grad)_d f = D_x M D_x f + D_y M D_y f (+ D_z M D_z f), with the value of
 * M on the midpoint of an edge the average of its two end nodes:
 *   (D_x M D_x f)_i = [M_{i+1/2} (f_{i+1} - f_i) - M_{i-1/2} (f_i - f_{i-1})] / dx^2,
 *   M_{i+1/2} = (M_i + M_{i+1}) / 2.  Periodic. */
void or_div_mgrad(const or_grid* g, const double* M, const double* f, double* out) {
  const double ih2 = 1.0 / (g->h * g->h);
  for (int k = 0; k < g->n[2]; ++k)
    for (int j = 0; j < g->n[1]; ++j)
      for (int i = 0; i < g->n[0]; ++i) {
        size_t c = gidx(g, i, j, k);
        size_t nb[3][2] = {{gidx(g, i + 1, j, k), gidx(g, i - 1, j, k)},
                           {gidx(g, i, j + 1, k), gidx(g, i, j - 1, k)},
                           {gidx(g, i, j, k + 1), gidx(g, i, j, k - 1)}};
        double s = 0.0;
        for (int d = 0; d < g->nd; ++d) {
          double mp = (M[c] + M[nb[d][0]]) / 2.0, mm = (M[c] + M[nb[d][1]]) / 2.0;
          s += (mp * (f[nb[d][0]] - f[c]) - mm * (f[c] - f[nb[d][1]])) * ih2;
        }
        out[c] = s;
      }
}

/* M_d = M((phi_new + phi_old)/2), M(phi) = 1 - phi^2 or M = 1. */
void or_mobility(const or_grid* g, int mobility, const double* pn, const double* po, double* M) {
  size_t N = npts(g);
  for (size_t q = 0; q < N; ++q) {
    double u = (pn[q] + po[q]) / 2.0;
    M[q] = mobility ? 1.0 - u * u : 1.0;
  }
}

/* Residual of Eq. (NSOP) P:257-263 with the mobility of p:
 *   F(Phi) = (Phi - psi)/dt - (grad . M_d grad)_d A(Phi, psi).
 * With M = 1 it is or_residual (whose Delta_d is the M = 1 case of P:208-212, R3). */
void or_residual_p(const or_grid* g, const or_params* p, double dt, const double* pn,
                   const double* po, double* F) {
  if (!p->mobility) { or_residual(g, p->gamma, dt, pn, po, F); return; }
  size_t N = npts(g);
  double* A = alloc0(N);
  double* M = alloc0(N);
  double* D = alloc0(N);
  or_dvd_derivative(g, p->gamma, pn, po, A);
  or_mobility(g, p->mobility, pn, po, M);
  or_div_mgrad(g, M, A, D);
  for (size_t q = 0; q < N; ++q) F[q] = (pn[q] - po[q]) / dt - D[q];
  free(A); free(M); free(D);
}

/* J v = dF/dPhi v (Eq. Jacobi) with the mobility of p: the product rule on
 * (grad . M_d grad) A with both factors depending on Phi,
 *   J v = v/dt - (grad . M_d grad)(dA/dPhi v) - (grad . (dM_d/dPhi v) grad) A,
 *   dA/dPhi v as in or_jacobian_apply, dM_d/dPhi v = M'(u) v / 2 = -u v for M = 1 - u^2. */
void or_jacobian_apply_p(const or_grid* g, const or_params* p, double dt, const double* pn,
                         const double* po, const double* v, double* Jv) {
  if (!p->mobility) { or_jacobian_apply(g, p->gamma, dt, pn, po, v, Jv); return; }
  size_t N = npts(g);
  double* L1 = alloc0(N);
  double* L2 = alloc0(N);
  double* dA = alloc0(N);
  double* A = alloc0(N);
  double* M = alloc0(N);
  double* Mv = alloc0(N);
  double* T1 = alloc0(N);
  double* T2 = alloc0(N);
  or_laplacian(g, v, L1);
  or_laplacian(g, L1, L2);
  for (size_t q = 0; q < N; ++q) {
    double a = pn[q], b = po[q];
    double c = (3.0 * a * a + 2.0 * a * b + b * b) / 4.0;
    dA[q] = 0.5 * ((1.0 - p->gamma) * v[q] + 2.0 * L1[q] + L2[q]) + c * v[q];
    Mv[q] = -((a + b) / 2.0) * v[q];
  }
  or_dvd_derivative(g, p->gamma, pn, po, A);
  or_mobility(g, p->mobility, pn, po, M);
  or_div_mgrad(g, M, dA, T1);
  or_div_mgrad(g, Mv, A, T2);
  for (size_t q = 0; q < N; ++q) Jv[q] = v[q] / dt - T1[q] - T2[q];
  free(L1); free(L2); free(dA); free(A); free(M); free(Mv); free(T1); free(T2);
}

/* ----------------------------------------------- Schwarz preconditioner P:381-437 */

int or_num_boxes(const or_grid* g, const or_params* p) {
  int nb = 1;
  for (int d = 0; d < g->nd; ++d) nb *= g->n[d] / p->ras_box[d];
  return nb;
}

/* Local subdomain operator A_k with the modified boundary condition of P:429-437:
 * phi = 0 on the 3-layer ring Omega_k^{delta+1} \ Omega_k^delta.  The local problem
 * lives on a padded grid of E+6 nodes per axis (E = b + 2o, R7); v_loc is zero on the
 * ring and values beyond the padded grid are zero, which is the same zero extension.
 * c_loc = (3Phi^2 + 2Phi psi + psi^2)/4 on the ext box (the Jacobian coefficient of
 * or_jacobian_apply).  Layout: x-fastest on the E[0] x E[1] (x E[2]) ext box. */
void or_local_jacobian_apply(const or_grid* g, const or_params* p, double dt,
                             const double* c_loc, const double* v_loc, double* w_loc) {
  int E[3] = {1, 1, 1}, P[3] = {1, 1, 1}, R[3] = {0, 0, 0};
  for (int d = 0; d < g->nd; ++d) {
    E[d] = p->ras_box[d] + 2 * p->ras_overlap;
    P[d] = E[d] + 6;
    R[d] = 3;
  }
  size_t NP = (size_t)P[0] * P[1] * P[2];
  double* pv = alloc0(NP);
  double* L1 = alloc0(NP);
  double* L2 = alloc0(NP);
  double* dA = alloc0(NP);
  double* L3 = alloc0(NP);
  const double ih2 = 1.0 / (g->h * g->h);
#define PI(i, j, k) ((size_t)(i) + (size_t)P[0] * ((size_t)(j) + (size_t)P[1] * (size_t)(k)))
#define LI(i, j, k) ((size_t)(i) + (size_t)E[0] * ((size_t)(j) + (size_t)E[1] * (size_t)(k)))
  for (int k = 0; k < E[2]; ++k)
    for (int j = 0; j < E[1]; ++j)
      for (int i = 0; i < E[0]; ++i) pv[PI(i + R[0], j + R[1], k + R[2])] = v_loc[LI(i, j, k)];
  /* zero-Dirichlet Laplacian on the padded grid: neighbours outside it are 0 */
  double* src[3] = {pv, L1, dA};
  double* dst[3] = {L1, L2, L3};
  for (int pass = 0; pass < 3; ++pass) {
    if (pass == 2) {
      /* dA = (1/2)[(1-gamma) v + 2 Delta v + Delta^2 v] + c v, c v = 0 on the ring */
      for (int k = 0; k < P[2]; ++k)
        for (int j = 0; j < P[1]; ++j)
          for (int i = 0; i < P[0]; ++i) {
            size_t q = PI(i, j, k);
            double cv = 0.0;
            int li = i - R[0], lj = j - R[1], lk = k - R[2];
            if (li >= 0 && li < E[0] && lj >= 0 && lj < E[1] && lk >= 0 && lk < E[2])
              cv = c_loc[LI(li, lj, lk)] * pv[q];
            dA[q] = 0.5 * ((1.0 - p->gamma) * pv[q] + 2.0 * L1[q] + L2[q]) + cv;
          }
    }
    const double* s = src[pass];
    double* o = dst[pass];
    for (int k = 0; k < P[2]; ++k)
      for (int j = 0; j < P[1]; ++j)
        for (int i = 0; i < P[0]; ++i) {
          double c = s[PI(i, j, k)];
          double xm = i > 0 ? s[PI(i - 1, j, k)] : 0.0, xp = i < P[0] - 1 ? s[PI(i + 1, j, k)] : 0.0;
          double ym = j > 0 ? s[PI(i, j - 1, k)] : 0.0, yp = j < P[1] - 1 ? s[PI(i, j + 1, k)] : 0.0;
          double acc = (xp - 2.0 * c + xm) * ih2 + (yp - 2.0 * c + ym) * ih2;
          if (g->nd == 3) {
            double zm = k > 0 ? s[PI(i, j, k - 1)] : 0.0, zp = k < P[2] - 1 ? s[PI(i, j, k + 1)] : 0.0;
            acc += (zp - 2.0 * c + zm) * ih2;
          }
          o[PI(i, j, k)] = acc;
        }
  }
  for (int k = 0; k < E[2]; ++k)
    for (int j = 0; j < E[1]; ++j)
      for (int i = 0; i < E[0]; ++i) {
        size_t q = PI(i + R[0], j + R[1], k + R[2]);
        w_loc[LI(i, j, k)] = pv[q] / dt - L3[q];
      }
#undef PI
#undef LI
  free(pv); free(L1); free(L2); free(dA); free(L3);
}

/* --------------------------------------------- ILU(k) subdomain solves, row f2
 * The paper's subdomain solvers (Table 1): incomplete LU with fill level
 * k of the subdomain matrix A_k in the natural (x-fastest) order of the ext box, LU being the
 * unlimited-fill case; the preconditioner applies U^{-1} L^{-1} per box.  Fill levels by the
 * standard rule lev(i,j) = min over k < min(i,j) of lev(i,k) + lev(k,j) + 1, nonzeros of A at
 * level 0; entries with lev <= k are kept.  The numeric factorisation is the IKJ variant. */

/* factor pattern of a sparse matrix given by a dense nonzero mask (row-major n x n): returns
 * lev[n*n] (-1 = not in the pattern) */
static int* ilu_levels(int n, const unsigned char* nz, int level) {
  int* lev = (int*)malloc((size_t)n * n * sizeof(int));
  for (size_t q = 0; q < (size_t)n * n; ++q) lev[q] = nz[q] ? 0 : -1;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < i; ++k) {
      int lik = lev[(size_t)i * n + k];
      if (lik < 0) continue;
      for (int j = k + 1; j < n; ++j) {
        int lkj = lev[(size_t)k * n + j];
        if (lkj < 0) continue;
        int l = lik + lkj + 1;
        if (l > level) continue;
        int* lij = &lev[(size_t)i * n + j];
        if (*lij < 0 || l < *lij) *lij = l;
      }
    }
  return lev;
}

/* IKJ incomplete LU on the kept pattern, in place on a dense row-major copy */
static void ilu_numeric(int n, const int* lev, double* a) {
  for (int i = 1; i < n; ++i)
    for (int k = 0; k < i; ++k) {
      if (lev[(size_t)i * n + k] < 0) continue;
      a[(size_t)i * n + k] /= a[(size_t)k * n + k];
      double lik = a[(size_t)i * n + k];
      for (int j = k + 1; j < n; ++j)
        if (lev[(size_t)i * n + j] >= 0 && lev[(size_t)k * n + j] >= 0)
          a[(size_t)i * n + j] -= lik * a[(size_t)k * n + j];
    }
  for (size_t q = 0; q < (size_t)n * n; ++q)
    if (lev[q] < 0) a[q] = 0.0;
}

void or_ilu_dense(int n, const double* A, int level, double* LU) {
  unsigned char* nz = (unsigned char*)malloc((size_t)n * n);
  for (size_t q = 0; q < (size_t)n * n; ++q) nz[q] = A[q] != 0.0;
  int* lev = ilu_levels(n, nz, level);
  memcpy(LU, A, (size_t)n * n * sizeof(double));
  ilu_numeric(n, lev, LU);
  free(lev); free(nz);
}

/* y = U^{-1} L^{-1} r with the combined dense factors */
static void ilu_solve(int n, const double* LU, const double* r, double* y) {
  for (int i = 0; i < n; ++i) {
    double s = r[i];
    for (int k = 0; k < i; ++k) s -= LU[(size_t)i * n + k] * y[k];
    y[i] = s;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int j = i + 1; j < n; ++j) s -= LU[(size_t)i * n + j] * y[j];
    y[i] = s / LU[(size_t)i * n + i];
  }
}

/* Givens rotation zeroing b in (a, b): r = sqrt(a^2 + b^2), c = a/r, s = b/r. */
static void givens(double a, double b, double* c, double* s) {
  double r = sqrt(a * a + b * b);
  if (r == 0.0) { *c = 1.0; *s = 0.0; return; }
  *c = a / r; *s = b / r;
}

/* The subdomain operator of one box.  M = 1, periodic: or_local_jacobian_apply (zero ring on
 * the padded grid, R8).  Variable mobility or mirror BCs: A_k = R_k^delta J (R_k^delta)^T, the
 * "directly generated" subdomain matrix of Eq. (Ak) P:422-428 (readings R8b, R23): v_loc
 * extended by zero to the whole grid, the global J of or_jacobian_apply_p, restricted to the
 * ext box; ext-box nodes outside the domain (mirror BCs) are no unknowns: never scattered, and
 * their rows are zero. */
typedef struct {
  const or_grid* g; const or_params* p; double dt; const double* c_loc;
  const double* pn; const double* po; int x0, y0, z0, E[3];
} local_op;

static void local_apply(const local_op* L, const double* v_loc, double* w_loc) {
  if (!L->p->mobility && !L->g->bc) {
    or_local_jacobian_apply(L->g, L->p, L->dt, L->c_loc, v_loc, w_loc);
    return;
  }
  size_t N = npts(L->g);
  double* vg = alloc0(N);
  double* wg = alloc0(N);
  for (int k = 0; k < L->E[2]; ++k)                  /* (R_k^delta)^T v_loc */
    for (int j = 0; j < L->E[1]; ++j)
      for (int i = 0; i < L->E[0]; ++i)
        if (in_domain(L->g, L->x0 + i, L->y0 + j, L->z0 + k))
          vg[gidx(L->g, L->x0 + i, L->y0 + j, L->z0 + k)] =
              v_loc[(size_t)i + (size_t)L->E[0] * ((size_t)j + (size_t)L->E[1] * k)];
  or_jacobian_apply_p(L->g, L->p, L->dt, L->pn, L->po, vg, wg);
  for (int k = 0; k < L->E[2]; ++k)                  /* R_k^delta */
    for (int j = 0; j < L->E[1]; ++j)
      for (int i = 0; i < L->E[0]; ++i)
        w_loc[(size_t)i + (size_t)L->E[0] * ((size_t)j + (size_t)L->E[1] * k)] =
            in_domain(L->g, L->x0 + i, L->y0 + j, L->z0 + k)
                ? wg[gidx(L->g, L->x0 + i, L->y0 + j, L->z0 + k)] : 0.0;
  free(vg); free(wg);
}

/* Fixed-work local solve (reading R9): exactly k steps of GMRES on A_k y = r with zero
 * initial guess, classical Gram-Schmidt applied twice (CGS2), Givens least squares;
 * early exit only on exact breakdown H(j+1,j) <= 1e-14 beta. */
static void local_gmres(const local_op* L, const double* r, double* y, size_t n) {
  const or_params* p = L->p;
  int k = p->ras_local_k;
  memset(y, 0, n * sizeof(double));
  double beta = or_norm2(n, r);
  if (beta == 0.0) return;
  double* V = alloc0((size_t)(k + 1) * n);
  double* w = alloc0(n);
  double* H = alloc0((size_t)(k + 1) * k);   /* H[i + (k+1) j] */
  double* cs = alloc0(k);
  double* sn = alloc0(k);
  double* gv = alloc0(k + 1);
  double* h2 = alloc0(k + 1);
  for (size_t q = 0; q < n; ++q) V[q] = r[q] / beta;
  gv[0] = beta;
  int jm = 0;
  for (int j = 0; j < k; ++j) {
    local_apply(L, V + (size_t)j * n, w);
    for (int pass = 0; pass < 2; ++pass) {         /* CGS2 */
      for (int i = 0; i <= j; ++i) {
        double s = 0.0;
        for (size_t q = 0; q < n; ++q) s += V[(size_t)i * n + q] * w[q];
        h2[i] = s;
      }
      for (int i = 0; i <= j; ++i) {
        for (size_t q = 0; q < n; ++q) w[q] -= h2[i] * V[(size_t)i * n + q];
        H[i + (k + 1) * j] += h2[i];
      }
    }
    double hn = or_norm2(n, w);
    H[(j + 1) + (k + 1) * j] = hn;
    for (int i = 0; i < j; ++i) {                 /* apply previous rotations */
      double a = H[i + (k + 1) * j], b = H[i + 1 + (k + 1) * j];
      H[i + (k + 1) * j] = cs[i] * a + sn[i] * b;
      H[i + 1 + (k + 1) * j] = -sn[i] * a + cs[i] * b;
    }
    givens(H[j + (k + 1) * j], H[j + 1 + (k + 1) * j], &cs[j], &sn[j]);
    H[j + (k + 1) * j] = cs[j] * H[j + (k + 1) * j] + sn[j] * H[j + 1 + (k + 1) * j];
    H[j + 1 + (k + 1) * j] = 0.0;
    gv[j + 1] = -sn[j] * gv[j];
    gv[j] = cs[j] * gv[j];
    jm = j + 1;
    if (hn <= 1e-14 * beta) break;
    for (size_t q = 0; q < n; ++q) V[(size_t)(j + 1) * n + q] = w[q] / hn;
  }
  double* yy = alloc0(jm);
  for (int i = jm - 1; i >= 0; --i) {            /* back substitution R yy = g */
    double s = gv[i];
    for (int l = i + 1; l < jm; ++l) s -= H[i + (k + 1) * l] * yy[l];
    yy[i] = s / H[i + (k + 1) * i];
  }
  for (int i = 0; i < jm; ++i)
    for (size_t q = 0; q < n; ++q) y[q] += yy[i] * V[(size_t)i * n + q];
  free(yy); free(V); free(w); free(H); free(cs); free(sn); free(gv); free(h2);
}

/* inv(A_k) r by ILU(level) of the assembled A_k (row f2): A_k column q = the local operator
 * applied to the unit vector e_q (Eq. Ak P:422-428 with the modified BC, or R J R^T with
 * variable mobility), dense storage (test sizes).  The paper's "LU" (Table 1) is the
 * unlimited-fill case: level n keeps every fill entry, i.e. the exact factorisation. */
static void local_ilu(const local_op* L, const double* r, double* y, size_t n) {
  double* A = alloc0(n * n);
  double* e = alloc0(n);
  double* col = alloc0(n);
  for (size_t q = 0; q < n; ++q) {
    e[q] = 1.0;
    local_apply(L, e, col);
    for (size_t i = 0; i < n; ++i) A[i * n + q] = col[i];
    e[q] = 0.0;
  }
  for (size_t q = 0; q < n; ++q) {   /* ext-box nodes outside the domain (R23): identity rows */
    const int i = (int)(q % L->E[0]), j = (int)((q / L->E[0]) % L->E[1]), k = (int)(q / ((size_t)L->E[0] * L->E[1]));
    if (!in_domain(L->g, L->x0 + i, L->y0 + j, L->z0 + k)) A[q * n + q] = 1.0;
  }
  double* LU = alloc0(n * n);
  or_ilu_dense((int)n, A, L->p->ras_local_solver == 2 ? (int)n : L->p->ras_ilu_level, LU);
  ilu_solve((int)n, LU, r, y);
  free(A); free(e); free(col); free(LU);
}

static void local_solve(const local_op* L, const double* r, double* y, size_t n) {
  if (L->p->ras_local_solver == 1 || L->p->ras_local_solver == 2) local_ilu(L, r, y, n);
  else local_gmres(L, r, y, n);
}

/* Additive Schwarz preconditioners, selected by p->ras_variant:
 *   0  left-RAS      z = sum_k (R_k^0)^T     inv(A_k) R_k^delta v    Eq. (eq:ras)
 *   1  classical AS  z = sum_k (R_k^delta)^T inv(A_k) R_k^delta v    Eq. (invM)
 *   2  right-RAS     z = sum_k (R_k^delta)^T inv(A_k) R_k^0 v        Eq. (eq:ash)
 * Boxes Omega_k of ras_box nodes in lexicographic (x-fastest) order; Omega_k^delta
 * extends each by ras_overlap mesh layers (R7) with periodic wrap (mirror BCs: clipped at the
 * physical boundary, R23); inv(A_k) is the
 * fixed-work local GMRES (R9).  R_k^delta keeps the ext-box entries of v, R_k^0 only the
 * owned ones (zeros elsewhere on the ext box); (R_k^0)^T writes only the owned
 * nodes (disjoint), (R_k^delta)^T adds the whole ext-box solution into z,
 * accumulated in box order. */
void or_ras_apply(const or_grid* g, const or_params* p, double dt, const double* pn,
                  const double* po, const double* v, double* z) {
  int b[3] = {1, 1, 1}, nb[3] = {1, 1, 1}, E[3] = {1, 1, 1}, o[3] = {0, 0, 0};
  for (int d = 0; d < g->nd; ++d) {
    b[d] = p->ras_box[d];
    nb[d] = g->n[d] / b[d];
    o[d] = p->ras_overlap;
    E[d] = b[d] + 2 * o[d];
  }
  const int restrict_owned = p->ras_variant == 2;     /* R_k^0 restriction */
  const int extend_owned = p->ras_variant == 0;       /* (R_k^0)^T extension */
  if (!extend_owned) memset(z, 0, npts(g) * sizeof(double));
  size_t n = (size_t)E[0] * E[1] * E[2];
  double* r = alloc0(n);
  double* c = alloc0(n);
  double* y = alloc0(n);
  for (int bz = 0; bz < nb[2]; ++bz)
    for (int by = 0; by < nb[1]; ++by)
      for (int bx = 0; bx < nb[0]; ++bx) {
        int x0 = bx * b[0] - o[0], y0 = by * b[1] - o[1], z0 = bz * b[2] - o[2];
        for (int k = 0; k < E[2]; ++k)          /* R_k^delta or R_k^0: gather with wrap */
          for (int j = 0; j < E[1]; ++j)
            for (int i = 0; i < E[0]; ++i) {
              size_t q = gidx(g, x0 + i, y0 + j, z0 + k);
              size_t l = (size_t)i + (size_t)E[0] * ((size_t)j + (size_t)E[1] * k);
              int owned = i >= o[0] && i < o[0] + b[0] && j >= o[1] && j < o[1] + b[1] &&
                          k >= o[2] && k < o[2] + b[2];
              int act = in_domain(g, x0 + i, y0 + j, z0 + k);
              r[l] = ((restrict_owned && !owned) || !act) ? 0.0 : v[q];
              c[l] = (3.0 * pn[q] * pn[q] + 2.0 * pn[q] * po[q] + po[q] * po[q]) / 4.0;
            }
        local_op L = {g, p, dt, c, pn, po, x0, y0, z0, {E[0], E[1], E[2]}};
        local_solve(&L, r, y, n);
        if (extend_owned) {
          for (int k = o[2]; k < o[2] + b[2]; ++k)   /* (R_k^0)^T: owned nodes only */
            for (int j = o[1]; j < o[1] + b[1]; ++j)
              for (int i = o[0]; i < o[0] + b[0]; ++i) {
                size_t l = (size_t)i + (size_t)E[0] * ((size_t)j + (size_t)E[1] * k);
                z[gidx(g, x0 + i, y0 + j, z0 + k)] = y[l];
              }
        } else {
          for (int k = 0; k < E[2]; ++k)             /* (R_k^delta)^T: add the ext box */
            for (int j = 0; j < E[1]; ++j)
              for (int i = 0; i < E[0]; ++i) {
                size_t l = (size_t)i + (size_t)E[0] * ((size_t)j + (size_t)E[1] * k);
                if (in_domain(g, x0 + i, y0 + j, z0 + k)) z[gidx(g, x0 + i, y0 + j, z0 + k)] += y[l];
              }
        }
      }
  free(r); free(c); free(y);
}

/* The contribution of ONE box k to the left-RAS output: its owned nodes of
 * (R_k^0)^T inv(A_k) R_k^delta v, written to z_owned (b[0] x b[1] (x b[2]), x-fastest).  Same
 * steps as the box loop of or_ras_apply; used to check sampled boxes at sizes where the full
 * loop is too slow for a test. */
void or_ras_apply_box(const or_grid* g, const or_params* p, double dt, const double* pn,
                      const double* po, const double* v, int box, double* z_owned) {
  int b[3] = {1, 1, 1}, nb[3] = {1, 1, 1}, E[3] = {1, 1, 1}, o[3] = {0, 0, 0};
  for (int d = 0; d < g->nd; ++d) {
    b[d] = p->ras_box[d];
    nb[d] = g->n[d] / b[d];
    o[d] = p->ras_overlap;
    E[d] = b[d] + 2 * o[d];
  }
  int bx = box % nb[0], by = (box / nb[0]) % nb[1], bz = box / (nb[0] * nb[1]);
  size_t n = (size_t)E[0] * E[1] * E[2];
  double* r = alloc0(n);
  double* c = alloc0(n);
  double* y = alloc0(n);
  int x0 = bx * b[0] - o[0], y0 = by * b[1] - o[1], z0 = bz * b[2] - o[2];
  for (int k = 0; k < E[2]; ++k)
    for (int j = 0; j < E[1]; ++j)
      for (int i = 0; i < E[0]; ++i) {
        size_t q = gidx(g, x0 + i, y0 + j, z0 + k);
        size_t l = (size_t)i + (size_t)E[0] * ((size_t)j + (size_t)E[1] * k);
        r[l] = in_domain(g, x0 + i, y0 + j, z0 + k) ? v[q] : 0.0;
        c[l] = (3.0 * pn[q] * pn[q] + 2.0 * pn[q] * po[q] + po[q] * po[q]) / 4.0;
      }
  local_op L = {g, p, dt, c, pn, po, x0, y0, z0, {E[0], E[1], E[2]}};
  local_solve(&L, r, y, n);
  for (int k = 0; k < b[2]; ++k)
    for (int j = 0; j < b[1]; ++j)
      for (int i = 0; i < b[0]; ++i) {
        size_t l = (size_t)(i + o[0]) + (size_t)E[0] * ((size_t)(j + o[1]) + (size_t)E[1] * (k + o[2]));
        z_owned[(size_t)i + (size_t)b[0] * ((size_t)j + (size_t)b[1] * k)] = y[l];
      }
  free(r); free(c); free(y);
}

/* ------------------------------------------------- Krylov, Newton, dt */

/* Right-preconditioned GMRES, Eq. (hjacobi), in flexible form (FGMRES: the
 * preconditioned vectors Z are stored because the fixed-work local solve makes H^{-1}
 * nonlinear, R9), restarted every gmres_restart iterations, CGS2, Givens, x0 = 0.
 * Stops when ||r|| <= max(xi_r ||b||, xi_a) or after gmres_maxit its.
 * precondition = 0 runs plain GMRES (H = I) for tests.  Returns 1 if converged. */
int or_fgmres(const or_grid* g, const or_params* p, double dt, const double* pn,
              const double* po, const double* b, double* x, int precondition, int* its_out) {
  size_t N = npts(g);
  int m = p->gmres_restart;
  double* V = alloc0((size_t)(m + 1) * N);
  double* Z = alloc0((size_t)m * N);
  double* w = alloc0(N);
  double* r = alloc0(N);
  double* H = alloc0((size_t)(m + 1) * m);
  double* cs = alloc0(m);
  double* sn = alloc0(m);
  double* gv = alloc0(m + 1);
  double* hh = alloc0(m + 1);
  double* yy = alloc0(m);
  double bnorm = or_norm2(N, b);
  double tol = fmax(p->gmres_rtol * bnorm, p->gmres_atol);
  int its = 0, converged = 0;
  memset(x, 0, N * sizeof(double));
  memcpy(r, b, N * sizeof(double));
  for (;;) {
    double beta = or_norm2(N, r);
    if (beta <= tol) { converged = 1; break; }
    if (its >= p->gmres_maxit) break;
    memset(H, 0, (size_t)(m + 1) * m * sizeof(double));
    memset(gv, 0, (m + 1) * sizeof(double));
    for (size_t q = 0; q < N; ++q) V[q] = r[q] / beta;
    gv[0] = beta;
    int jm = 0, stop = 0;
    for (int j = 0; j < m; ++j) {
      double* zj = Z + (size_t)j * N;
      /* ILU with reuse (R10): the subdomain matrices of the step's first Newton
       * iteration, Phi_0 = psi */
      const double* pre = (p->ras_local_solver != 0 && p->ras_ilu_reuse) ? po : pn;
      if (precondition) or_ras_apply(g, p, dt, pre, po, V + (size_t)j * N, zj);
      else memcpy(zj, V + (size_t)j * N, N * sizeof(double));
      or_jacobian_apply_p(g, p, dt, pn, po, zj, w);
      for (int pass = 0; pass < 2; ++pass) {
        for (int i = 0; i <= j; ++i) {
          double s = 0.0;
          for (size_t q = 0; q < N; ++q) s += V[(size_t)i * N + q] * w[q];
          hh[i] = s;
        }
        for (int i = 0; i <= j; ++i) {
          for (size_t q = 0; q < N; ++q) w[q] -= hh[i] * V[(size_t)i * N + q];
          H[i + (m + 1) * j] += hh[i];
        }
      }
      double hn = or_norm2(N, w);
      H[j + 1 + (m + 1) * j] = hn;
      for (int i = 0; i < j; ++i) {
        double a = H[i + (m + 1) * j], bb = H[i + 1 + (m + 1) * j];
        H[i + (m + 1) * j] = cs[i] * a + sn[i] * bb;
        H[i + 1 + (m + 1) * j] = -sn[i] * a + cs[i] * bb;
      }
      givens(H[j + (m + 1) * j], H[j + 1 + (m + 1) * j], &cs[j], &sn[j]);
      H[j + (m + 1) * j] = cs[j] * H[j + (m + 1) * j] + sn[j] * H[j + 1 + (m + 1) * j];
      H[j + 1 + (m + 1) * j] = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      ++its;
      jm = j + 1;
      double res = fabs(gv[j + 1]);
      if (hn <= 1e-14 * beta) { stop = 1; converged = 1; break; }   /* happy breakdown */
      for (size_t q = 0; q < N; ++q) V[(size_t)(j + 1) * N + q] = w[q] / hn;
      if (res <= tol) { stop = 1; converged = 1; break; }
      if (its >= p->gmres_maxit) { stop = 1; break; }
    }
    for (int i = jm - 1; i >= 0; --i) {
      double s = gv[i];
      for (int l = i + 1; l < jm; ++l) s -= H[i + (m + 1) * l] * yy[l];
      yy[i] = s / H[i + (m + 1) * i];
    }
    for (int i = 0; i < jm; ++i)                      /* x += Z y (flexible form) */
      for (size_t q = 0; q < N; ++q) x[q] += yy[i] * Z[(size_t)i * N + q];
    if (stop) break;
    or_jacobian_apply_p(g, p, dt, pn, po, x, w);       /* true residual at restart */
    for (size_t q = 0; q < N; ++q) r[q] = b[q] - w[q];
  }
  if (its_out) *its_out = its;
  free(V); free(Z); free(w); free(r); free(H); free(cs); free(sn); free(gv); free(hh); free(yy);
  return converged;
}

/* Inexact Newton, Eqs. (newton), (Jacobi) P:344-363: Phi_0 = psi,
 * Phi_{m+1} = Phi_m + lambda_m S_m with J_m S_m = -F(Phi_m) solved by FGMRES + left-RAS;
 * lambda_m by backtracking halving with sufficient decrease
 * ||F(Phi + lambda S)|| <= (1 - c1 lambda) ||F(Phi)|| (R16);
 * stop when ||F(Phi_{m+1})|| <= max(eps_r ||F(Phi_0)||, eps_a).
 * `source` (may be NULL) is subtracted from F: used only by the manufactured-solution
 * test (R17).  Returns 1 on convergence; phi_new holds the last iterate either way. */
int or_newton(const or_grid* g, const or_params* p, double dt, const double* po,
              const double* source, double* pn, or_newton_info* info) {
  size_t N = npts(g);
  double* F = alloc0(N);
  double* Ft = alloc0(N);
  double* S = alloc0(N);
  double* b = alloc0(N);
  double* trial = alloc0(N);
  memcpy(pn, po, N * sizeof(double));
  or_residual_p(g, p, dt, pn, po, F);
  if (source) for (size_t q = 0; q < N; ++q) F[q] -= source[q];
  double n0 = or_norm2(N, F), nrm = n0;
  double stop = fmax(p->newton_rtol * n0, p->newton_atol);
  or_newton_info inf = {0, 0, 0, 0, n0, n0};
  int ok = 1;
  while (!(nrm <= stop)) {
    if (inf.newton_its >= p->newton_maxit || !isfinite(nrm)) { ok = 0; break; }
    for (size_t q = 0; q < N; ++q) b[q] = -F[q];
    int its = 0;
    or_fgmres(g, p, dt, pn, po, b, S, 1, &its);
    inf.gmres_its += its;
    double lambda = 1.0;
    int accepted = 0;
    for (int t = 0; t <= 40 && lambda >= p->ls_min_lambda; ++t) {
      for (size_t q = 0; q < N; ++q) trial[q] = pn[q] + lambda * S[q];
      or_residual_p(g, p, dt, trial, po, Ft);
      if (source) for (size_t q = 0; q < N; ++q) Ft[q] -= source[q];
      double nt = or_norm2(N, Ft);
      if (nt <= (1.0 - p->ls_c1 * lambda) * nrm) { accepted = 1; nrm = nt; break; }
      lambda *= 0.5;
      inf.ls_backtracks++;
    }
    if (!accepted) { ok = 0; break; }
    memcpy(pn, trial, N * sizeof(double));
    memcpy(F, Ft, N * sizeof(double));
    inf.newton_its++;
  }
  inf.converged = ok;
  inf.res_final = nrm;
  if (info) *info = inf;
  free(F); free(Ft); free(S); free(b); free(trial);
  return ok;
}

/* Adaptive step, Eq. (sencondt) P:325-327:
 *   dt_n = max(dt_min, dt_max / sqrt(1 + eta |F'|^2)),  F' = (F_d^n - F_d^{n-1}) / dt_{n-1} */
double or_next_dt(double dt_min, double dt_max, double eta, double F_n, double F_nm1,
                  double dt_nm1) {
  double Fp = fabs((F_n - F_nm1) / dt_nm1);
  return fmax(dt_min, dt_max / sqrt(1.0 + eta * Fp * Fp));
}
