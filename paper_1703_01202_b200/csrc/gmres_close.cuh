// gmres_close.cuh -- end of an Arnoldi step on the device (NEXT row f1), shared by the
// device-resident FGMRES kernels (krylov.cu k_axpy_norm, tail2d.cu k_arnoldi_tail).
#pragma once

#include "pfc_internal.h"

namespace {

// End of Arnoldi step j on the device (f1): Hessenberg column j = h1 + h2 (CGS2) and
// h_{j+1,j} = ||w||, reduced by the previous Givens rotations and a new one, residual estimate
// |g_{j+1}|, and the stopping decision of the host loop it replaces: non-finite,
// happy breakdown h_{j+1,j} <= 1e-14 beta, ||r|| <= tol, its >= maxit, end of the cycle.
__device__ __noinline__ void arnoldi_close(pfc_gmres_dev* gm, int j, const double* h1, const double* h2,
                              double nrm2) {
  const int m = gm->m, ld = m + 1;
  double* H = gm->H;
  const double hn = sqrt(nrm2);
  for (int i = 0; i <= j; ++i) H[i + ld * j] = h1[i] + h2[i];
  H[j + 1 + ld * j] = hn;
  // products rounded before the sums (__dmul_rn / __dadd_rn: no FMA contraction), as the host
  // loop of pfc.cu rounds them, so the device-resident paths are bitwise equal to it
  for (int i = 0; i < j; ++i) {
    const double a = H[i + ld * j], b = H[i + 1 + ld * j];
    H[i + ld * j] = __dadd_rn(__dmul_rn(gm->cs[i], a), __dmul_rn(gm->sn[i], b));
    H[i + 1 + ld * j] = __dadd_rn(__dmul_rn(-gm->sn[i], a), __dmul_rn(gm->cs[i], b));
  }
  const double a = H[j + ld * j], b = H[j + 1 + ld * j];
  const double r = sqrt(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)));
  const double c = r == 0.0 ? 1.0 : a / r, s = r == 0.0 ? 0.0 : b / r;
  gm->cs[j] = c;
  gm->sn[j] = s;
  H[j + ld * j] = __dadd_rn(__dmul_rn(c, a), __dmul_rn(s, b));
  H[j + 1 + ld * j] = 0.0;
  gm->g[j + 1] = -s * gm->g[j];
  gm->g[j] = c * gm->g[j];
  gm->its += 1;
  gm->jm = j + 1;
  const double res = fabs(gm->g[j + 1]);
  gm->res = res;
  int reason = PFC_GM_RUNNING;
  if (!isfinite(res)) reason = PFC_GM_NONFINITE;
  else if (hn <= 1e-14 * gm->beta) reason = PFC_GM_HAPPY;
  else {
    gm->ihn = 1.0 / hn;
    if (res <= gm->tol) reason = PFC_GM_CONVERGED;
    else if (gm->its >= gm->maxit) reason = PFC_GM_MAXIT;
    else if (j + 1 == m) reason = PFC_GM_RESTART;
  }
  gm->reason = reason;
  __threadfence();
  gm->stop = reason != PFC_GM_RUNNING;
  if (gm->graph) {   // the device-resident graph step (newton_graph.cu): next SWITCH body
    gm->klaunch += gm->kstep[j];
    cudaGraphSetConditional(gm->hSW, (unsigned)(j + 1));
    cudaGraphSetConditional(gm->hA, reason == PFC_GM_RUNNING ? 1u : 0u);
  }
}

}  // namespace
