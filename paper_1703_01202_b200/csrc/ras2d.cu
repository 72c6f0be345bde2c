// ras2d.cu -- left restricted additive Schwarz apply (K4), 2D, sm_100a.
//
//   z = sum_k (R_k^0)^T inv(A_k) R_k^delta v          Eq. (eq:ras) P:398-409
//
// One CTA per subdomain box Omega_k (b_x x b_y owned nodes).  The CTA gathers v and the
// Jacobian coefficient c on the extended box Omega_k^delta (E = b + 2o nodes per axis,
// periodic wrap = restriction R_k^delta), then runs exactly k steps of GMRES on
// A_k y = R_k^delta v entirely in shared memory (reading R9: fixed-work local solve, zero
// initial guess, CGS2, Givens, early exit only on exact breakdown), and writes only the owned
// nodes (R_k^0)^T -- disjoint writes, no atomics.
//
// A_k is the local Jacobian with phi = 0 on the 3-layer ring around the extended box
// (modified subdomain BC): the Krylov vector is copied into the interior of a
// zero-padded (E+6)^2 array whose ring is never written, and the local J v is the same
// three-stage composed stencil as K2 (halo 2 -> 1 -> 0 on the padded grid):
//   L1 = Delta v,  B = ((1-gamma)/2 + c) v + L1 + Delta L1 / 2,  w = v/dt - Delta B.
// Shared memory: basis V (k+1 vectors of E^2), c, w, three padded planes, Hessenberg.
#include "pfc_device.cuh"
#include "pfc_internal.h"

namespace {

constexpr int NT = 512;
constexpr int KMAX = PFC_MAX_LOCAL_K;

struct RasArgs {
  const double* v;
  const double* c;
  double* z;
  int nx, ny;
  int bx, by, o;
  int k;
  double idt, gamma, ih2;
};

__global__ void __launch_bounds__(NT, 1) ras2d_kernel(RasArgs p) {
  extern __shared__ unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                         ~uintptr_t(127));
  const int Ex = p.bx + 2 * p.o, Ey = p.by + 2 * p.o;
  const int n = Ex * Ey;
  const int Px = Ex + 6, Py = Ey + 6;
  const int np = Px * Py;
  const int k = p.k;
  double* V = sm;                        // (k+1) n
  double* cl = V + (size_t)(k + 1) * n;  // n
  double* w = cl + n;                    // n
  double* pv = w + n;                    // np (zero ring)
  double* pl = pv + np;                  // np
  double* pb = pl + np;                  // np
  double* H = pb + np;                   // (k+1) k, column-major H[i + (k+1) j]
  double* gv = H + (k + 1) * k;          // k+1
  double* cs = gv + (k + 1);             // k
  double* sn = cs + k;                   // k
  double* yv = sn + k;                   // k
  double* hs = yv + k;                   // 2 (KMAX+1) : h1 | h2
  double* red = hs + 2 * (KMAX + 1);     // 32 (KMAX+1)
  double* scal = red + 32 * (KMAX + 1);  // 4: beta, hn, jm flag

  const int tid = threadIdx.x;
  const int nbx = p.nx / p.bx;
  const int ibx = blockIdx.x % nbx, iby = blockIdx.x / nbx;
  const int gx0 = ibx * p.bx - p.o, gy0 = iby * p.by - p.o;
  const double ih2 = p.ih2, idt = p.idt, alpha = 0.5 * (1.0 - p.gamma);

  // R_k^delta: gather v and c on the extended box (periodic wrap)
  double acc[KMAX + 1];
  acc[0] = 0.0;
  for (int l = tid; l < n; l += NT) {
    int li = l % Ex, lj = l / Ex;
    size_t g = (size_t)wrapi(gx0 + li, p.nx) + (size_t)p.nx * wrapi(gy0 + lj, p.ny);
    double vv = p.v[g];
    V[l] = vv;
    cl[l] = p.c[g];
    acc[0] += vv * vv;
  }
  for (int q = tid; q < 3 * np; q += NT) pv[q] = 0.0;   // pv, pl, pb contiguous
  for (int q = tid; q < (k + 1) * k; q += NT) H[q] = 0.0;
  for (int q = tid; q < k + 1; q += NT) gv[q] = 0.0;
  {
    double a1[1] = {acc[0]};
    block_sum_multi<1>(a1, red, scal);
  }
  const double beta = sqrt(scal[0]);
  if (beta == 0.0) {
    for (int l = tid; l < p.bx * p.by; l += NT) {
      int li = l % p.bx, lj = l / p.bx;
      p.z[(size_t)(ibx * p.bx + li) + (size_t)p.nx * (iby * p.by + lj)] = 0.0;
    }
    return;
  }
  const double ib = 1.0 / beta;
  for (int l = tid; l < n; l += NT) V[l] *= ib;
  if (tid == 0) gv[0] = beta;

  int jm = 0;
  for (int j = 0; j < k; ++j) {
    const double* Vj = V + (size_t)j * n;
    // A_k V_j: interior of the zero-padded array
    for (int l = tid; l < n; l += NT) {
      int li = l % Ex, lj = l / Ex;
      pv[(lj + 3) * Px + li + 3] = Vj[l];
    }
    __syncthreads();
    {   // L1 = Delta v on padded [1, P-1)
      const int wx = Px - 2, cnt = wx * (Py - 2);
      for (int q = tid; q < cnt; q += NT) {
        int f = (1 + q / wx) * Px + 1 + q % wx;
        pl[f] = ih2 * ((pv[f - 1] + pv[f + 1]) + (pv[f - Px] + pv[f + Px]) - 4.0 * pv[f]);
      }
    }
    __syncthreads();
    {   // B on padded [2, P-2)
      const int wx = Px - 4, cnt = wx * (Py - 4);
      for (int q = tid; q < cnt; q += NT) {
        int pi = 2 + q % wx, pj = 2 + q / wx;
        int f = pj * Px + pi;
        double vv = pv[f];
        int li = pi - 3, lj = pj - 3;
        double cv = (li >= 0 && li < Ex && lj >= 0 && lj < Ey) ? cl[lj * Ex + li] * vv : 0.0;
        double lapl = ih2 * ((pl[f - 1] + pl[f + 1]) + (pl[f - Px] + pl[f + Px]) - 4.0 * pl[f]);
        pb[f] = alpha * vv + cv + pl[f] + 0.5 * lapl;
      }
    }
    __syncthreads();
    // w = v/dt - Delta B on the box, and CGS2 pass-1 dots
#pragma unroll
    for (int i = 0; i <= KMAX; ++i) acc[i] = 0.0;
    for (int l = tid; l < n; l += NT) {
      int li = l % Ex, lj = l / Ex;
      int f = (lj + 3) * Px + li + 3;
      double lapb = ih2 * ((pb[f - 1] + pb[f + 1]) + (pb[f - Px] + pb[f + Px]) - 4.0 * pb[f]);
      double ww = pv[f] * idt - lapb;
      w[l] = ww;
#pragma unroll
      for (int i = 0; i <= KMAX; ++i)
        if (i <= j) acc[i] += V[(size_t)i * n + l] * ww;
    }
    block_sum_multi<KMAX + 1>(acc, red, hs, j + 1);
    // w -= V h1 ; pass-2 dots
#pragma unroll
    for (int i = 0; i <= KMAX; ++i) acc[i] = 0.0;
    for (int l = tid; l < n; l += NT) {
      double ww = w[l];
#pragma unroll
      for (int i = 0; i <= KMAX; ++i)
        if (i <= j) ww -= hs[i] * V[(size_t)i * n + l];
#pragma unroll
      for (int i = 0; i <= KMAX; ++i)
        if (i <= j) acc[i] += V[(size_t)i * n + l] * ww;
      w[l] = ww;
    }
    block_sum_multi<KMAX + 1>(acc, red, hs + (KMAX + 1), j + 1);
    // w -= V h2 ; |w|^2
    double a1[1] = {0.0};
    for (int l = tid; l < n; l += NT) {
      double ww = w[l];
#pragma unroll
      for (int i = 0; i <= KMAX; ++i)
        if (i <= j) ww -= hs[KMAX + 1 + i] * V[(size_t)i * n + l];
      w[l] = ww;
      a1[0] += ww * ww;
    }
    block_sum_multi<1>(a1, red, scal + 1);
    // Hessenberg column j, Givens (one thread)
    if (tid == 0) {
      const int ld = k + 1;
      const double hn = sqrt(scal[1]);
      for (int i = 0; i <= j; ++i) H[i + ld * j] = hs[i] + hs[KMAX + 1 + i];
      H[j + 1 + ld * j] = hn;
      for (int i = 0; i < j; ++i) {
        double a = H[i + ld * j], b = H[i + 1 + ld * j];
        H[i + ld * j] = cs[i] * a + sn[i] * b;
        H[i + 1 + ld * j] = -sn[i] * a + cs[i] * b;
      }
      double a = H[j + ld * j], b = H[j + 1 + ld * j];
      double r = sqrt(a * a + b * b);
      double cc = 1.0, ss = 0.0;
      if (r != 0.0) { cc = a / r; ss = b / r; }
      cs[j] = cc; sn[j] = ss;
      H[j + ld * j] = cc * a + ss * b;
      H[j + 1 + ld * j] = 0.0;
      gv[j + 1] = -ss * gv[j];
      gv[j] = cc * gv[j];
      scal[2] = (hn <= 1e-14 * beta) ? 1.0 : 0.0;
      scal[3] = hn;
    }
    __syncthreads();
    jm = j + 1;
    if (scal[2] != 0.0) break;           // exact breakdown (uniform)
    const double ihn = 1.0 / scal[3];
    double* Vn = V + (size_t)(j + 1) * n;
    for (int l = tid; l < n; l += NT) Vn[l] = w[l] * ihn;
    // (the next iteration's first __syncthreads orders these writes)
  }
  if (tid == 0) {   // back substitution R y = g
    const int ld = k + 1;
    for (int i = jm - 1; i >= 0; --i) {
      double s = gv[i];
      for (int l = i + 1; l < jm; ++l) s -= H[i + ld * l] * yv[l];
      yv[i] = s / H[i + ld * i];
    }
  }
  __syncthreads();
  // (R_k^0)^T: owned nodes only, y = V yv
  for (int l = tid; l < p.bx * p.by; l += NT) {
    int li = l % p.bx, lj = l / p.bx;
    int ll = (lj + p.o) * Ex + li + p.o;
    double s = 0.0;
    for (int i = 0; i < jm; ++i) s += yv[i] * V[(size_t)i * n + ll];
    p.z[(size_t)(ibx * p.bx + li) + (size_t)p.nx * (iby * p.by + lj)] = s;
  }
}

size_t ras2d_smem_bytes(int bx, int by, int o, int k) {
  const size_t Ex = bx + 2 * o, Ey = by + 2 * o, n = Ex * Ey, np = (Ex + 6) * (Ey + 6);
  size_t d = (size_t)(k + 1) * n + 2 * n + 3 * np + (size_t)(k + 1) * k + (k + 1) + 3 * k +
             2 * (KMAX + 1) + 32 * (KMAX + 1) + 4;
  return d * sizeof(double) + 128;
}

}  // namespace

int ras2d_plan(pfc_ctx* ctx) {
  const pfc_config& c = ctx->cfg;
  size_t sm = ras2d_smem_bytes(c.ras_box[0], c.ras_box[1], c.ras_overlap, c.ras_local_k);
  if (sm > 227 * 1024) return 0;
  ctx->ras_smem = (int)sm;
  ctx->ras_threads = NT;
  ctx->ras_cluster = 1;
  return 1;
}

cudaError_t launch_ras_2d(pfc_ctx* ctx, const double* v, const double* c, double dt, double* z) {
  const pfc_config& cf = ctx->cfg;
  static int attr_bytes = 0;
  if (ctx->ras_smem > attr_bytes) {
    cudaError_t e = cudaFuncSetAttribute(ras2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         ctx->ras_smem);
    if (e != cudaSuccess) return e;
    attr_bytes = ctx->ras_smem;
  }
  RasArgs p{v, c, z, cf.n[0], cf.n[1], cf.ras_box[0], cf.ras_box[1], cf.ras_overlap,
            cf.ras_local_k, 1.0 / dt, cf.gamma, ctx->ih2};
  const int nb = (cf.n[0] / cf.ras_box[0]) * (cf.n[1] / cf.ras_box[1]);
  ras2d_kernel<<<nb, NT, ctx->ras_smem, ctx->stream>>>(p);
  ctx->launches++;
  return cudaGetLastError();
}
