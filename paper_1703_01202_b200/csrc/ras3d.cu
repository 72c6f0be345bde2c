// ras3d.cu -- restricted / classical additive Schwarz apply (K4), 3D, sm_100a.  First version.
//
// Same algorithm as ras2d.cu (Eq. eq:ras P:398-409, modified subdomain BC P:429-437, fixed-work
// local GMRES, reading R9).  A 16^3 box with overlap 2 has 8000 extended-box unknowns, so the
// k+1 Krylov vectors (704 KB) and the zero-padded 26^3 work arrays do not fit one CTA's shared
// memory.  This version keeps them in a per-CTA global scratch region (sized for the resident
// CTAs only, so it stays mostly L2-resident) and runs a persistent grid: CTA b handles boxes
// b, b + G, b + 2G, ...  Reductions are block-level and deterministic.
#include "pfc_device.cuh"
#include "pfc_internal.h"
#include "ras_common.cuh"

namespace {

constexpr int NT = 512;
constexpr int KMAX = PFC_MAX_LOCAL_K;

struct Ras3Args {
  const double* v;
  const double* c;
  double* z;
  double* scratch;
  size_t scratch_per_cta;
  int nx, ny, nz;
  int bx, by, bz, o;
  int k;
  double idt, gamma, ih2;
  int restrict_owned;   // right-RAS: R_k^0 (v zero outside the owned box)
  double* y_ext;        // AS / right-RAS: ext-box solutions [box][ext node] for (R_k^delta)^T
  const int* gate;   // device-resident FGMRES: skip the launch when *gate != 0 (f1)
  // variable mobility (row f3): iterate Phi, psi and its A; A_k = R J R^T (reading R8b)
  const double* phi;
  const double* psi;
  const double* A;
  int mobility;
  unsigned long long* jcnt;   // profiling: Arnoldi steps taken (ras_count)
  // Neumann-type mirror BCs (row f3, reading R23; round 2 in 3D): subdomains clipped at the
  // walls (ext-box nodes outside the domain are no unknowns), the padded grid carries the
  // mirror ghosts of v (the even extension) and c of the even extension, as in ras2d_kernel
  int mirror;
  const double* dtp;   // graph path (f1): dt on the device
};

// index along an axis: periodic wrap, or the mirror partner (R23: node -1 is node 0)
__device__ __forceinline__ int axis3(int x, int n, int mirror) {
  if (!mirror) return wrapi(x, n);
  return x < 0 ? -1 - x : (x >= n ? 2 * n - 1 - x : x);
}

__global__ void __launch_bounds__(NT, 1) ras3d_kernel(Ras3Args p) {
  __shared__ double H[(KMAX + 1) * KMAX];
  __shared__ double gv[KMAX + 1], cs[KMAX], sn[KMAX], yv[KMAX];
  __shared__ double hs[2 * (KMAX + 1)];
  __shared__ double red[32 * (KMAX + 1)];
  __shared__ double scal[4];

  const int Ex = p.bx + 2 * p.o, Ey = p.by + 2 * p.o, Ez = p.bz + 2 * p.o;
  const int n = Ex * Ey * Ez;
  const int Px = Ex + 6, Py = Ey + 6, Pz = Ez + 6;
  const int np = Px * Py * Pz;
  const int PP = Px * Py;
  const int k = p.k;
  double* V = p.scratch + p.scratch_per_cta * blockIdx.x;
  double* cl = V + (size_t)(k + 1) * n;
  double* w = cl + n;
  double* pv = w + n;
  double* pl = pv + np;
  double* pb = pl + np;
  double* pm = pb + np;      // mobility: M, A, u on the padded grid (scratch sized for them)
  double* pa = pm + np;
  double* pu = pa + np;
  double* pc = pm + (p.mobility ? 3 * np : 0);                   // mirror: c of the even ext.
  int* gp = reinterpret_cast<int*>(pc + (p.mirror ? np : 0));    // mirror: ghost -> partner

  if (p.gate && *p.gate) return;
  const int tid = threadIdx.x;
  const int nbx = p.nx / p.bx, nby = p.ny / p.by, nbz = p.nz / p.bz;
  const int nboxes = nbx * nby * nbz;
  const double ih2 = p.ih2, idt = dt_inv(p.dtp, p.idt), alpha = 0.5 * (1.0 - p.gamma);
  const size_t NX = p.nx, NXY = (size_t)p.nx * p.ny;

  // zero padded arrays once (the ring is never written)
  for (int q = tid; q < 3 * np; q += NT) pv[q] = 0.0;

  for (int box = blockIdx.x; box < nboxes; box += gridDim.x) {
    const int ibx = box % nbx, iby = (box / nbx) % nby, ibz = box / (nbx * nby);
    const int gx0 = ibx * p.bx - p.o, gy0 = iby * p.by - p.o, gz0 = ibz * p.bz - p.o;
    double acc[KMAX + 1];
    acc[0] = 0.0;
    __syncthreads();
    if (p.mirror)   // the previous box may have left mirror ghosts on the ring
      for (int q = tid; q < np; q += NT) pv[q] = 0.0;
    auto in_dom = [&](int x, int y, int z) {
      return !p.mirror || (x >= 0 && x < p.nx && y >= 0 && y < p.ny && z >= 0 && z < p.nz);
    };
    for (int l = tid; l < n; l += NT) {
      int li = l % Ex, lj = (l / Ex) % Ey, lk = l / (Ex * Ey);
      const bool act = in_dom(gx0 + li, gy0 + lj, gz0 + lk);   // an unknown of A_k
      size_t g = (size_t)axis3(gx0 + li, p.nx, p.mirror) + NX * axis3(gy0 + lj, p.ny, p.mirror) +
                 NXY * axis3(gz0 + lk, p.nz, p.mirror);
      const bool owned = li >= p.o && li < p.o + p.bx && lj >= p.o && lj < p.o + p.by &&
                         lk >= p.o && lk < p.o + p.bz;
      double vv = ((p.restrict_owned && !owned) || !act) ? 0.0 : p.v[g];
      V[l] = vv;
      cl[l] = p.c[g];
      acc[0] += vv * vv;
    }
    // mirror: does this box's padded grid reach past a wall (then it has ghost positions)?
    const bool ghosts = p.mirror && (gx0 - 3 < 0 || gy0 - 3 < 0 || gz0 - 3 < 0 ||
                                     gx0 + Px - 3 > p.nx || gy0 + Py - 3 > p.ny ||
                                     gz0 + Pz - 3 > p.nz);
    if (p.mirror) {   // c of the even extension on the padded grid; ghost -> partner map
      for (int q = tid; q < np; q += NT) {
        const int pi = q % Px, pj = (q / Px) % Py, pk = q / PP;
        const int x = gx0 + pi - 3, y = gy0 + pj - 3, z = gz0 + pk - 3;
        const bool inext = pi >= 3 && pi < Px - 3 && pj >= 3 && pj < Py - 3 && pk >= 3 &&
                           pk < Pz - 3;
        const bool ghost = !in_dom(x, y, z);
        const size_t g = (size_t)axis3(x, p.nx, 1) + NX * axis3(y, p.ny, 1) +
                         NXY * axis3(z, p.nz, 1);
        pc[q] = (inext || ghost) ? p.c[g] : 0.0;
        int part = -1;
        if (ghost) {   // the mirror image inside the ext box, else the zero of the modified BC
          const int mi = axis3(x, p.nx, 1) - gx0 + 3, mj = axis3(y, p.ny, 1) - gy0 + 3,
                    mk = axis3(z, p.nz, 1) - gz0 + 3;
          part = (mi >= 3 && mi < Px - 3 && mj >= 3 && mj < Py - 3 && mk >= 3 && mk < Pz - 3)
                     ? mk * PP + mj * Px + mi : -2;
        }
        gp[q] = part;
      }
    }
    if (p.mobility) {   // M = 1 - u^2, A, u of the iterate on the ext box and its +1 ring
      for (int q = tid; q < np; q += NT) {
        const int pi = q % Px, pj = (q / Px) % Py, pk = q / PP;
        double m = 0.0, a = 0.0, u = 0.0;
        if (pi >= 2 && pi < Px - 2 && pj >= 2 && pj < Py - 2 && pk >= 2 && pk < Pz - 2) {
          const size_t g = (size_t)axis3(gx0 + pi - 3, p.nx, p.mirror) +
                           NX * axis3(gy0 + pj - 3, p.ny, p.mirror) +
                           NXY * axis3(gz0 + pk - 3, p.nz, p.mirror);   // mirror: even ext.
          u = 0.5 * (p.phi[g] + p.psi[g]);
          m = 1.0 - u * u;
          a = p.A[g];
        }
        pm[q] = m; pa[q] = a; pu[q] = u;
      }
    }
    for (int q = tid; q < (k + 1) * k; q += NT) H[q] = 0.0;
    for (int q = tid; q < k + 1; q += NT) gv[q] = 0.0;
    {
      double a1[1] = {acc[0]};
      block_sum_multi<1>(a1, red, scal);
    }
    const double beta = sqrt(scal[0]);
    if (beta == 0.0) {
      if (tid == 0) ras_count(p.jcnt, 0);
      if (p.y_ext) {
        for (int l = tid; l < n; l += NT) p.y_ext[(size_t)box * n + l] = 0.0;
        continue;
      }
      for (int l = tid; l < p.bx * p.by * p.bz; l += NT) {
        int li = l % p.bx, lj = (l / p.bx) % p.by, lk = l / (p.bx * p.by);
        p.z[(size_t)(ibx * p.bx + li) + NX * (iby * p.by + lj) + NXY * (ibz * p.bz + lk)] = 0.0;
      }
      continue;
    }
    const double ib = 1.0 / beta;
    for (int l = tid; l < n; l += NT) V[l] *= ib;
    if (tid == 0) gv[0] = beta;

    int jm = 0;
    for (int j = 0; j < k; ++j) {
      const double* Vj = V + (size_t)j * n;
      for (int l = tid; l < n; l += NT) {
        int li = l % Ex, lj = (l / Ex) % Ey, lk = l / (Ex * Ey);
        pv[(lk + 3) * PP + (lj + 3) * Px + li + 3] = Vj[l];
      }
      __syncthreads();
      if (ghosts) {   // mirror ghosts of V_j (the even extension; partners outside the box: 0)
        for (int q = tid; q < np; q += NT) {
          const int g = gp[q];
          if (g >= 0) pv[q] = pv[g];
          else if (g == -2) pv[q] = 0.0;
        }
        __syncthreads();
      }
      {
        const int wx = Px - 2, wy = Py - 2, cnt = wx * wy * (Pz - 2);
        for (int q = tid; q < cnt; q += NT) {
          int f = (1 + q / (wx * wy)) * PP + (1 + (q / wx) % wy) * Px + 1 + q % wx;
          pl[f] = ih2 * ((pv[f - 1] + pv[f + 1]) + (pv[f - Px] + pv[f + Px]) +
                         (pv[f - PP] + pv[f + PP]) - 6.0 * pv[f]);
        }
      }
      __syncthreads();
      {
        const int wx = Px - 4, wy = Py - 4, cnt = wx * wy * (Pz - 4);
        for (int q = tid; q < cnt; q += NT) {
          int pi = 2 + q % wx, pj = 2 + (q / wx) % wy, pk = 2 + q / (wx * wy);
          int f = pk * PP + pj * Px + pi;
          double vv = pv[f];
          int li = pi - 3, lj = pj - 3, lk = pk - 3;
          double cv = p.mirror ? pc[f] * vv
                      : (li >= 0 && li < Ex && lj >= 0 && lj < Ey && lk >= 0 && lk < Ez)
                          ? cl[(lk * Ey + lj) * Ex + li] * vv
                          : 0.0;
          double lapl = ih2 * ((pl[f - 1] + pl[f + 1]) + (pl[f - Px] + pl[f + Px]) +
                               (pl[f - PP] + pl[f + PP]) - 6.0 * pl[f]);
          pb[f] = alpha * vv + cv + pl[f] + 0.5 * lapl;
        }
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i <= KMAX; ++i) acc[i] = 0.0;
      for (int l = tid; l < n; l += NT) {
        int li = l % Ex, lj = (l / Ex) % Ey, lk = l / (Ex * Ey);
        int f = (lk + 3) * PP + (lj + 3) * Px + li + 3;
        double ww;
        if (p.mobility) {   // v/dt - (grad . M grad) B - (grad . (-u v) grad) A
          auto dmg = [&](const double* mm0, const double* g, bool dm) {
            auto mm = [&](int q) { return dm ? -pu[q] * pv[q] : mm0[q]; };
            const double mc = mm(f), gc = g[f];
            double s = 0.0;
            const int off[3] = {1, Px, PP};
            for (int d = 0; d < 3; ++d)
              s += 0.5 * (mc + mm(f + off[d])) * (g[f + off[d]] - gc) -
                   0.5 * (mc + mm(f - off[d])) * (gc - g[f - off[d]]);
            return ih2 * s;
          };
          ww = pv[f] * idt - dmg(pm, pb, false) - dmg(nullptr, pa, true);
        } else {
          double lapb = ih2 * ((pb[f - 1] + pb[f + 1]) + (pb[f - Px] + pb[f + Px]) +
                               (pb[f - PP] + pb[f + PP]) - 6.0 * pb[f]);
          ww = pv[f] * idt - lapb;
        }
        if (p.mirror && !in_dom(gx0 + li, gy0 + lj, gz0 + lk)) ww = 0.0;   // not an unknown
        w[l] = ww;
#pragma unroll
        for (int i = 0; i <= KMAX; ++i)
          if (i <= j) acc[i] += V[(size_t)i * n + l] * ww;
      }
      block_sum_multi<KMAX + 1>(acc, red, hs, j + 1);
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
      if (scal[2] != 0.0) break;
      const double ihn = 1.0 / scal[3];
      double* Vn = V + (size_t)(j + 1) * n;
      for (int l = tid; l < n; l += NT) Vn[l] = w[l] * ihn;
    }
    if (tid == 0) {
      const int ld = k + 1;
      for (int i = jm - 1; i >= 0; --i) {
        double s = gv[i];
        for (int l = i + 1; l < jm; ++l) s -= H[i + ld * l] * yv[l];
        yv[i] = s / H[i + ld * i];
      }
      ras_count(p.jcnt, jm);
    }
    __syncthreads();
    if (p.y_ext) {   // (R_k^delta)^T: the whole ext-box solution, summed by ras_extend
      for (int l = tid; l < n; l += NT) {
        double s = 0.0;
        for (int i = 0; i < jm; ++i) s += yv[i] * V[(size_t)i * n + l];
        p.y_ext[(size_t)box * n + l] = s;
      }
      continue;
    }
    for (int l = tid; l < p.bx * p.by * p.bz; l += NT) {
      int li = l % p.bx, lj = (l / p.bx) % p.by, lk = l / (p.bx * p.by);
      int ll = ((lk + p.o) * Ey + lj + p.o) * Ex + li + p.o;
      double s = 0.0;
      for (int i = 0; i < jm; ++i) s += yv[i] * V[(size_t)i * n + ll];
      p.z[(size_t)(ibx * p.bx + li) + NX * (iby * p.by + lj) + NXY * (ibz * p.bz + lk)] = s;
    }
  }
}

size_t ras3d_scratch_per_cta(const pfc_config& c) {
  const size_t Ex = c.ras_box[0] + 2 * c.ras_overlap, Ey = c.ras_box[1] + 2 * c.ras_overlap,
               Ez = c.ras_box[2] + 2 * c.ras_overlap;
  const size_t n = Ex * Ey * Ez, np = (Ex + 6) * (Ey + 6) * (Ez + 6);
  size_t d = (size_t)(c.ras_local_k + 1) * n + 2 * n + (c.mobility ? 6 : 3) * np +
             (c.bc == PFC_BC_MIRROR ? np + (np + 1) / 2 : 0);   // mirror: pc, gp
  return (d + 31) & ~size_t(31);
}

}  // namespace

int ras3d_plan(pfc_ctx* ctx) {
  ctx->ras_smem = 0;
  ctx->ras_threads = NT;
  ctx->ras_cluster = 1;
  return 1;
}

size_t ras3d_scratch_doubles(pfc_ctx* ctx, int* grid) {
  const pfc_config& c = ctx->cfg;
  const int nboxes = (c.n[0] / c.ras_box[0]) * (c.n[1] / c.ras_box[1]) * (c.n[2] / c.ras_box[2]);
  int g = 148 * 2;
  if (g > nboxes) g = nboxes;
  *grid = g;
  return ras3d_scratch_per_cta(c) * g;
}

cudaError_t launch_ras_3d(pfc_ctx* ctx, const double* v, const double* c, double dt, double* z,
                          double* scratch) {
  const pfc_config& cf = ctx->cfg;
  int grid = 0;
  ras3d_scratch_doubles(ctx, &grid);
  Ras3Args p{v, c, z, scratch, ras3d_scratch_per_cta(cf), cf.n[0], cf.n[1], cf.n[2],
             cf.ras_box[0], cf.ras_box[1], cf.ras_box[2], cf.ras_overlap, cf.ras_local_k,
             1.0 / dt, cf.gamma, ctx->ih2, cf.ras_variant == PFC_RAS_RIGHT,
             cf.ras_variant == PFC_RAS_LEFT ? nullptr : ctx->ras_y, ctx->gate,
             ctx->mob_phi, ctx->mob_psi, ctx->mob_A, cf.mobility,
             ctx->prof ? ctx->d_jcnt : nullptr, cf.bc == PFC_BC_MIRROR};
  p.dtp = ctx->dtdev;
  ras3d_kernel<<<grid, NT, 0, ctx->stream>>>(p);
  ctx->launches++;
  {
    const double nb = (double)(cf.n[0] / cf.ras_box[0]) * (cf.n[1] / cf.ras_box[1]) *
                      (cf.n[2] / cf.ras_box[2]);
    const double ebox = (double)(cf.ras_box[0] + 2 * cf.ras_overlap) *
                        (cf.ras_box[1] + 2 * cf.ras_overlap) * (cf.ras_box[2] + 2 * cf.ras_overlap);
    const double next = nb * ebox;
    const double nout = cf.ras_variant == PFC_RAS_LEFT ? (double)ctx->N : next;
    pfc_account(ctx, PFC_K_RAS, 8.0 * (2.0 * next + nout), 0.0);
    ras_flop_model(ctx, ebox, 31.0, nout / nb);   // flops from the step counters
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || cf.ras_variant == PFC_RAS_LEFT) return e;
  return launch_ras_extend(ctx, z);
}
