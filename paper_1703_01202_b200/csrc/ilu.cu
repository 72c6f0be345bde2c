// ilu.cu -- ILU(k) subdomain solves of the Schwarz preconditioner (NEXT row f2), sm_100a.
//
// The paper's subdomain solvers (Table 1): incomplete LU with fill level
// k of A_k in the natural (x-fastest) order of the extended box, with the option of reusing
// the factors of the step's first Newton iteration (reading R10).  A_k is the
// zero-ring subdomain matrix (= R J R^T for M = 1, reading R8):
//   A_ij = W[class(x_j - x_i)] + (j == i ? 2d h^-2 c_i : |x_j - x_i|_1 == 1 ? -h^-2 c_j : 0)
// with W the class weights of v/dt - alpha Delta v - Delta^2 v - Delta^3 v / 2 (the 25 / 63
// point radius-3 stencil truncated at the box) and the second term from -Delta(c v).
//
// Everything structural is built once on the host at pfc_create, identical for every box: the
// pattern of A (the truncated stencil), the ILU(k) fill pattern by the standard level rule,
// the IKJ operation list of each row (divide a_ik by a_kk, then a_ij -= a_ik a_kj for the kept
// j > k), and the level schedules of the factorisation / forward solve (a row depends on its
// L entries) and of the backward solve (on its U entries).  The device then runs, one CTA per
// box, (1) the numeric factorisation into the box's value array, level by level, one warp per
// row: its values, pivots and every a_kj it needs fetched in one round trip, then the IKJ loop
// in shared memory (lane 0 divides, the lanes apply that k's distinct updates), and (2) per
// preconditioner apply, the forward and backward solves, one WARP per box, the rows of each
// level on the lanes (warp-synchronous; many boxes per SM hide the factor-read latency); the
// value array is laid out as [L block | U block].
// Same operations as the oracle (or_ilu_dense / ilu_solve) per entry; the parallel order only
// regroups independent updates and the triangular-solve dot products.
//
// Mirror walls (PFC_BC_MIRROR, reading R23; round 2): A_k = R J R^T with the mirror J, the
// ext box clipped at the walls.  The stencil point x_i + d of an in-domain row lands on the
// mirror image of that node, so near a wall several offsets d hit one column: the entry is the
// SUM of their class weights (and of the -h^-2 c_j of the unit offsets, which may hit the row's
// own node); ext-box nodes outside the domain are no unknowns and get identity rows, as in the
// oracle (local_ilu).  The pattern, its ILU(k) fill and the schedules then depend on where the
// box sits relative to the walls: one symbolic factorisation per CLASS of boxes (per axis: the
// clipped layers and the distance of the ext box to either wall, capped at the stencil radius;
// <= 3^d classes on the configs' grids), one launch per class over that class's box list.  The
// periodic grid is the single-class case with the original per-entry class table.
#include "pfc_device.cuh"
#include "pfc_internal.h"

#include <cstdlib>

#include <algorithm>
#include <map>
#include <vector>

namespace {

constexpr int NT = 512;

int wclass(int a, int b, int c) {   // class of the sorted |offset|: 000 001 002 011 003 012 111
  const int s = a + b + c;
  if (s == 0) return 0;
  if (s == 1) return 1;
  if (s == 2) return (a == 2 || b == 2 || c == 2) ? 2 : 3;
  if (a == 3 || b == 3 || c == 3) return 4;
  return (a == 1 && b == 1 && c == 1) ? 6 : 5;
}

struct IluArgs {
  const double* v;      // apply: input field
  const double* c;      // factor: Jacobian coefficient field
  double* z;            // apply: output (owned nodes) or nullptr with y_ext
  double* y_ext;        // AS / right-RAS: ext-box solutions [box][ext node]
  double* vals;         // [box][nnz] factor values
  const int* lptr;      // factor pattern, L block (strictly lower entries of every row) ...
  const int* lcol;
  const int* uptr;      // ... then the U block (diagonal first, then the upper entries)
  const int* ucol;
  int nL, nU;           // value position of U entry t of row i: nL + uptr[i] + t
  const int* ecls;      // per entry: linear-weight class, -1 for fill
  const int* ectype;    // per entry: 0 none, 1 -h^-2 c_j, 2 +2d h^-2 c_i, 3 identity row
  const double* elin;   // mirror classes: per entry, the summed dt-free class weights (else null)
  const int* eccnt;     // mirror classes: per entry, the number of unit offsets that hit the column
  const int* boxes;     // this launch's boxes (global box ids), or null = every box in order
  int mirror;           // PFC_BC_MIRROR: ext-box nodes outside the domain are identity rows
  double idt;           // 1/dt (mirror classes: added to the in-domain diagonal)
  const int* ukptr;     // updates of L entry q: [ukptr[q], ukptr[q+1]) of ...
  const int* usrc;      // ... the value position of a_kj (final row k)
  const int* udst;      // ... and the slot of a_ij within row i
  const int* flev_ptr;  // forward / factorisation levels
  const int* flev_row;
  const int* blev_ptr;  // backward levels
  const int* blev_row;
  int nflev, nblev, n, nnz, maxrow, maxupd;
  int nx, ny, nz, bx, by, bz, o, nd;
  double W[7];
  double ih2;
  int restrict_owned;
  const int* gate;
};

__device__ __forceinline__ void box_origin(const IluArgs& p, int box, int& gx0, int& gy0,
                                           int& gz0, int& ibx, int& iby, int& ibz) {
  const int nbx = p.nx / p.bx, nby = p.ny / p.by;
  ibx = box % nbx; iby = (box / nbx) % nby; ibz = box / (nbx * nby);
  gx0 = ibx * p.bx - p.o; gy0 = iby * p.by - p.o; gz0 = p.nd == 3 ? ibz * p.bz - p.o : 0;
}

__device__ __forceinline__ size_t gnode(const IluArgs& p, int l, int gx0, int gy0, int gz0) {
  const int Ex = p.bx + 2 * p.o, Ey = p.by + 2 * p.o;
  const int li = l % Ex, lj = (l / Ex) % Ey, lk = l / (Ex * Ey);
  return (size_t)wrapi(gx0 + li, p.nx) + (size_t)p.nx * wrapi(gy0 + lj, p.ny) +
         (size_t)p.nx * p.ny * (p.nd == 3 ? wrapi(gz0 + lk, p.nz) : 0);
}
// mirror walls: is ext-box node l an unknown (inside the domain)?
__device__ __forceinline__ bool in_dom(const IluArgs& p, int l, int gx0, int gy0, int gz0) {
  if (!p.mirror) return true;
  const int Ex = p.bx + 2 * p.o, Ey = p.by + 2 * p.o;
  const int x = gx0 + l % Ex, y = gy0 + (l / Ex) % Ey, z = p.nd == 3 ? gz0 + l / (Ex * Ey) : 0;
  return x >= 0 && x < p.nx && y >= 0 && y < p.ny && z >= 0 && z < p.nz;
}

// numeric ILU(k) of every box: A values from the class weights and c, then IKJ by levels
__global__ void __launch_bounds__(NT) k_ilu_factor(const IluArgs p) {
  const int box = p.boxes ? p.boxes[blockIdx.x] : blockIdx.x;
  int gx0, gy0, gz0, ibx, iby, ibz;
  box_origin(p, box, gx0, gy0, gz0, ibx, iby, ibz);
  double* a = p.vals + (size_t)blockIdx.x * p.nnz;
  const int d2 = 2 * p.nd;
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) {
    const double ci = in_dom(p, i, gx0, gy0, gz0) ? p.c[gnode(p, i, gx0, gy0, gz0)] : 0.0;
    auto set = [&](int q, int col) {
      const int ct = p.ectype[q];
      double val;
      if (p.elin) {   // mirror class: summed weights; columns of in-domain rows are in-domain
        val = p.elin[q];
        if (ct == 2) val += p.idt + d2 * p.ih2 * ci;
        const int cc = p.eccnt[q];
        if (cc) val -= cc * (p.ih2 * p.c[gnode(p, col, gx0, gy0, gz0)]);
      } else {
        const int cl = p.ecls[q];
        val = cl >= 0 ? p.W[cl] : 0.0;
        if (ct == 2) val += d2 * p.ih2 * ci;
        else if (ct == 1) val -= p.ih2 * p.c[gnode(p, col, gx0, gy0, gz0)];
      }
      a[q] = val;
    };
    for (int q = p.lptr[i]; q < p.lptr[i + 1]; ++q) set(q, p.lcol[q]);
    for (int t = p.uptr[i]; t < p.uptr[i + 1]; ++t) set(p.nL + t, p.ucol[t]);
  }
  __syncthreads();
  // IKJ by levels, one warp per row.  Everything the row needs is read in one round trip:
  // its own values, the pivots a_kk and every a_kj of its updates (rows k are final: earlier
  // levels); then the k loop runs in shared memory (lane 0 divides a_ik, the lanes apply the
  // distinct updates a_ij -= a_ik a_kj) and the row is written back.
  extern __shared__ double fsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* rb = fsm + (size_t)wid * (2 * p.maxrow + p.maxupd);
  double* piv = rb + p.maxrow;
  double* us = piv + p.maxrow;
  // the row's index data too (the k loop must not wait on global loads)
  const int nw = blockDim.x >> 5;     // warps of this launch (fewer when the rows are long)
  int* ibase = reinterpret_cast<int*>(fsm + (size_t)nw * (2 * p.maxrow + p.maxupd));
  int* uk = ibase + (size_t)wid * (p.maxrow + 1 + p.maxupd);
  int* ud = uk + p.maxrow + 1;
  for (int L = 0; L < p.nflev; ++L) {
    for (int r = p.flev_ptr[L] + wid; r < p.flev_ptr[L + 1]; r += nw) {
      const int i = p.flev_row[r];
      const int l0 = p.lptr[i], nLi = p.lptr[i + 1] - l0;
      const int u0 = p.nL + p.uptr[i], nUi = p.uptr[i + 1] - p.uptr[i];
      const int g0 = p.ukptr[l0], ng = p.ukptr[l0 + nLi] - g0;
      for (int t = lane; t < nLi + nUi; t += 32) rb[t] = t < nLi ? a[l0 + t] : a[u0 + t - nLi];
      for (int t = lane; t < nLi; t += 32) piv[t] = a[p.nL + p.uptr[p.lcol[l0 + t]]];
      for (int u = lane; u < ng; u += 32) {
        us[u] = a[p.usrc[g0 + u]];
        ud[u] = p.udst[g0 + u];
      }
      for (int t = lane; t <= nLi; t += 32) uk[t] = p.ukptr[l0 + t] - g0;
      __syncwarp();
      for (int t = 0; t < nLi; ++t) {
        if (lane == 0) rb[t] = rb[t] / piv[t];
        __syncwarp();
        const double lik = rb[t];
        const int e1 = uk[t + 1];
        for (int u = uk[t] + lane; u < e1; u += 32) rb[ud[u]] -= lik * us[u];
        __syncwarp();
      }
      for (int t = lane; t < nLi + nUi; t += 32) {
        if (t < nLi) a[l0 + t] = rb[t];
        else a[u0 + t - nLi] = rb[t];
      }
      __syncwarp();
    }
    __syncthreads();
  }
}

// z = sum_k (R_k^0)^T U^{-1} L^{-1} R_k^delta v (left-RAS) or the ext-box solutions.
// One WARP per box, warp-synchronous (no block barriers): the sweeps are chains of levels with
// a few rows each, so the rows of a level go to the lanes and many boxes per SM hide the
// latency of the (L2 / HBM) factor reads.  y of each warp's box lives in shared memory.
constexpr int AWMAX = 4;   // boxes (warps) per CTA at most (shared memory: one y per warp)
__global__ void __launch_bounds__(AWMAX * 32) k_ilu_apply(const IluArgs p, int nbox) {
  extern __shared__ double ysh[];
  if (p.gate && *p.gate) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int bl = blockIdx.x * (blockDim.x >> 5) + wid;   // position in this launch's box list
  if (bl >= nbox) return;                      // whole warps only
  const int box = p.boxes ? p.boxes[bl] : bl;
  double* y = ysh + (size_t)wid * p.n;
  int gx0, gy0, gz0, ibx, iby, ibz;
  box_origin(p, box, gx0, gy0, gz0, ibx, iby, ibz);
  const double* a = p.vals + (size_t)bl * p.nnz;
  const int Ex = p.bx + 2 * p.o, Ey = p.by + 2 * p.o;
  for (int l = lane; l < p.n; l += 32) {
    const int li = l % Ex, lj = (l / Ex) % Ey, lk = l / (Ex * Ey);
    const bool owned = li >= p.o && li < p.o + p.bx && lj >= p.o && lj < p.o + p.by &&
                       (p.nd == 2 || (lk >= p.o && lk < p.o + p.bz));
    y[l] = ((p.restrict_owned && !owned) || !in_dom(p, l, gx0, gy0, gz0))
               ? 0.0 : p.v[gnode(p, l, gx0, gy0, gz0)];
  }
  __syncwarp();
  // Both sweeps: rows of a level on the lanes.  The factor values and column indices of a row
  // do not depend on the sweep, so the first NPRE entries of the lane's first row of level
  // L+2 are loaded while level L computes: the factors of all boxes (e.g. 265 MB at cfg2) live
  // in HBM, and each level would otherwise wait on a DRAM round trip.  Longer rows and further
  // rows of a level load as before.  Same subtractions in the same order.
  constexpr int NPRE = 16;
  struct Pre { int i, q0, q1; double av[NPRE]; int cv[NPRE]; };
  auto fetch = [&](const int* lev_ptr, const int* lev_row, int nlev, const int* ptr,
                   const int* col, const double* val, int L, bool upper, Pre& P) {
    P.i = -1;
    if (L >= nlev) return;
    const int r = __ldg(lev_ptr + L) + lane;
    if (r >= __ldg(lev_ptr + L + 1)) return;
    P.i = __ldg(lev_row + r);
    P.q0 = __ldg(ptr + P.i) + (upper ? 1 : 0);   // U: the diagonal is read separately
    P.q1 = __ldg(ptr + P.i + 1);
#pragma unroll
    for (int t = 0; t < NPRE; ++t) {
      P.av[t] = P.q0 + t < P.q1 ? val[P.q0 + t] : 0.0;
      P.cv[t] = P.q0 + t < P.q1 ? __ldg(col + P.q0 + t) : P.i;
    }
  };
  auto row_sum = [&](const int* col, const double* val, int i, int q0, int q1, double s) {
    for (int q = q0; q < q1; q += 8) {         // 8 independent loads in flight, then the
      double av[8];                            // subtractions in ascending order
      int cv[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        av[t] = q + t < q1 ? val[q + t] : 0.0;
        cv[t] = q + t < q1 ? __ldg(col + q + t) : i;
      }
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (q + t < q1) s -= av[t] * y[cv[t]];
    }
    return s;
  };
  // A level holding ONE long row (every level of the complete-fill LU, whose rows chain
  // i-1 -> i): the whole warp takes the row, lanes split its entries (coalesced loads), and a
  // fixed-order warp sum closes it (a different summation order than the serial one: rounding
  // only).  s = y[i] - sum_q val[q] y[col[q]].
  auto row_warp = [&](const int* col, const double* val, int q0, int q1, double yi) {
    double part = 0.0;
    for (int q = q0 + lane; q < q1; q += 32) part = fma(val[q], y[__ldg(col + q)], part);
    return yi - warp_sum(part);
  };
  constexpr int LONG = 24;   // entries from which a single-row level goes to the whole warp
  {   // L y = r (unit lower)
    Pre cur, nx1, nx2;
    fetch(p.flev_ptr, p.flev_row, p.nflev, p.lptr, p.lcol, a, 0, false, cur);
    fetch(p.flev_ptr, p.flev_row, p.nflev, p.lptr, p.lcol, a, 1, false, nx1);
    for (int L = 0; L < p.nflev; ++L) {
      const int rs = __ldg(p.flev_ptr + L);
      if (__ldg(p.flev_ptr + L + 1) - rs == 1) {
        const int i = __ldg(p.flev_row + rs), q0 = __ldg(p.lptr + i), q1 = __ldg(p.lptr + i + 1);
        if (q1 - q0 >= LONG) {
          const double s = row_warp(p.lcol, a, q0, q1, y[i]);
          __syncwarp();
          if (lane == 0) y[i] = s;
          __syncwarp();
          fetch(p.flev_ptr, p.flev_row, p.nflev, p.lptr, p.lcol, a, L + 2, false, nx2);
          cur = nx1;
          nx1 = nx2;
          continue;
        }
      }
      fetch(p.flev_ptr, p.flev_row, p.nflev, p.lptr, p.lcol, a, L + 2, false, nx2);
      if (cur.i >= 0) {
        double s = y[cur.i];
#pragma unroll
        for (int t = 0; t < NPRE; ++t)
          if (cur.q0 + t < cur.q1) s -= cur.av[t] * y[cur.cv[t]];
        y[cur.i] = row_sum(p.lcol, a, cur.i, cur.q0 + NPRE, cur.q1, s);
      }
      for (int r = p.flev_ptr[L] + lane + 32; r < p.flev_ptr[L + 1]; r += 32) {
        const int i = p.flev_row[r];
        y[i] = row_sum(p.lcol, a, i, __ldg(p.lptr + i), __ldg(p.lptr + i + 1), y[i]);
      }
      __syncwarp();
      cur = nx1;
      nx1 = nx2;
    }
  }
  const double* u = a + p.nL;
  {   // U x = y
    Pre cur, nx1, nx2;
    fetch(p.blev_ptr, p.blev_row, p.nblev, p.uptr, p.ucol, u, 0, true, cur);
    fetch(p.blev_ptr, p.blev_row, p.nblev, p.uptr, p.ucol, u, 1, true, nx1);
    for (int L = 0; L < p.nblev; ++L) {
      const int rs = __ldg(p.blev_ptr + L);
      if (__ldg(p.blev_ptr + L + 1) - rs == 1) {
        const int i = __ldg(p.blev_row + rs), t0 = __ldg(p.uptr + i), t1 = __ldg(p.uptr + i + 1);
        if (t1 - t0 - 1 >= LONG) {
          const double s = row_warp(p.ucol, u, t0 + 1, t1, y[i]) / u[t0];
          __syncwarp();
          if (lane == 0) y[i] = s;
          __syncwarp();
          fetch(p.blev_ptr, p.blev_row, p.nblev, p.uptr, p.ucol, u, L + 2, true, nx2);
          cur = nx1;
          nx1 = nx2;
          continue;
        }
      }
      fetch(p.blev_ptr, p.blev_row, p.nblev, p.uptr, p.ucol, u, L + 2, true, nx2);
      if (cur.i >= 0) {
        const double dii = u[cur.q0 - 1];
        double s = y[cur.i];
#pragma unroll
        for (int t = 0; t < NPRE; ++t)
          if (cur.q0 + t < cur.q1) s -= cur.av[t] * y[cur.cv[t]];
        y[cur.i] = row_sum(p.ucol, u, cur.i, cur.q0 + NPRE, cur.q1, s) / dii;
      }
      for (int r = p.blev_ptr[L] + lane + 32; r < p.blev_ptr[L + 1]; r += 32) {
        const int i = p.blev_row[r];
        const int t0 = __ldg(p.uptr + i);
        y[i] = row_sum(p.ucol, u, i, t0 + 1, __ldg(p.uptr + i + 1), y[i]) / u[t0];
      }
      __syncwarp();
      cur = nx1;
      nx1 = nx2;
    }
  }
  if (p.y_ext) {
    for (int l = lane; l < p.n; l += 32) p.y_ext[(size_t)box * p.n + l] = y[l];
    return;
  }
  const int nown = p.bx * p.by * (p.nd == 3 ? p.bz : 1);
  for (int l = lane; l < nown; l += 32) {
    const int li = l % p.bx, lj = (l / p.bx) % p.by, lk = l / (p.bx * p.by);
    const int e = (li + p.o) + Ex * ((lj + p.o) + Ey * (p.nd == 3 ? lk + p.o : 0));
    p.z[(size_t)(ibx * p.bx + li) + (size_t)p.nx * (iby * p.by + lj) +
        (size_t)p.nx * p.ny * (p.nd == 3 ? ibz * p.bz + lk : 0)] = y[e];
  }
}

}  // namespace

// ---------------------------------------------------------------- host: symbolic setup

// one class of boxes: pattern, IKJ lists, schedules and the factor values of its boxes
struct IluClass {
  int nnz = 0, nflev = 0, nblev = 0;
  int nL = 0, nU = 0, maxrow = 0, maxupd = 0;
  int maxlev = 1;                 // rows of the widest factorisation level
  int* d_ukptr = nullptr; int* d_usrc = nullptr; int* d_udst = nullptr;
  int* d_lptr = nullptr; int* d_lcol = nullptr; int* d_uptr = nullptr; int* d_ucol = nullptr;
  int* d_ecls = nullptr; int* d_ectype = nullptr; int* d_eccnt = nullptr;
  double* d_elin = nullptr;
  int* d_flev_ptr = nullptr; int* d_flev_row = nullptr;
  int* d_blev_ptr = nullptr; int* d_blev_row = nullptr;
  int* d_boxes = nullptr;         // global ids of the class's boxes (null: every box in order)
  double* d_vals = nullptr;
  size_t nbox = 0;
};

struct pfc_ilu {
  int n = 0;
  size_t nbox = 0;        // all boxes
  size_t nnz_total = 0;   // factor entries over all boxes
  std::vector<IluClass> cls;
};

static bool up(pfc_ctx* ctx, int** d, const std::vector<int>& h) {
  if (cudaMalloc(d, std::max<size_t>(h.size(), 1) * sizeof(int)) != cudaSuccess) return false;
  return cudaMemcpy(*d, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess;
}

constexpr size_t kSmemPlan = 200 * 1024;

// dt-free class weights of the linear part (as in ras2d.cu / ras3d_col.cu);
// class 0 gets 1/dt at factor time
static void class_weights(const pfc_ctx* ctx, double* W) {
  const pfc_config& cf = ctx->cfg;
  const double ih2 = ctx->ih2, ih4 = ih2 * ih2, ih6 = ih4 * ih2, al = 0.5 * (1.0 - cf.gamma);
  if (cf.ndim == 2) {
    W[0] = 4.0 * al * ih2 - 20.0 * ih4 + 56.0 * ih6;
    W[1] = -al * ih2 + 8.0 * ih4 - 28.5 * ih6;
    W[2] = -ih4 + 6.0 * ih6;
    W[3] = -2.0 * ih4 + 12.0 * ih6;
    W[4] = -0.5 * ih6;
    W[5] = -1.5 * ih6;
    W[6] = 0.0;
  } else {
    W[0] = 6.0 * al * ih2 - 42.0 * ih4 + 162.0 * ih6;
    W[1] = -al * ih2 + 12.0 * ih4 - 61.5 * ih6;
    W[2] = -ih4 + 9.0 * ih6;
    W[3] = -2.0 * ih4 + 18.0 * ih6;
    W[4] = -0.5 * ih6;
    W[5] = -1.5 * ih6;
    W[6] = -3.0 * ih6;
  }
}

// Symbolic factorisation of one class.  g0 = global coordinates of ext-box node (0,0,0) of a
// box of the class (mirror walls only; the class fixes g0 up to shifts that change nothing).
static pfc_status build_class(pfc_ctx* ctx, const int* E, const int* g0, bool mirror,
                              IluClass* I) {
  const pfc_config& c = ctx->cfg;
  const int nd = c.ndim;
  const int n = E[0] * E[1] * E[2];
  auto pos = [&](int i, int j, int k) { return i + E[0] * (j + E[1] * k); };
  // ext-box coordinate of stencil point l + d on one axis, or -1: outside the ext box (the
  // zero ring of R8); mirror walls: the even extension's image of a point beyond a wall (R23)
  auto target = [&](int ax, int l, int d) {
    int t = l + d;
    if (mirror) {
      int g = g0[ax] + t;
      if (g < 0) g = -1 - g;
      else if (g >= c.n[ax]) g = 2 * c.n[ax] - 1 - g;
      t = g - g0[ax];
    }
    return (t < 0 || t >= E[ax]) ? -1 : t;
  };
  auto inside = [&](int i, int j, int k) {
    if (!mirror) return true;
    const int l[3] = {i, j, k};
    for (int d = 0; d < nd; ++d)
      if (g0[d] + l[d] < 0 || g0[d] + l[d] >= c.n[d]) return false;
    return true;
  };
  // pattern of A: the radius-3 L1 stencil truncated at the box, per row a map col -> level
  struct Meta { int cnt[7] = {0, 0, 0, 0, 0, 0, 0}; int ccnt = 0; int ct = 0; };
  std::vector<std::map<int, int>> rows(n);
  std::vector<std::map<int, Meta>> meta(n);
  const int R = 3;
  for (int k = 0; k < E[2]; ++k)
    for (int j = 0; j < E[1]; ++j)
      for (int i = 0; i < E[0]; ++i) {
        const int r = pos(i, j, k);
        if (!inside(i, j, k)) {      // no unknown: identity row
          rows[r][r] = 0;
          meta[r][r].ct = 3;
          continue;
        }
        for (int dz = (nd == 3 ? -R : 0); dz <= (nd == 3 ? R : 0); ++dz)
          for (int dy = -R; dy <= R; ++dy)
            for (int dx = -R; dx <= R; ++dx) {
              const int ax = std::abs(dx), ay = std::abs(dy), az = std::abs(dz);
              if (ax + ay + az > R) continue;
              const int ii = target(0, i, dx), jj = target(1, j, dy);
              const int kk = nd == 3 ? target(2, k, dz) : 0;
              if (ii < 0 || jj < 0 || kk < 0) continue;
              int s[3] = {ax, ay, az};
              std::sort(s, s + 3);
              const int col = pos(ii, jj, kk);
              rows[r][col] = 0;
              Meta& m = meta[r][col];
              m.cnt[wclass(s[0], s[1], s[2])]++;
              if (ax + ay + az == 1) m.ccnt++;
              if (col == r) m.ct = 2;
              else if (m.ct == 0 && ax + ay + az == 1) m.ct = 1;
            }
      }
  // ILU(k) fill levels, row by row (rows k < i are final when row i is processed); the paper's
  // LU (Table 1) keeps every fill entry: the exact factorisation in natural order
  const int level = c.ras_local_solver == PFC_LOCAL_LU ? n : c.ras_ilu_level;
  for (int i = 0; i < n; ++i) {
    auto& ri = rows[i];
    for (auto it = ri.begin(); it != ri.end() && it->first < i; ++it) {
      const int kk = it->first, lik = it->second;
      for (auto jt = rows[kk].upper_bound(kk); jt != rows[kk].end(); ++jt) {
        const int l = lik + jt->second + 1;
        if (l > level) continue;
        auto f = ri.find(jt->first);
        if (f == ri.end()) ri[jt->first] = l;          // new fill (j > k: visited later if < i)
        else if (l < f->second) f->second = l;
      }
    }
  }
  // value positions: the L block (strictly lower entries of every row, in row order), then the
  // U block (diagonal first, then the upper entries, in row order)
  std::vector<int> lptr(n + 1, 0), uptr(n + 1, 0), lcol, ucol, ecls, ectype, eccnt;
  std::vector<double> elin;
  std::vector<std::map<int, int>> where(n);
  for (int i = 0; i < n; ++i) {
    for (auto& e : rows[i])
      if (e.first < i) lcol.push_back(e.first);
    lptr[i + 1] = (int)lcol.size();
    ucol.push_back(i);
    for (auto& e : rows[i])
      if (e.first > i) ucol.push_back(e.first);
    uptr[i + 1] = (int)ucol.size();
  }
  const int nL = (int)lcol.size(), nU = (int)ucol.size(), nnz = nL + nU;
  ecls.assign(nnz, -1);
  ectype.assign(nnz, 0);
  if (mirror) {
    eccnt.assign(nnz, 0);
    elin.assign(nnz, 0.0);
  }
  double Wn[7];
  class_weights(ctx, Wn);
  for (int i = 0; i < n; ++i) {
    for (int q = lptr[i]; q < lptr[i + 1]; ++q) where[i][lcol[q]] = q;
    for (int t = uptr[i]; t < uptr[i + 1]; ++t) where[i][ucol[t]] = nL + t;
    for (auto& w : where[i]) {
      auto m = meta[i].find(w.first);
      if (m == meta[i].end()) continue;
      const Meta& mm = m->second;
      ectype[w.second] = mm.ct;
      if (!mirror) {   // exactly one offset per column: its class, as before
        for (int cl = 0; cl < 7; ++cl)
          if (mm.cnt[cl]) ecls[w.second] = cl;
      } else if (mm.ct == 3) {
        elin[w.second] = 1.0;
      } else {
        double v = 0.0;
        for (int cl = 0; cl < 7; ++cl) v += mm.cnt[cl] * Wn[cl];
        elin[w.second] = v;
        eccnt[w.second] = mm.ccnt;
      }
    }
  }
  // IKJ updates per row: for the L entry q of row i (column k, ascending), the updates
  // a_ij -= a_ik a_kj over the kept j > k are [ukptr[q], ukptr[q+1]) of the flat lists usrc
  // (value position of a_kj in the final row k) and udst (slot of a_ij in row i: L entries
  // 0..nLi-1, then the U entries)
  std::vector<int> ukptr(nL + 1, 0), usrc, udst;
  std::vector<int> flev(n, 0), blev(n, 0);
  int maxupd = 0;
  for (int i = 0; i < n; ++i) {
    const int nLi = lptr[i + 1] - lptr[i];
    int rowupd = 0;
    for (int q = lptr[i]; q < lptr[i + 1]; ++q) {
      const int kk = lcol[q];
      flev[i] = std::max(flev[i], flev[kk] + 1);
      for (auto jt = rows[kk].upper_bound(kk); jt != rows[kk].end(); ++jt) {
        auto w = where[i].find(jt->first);
        if (w == where[i].end()) continue;
        usrc.push_back(where[kk][jt->first]);
        const int pos = w->second;
        udst.push_back(pos < nL ? pos - lptr[i] : nLi + (pos - nL - uptr[i]));
      }
      ukptr[q + 1] = (int)usrc.size();
      rowupd += ukptr[q + 1] - ukptr[q];
    }
    maxupd = std::max(maxupd, rowupd);
  }
  for (int i = n - 1; i >= 0; --i)
    for (auto jt = rows[i].upper_bound(i); jt != rows[i].end(); ++jt)
      blev[i] = std::max(blev[i], blev[jt->first] + 1);
  auto group = [&](const std::vector<int>& lev, std::vector<int>& ptr, std::vector<int>& rr) {
    const int nl = *std::max_element(lev.begin(), lev.end()) + 1;
    ptr.assign(nl + 1, 0);
    for (int i = 0; i < n; ++i) ptr[lev[i] + 1]++;
    for (int l = 0; l < nl; ++l) ptr[l + 1] += ptr[l];
    rr.assign(n, 0);
    std::vector<int> fill(ptr.begin(), ptr.end() - 1);
    for (int i = 0; i < n; ++i) rr[fill[lev[i]]++] = i;
    return nl;
  };
  std::vector<int> fptr, frow, bptr, brow;
  I->nnz = nnz; I->nL = nL; I->nU = nU; I->maxupd = maxupd;
  for (int i = 0; i < n; ++i)
    I->maxrow = std::max(I->maxrow, (lptr[i + 1] - lptr[i]) + (uptr[i + 1] - uptr[i]));
  I->nflev = group(flev, fptr, frow);
  for (int l = 0; l < I->nflev; ++l) I->maxlev = std::max(I->maxlev, fptr[l + 1] - fptr[l]);
  I->nblev = group(blev, bptr, brow);
  if (!up(ctx, &I->d_lptr, lptr) || !up(ctx, &I->d_lcol, lcol) || !up(ctx, &I->d_uptr, uptr) ||
      !up(ctx, &I->d_ucol, ucol) ||
      !up(ctx, &I->d_ecls, ecls) || !up(ctx, &I->d_ectype, ectype) ||
      !up(ctx, &I->d_ukptr, ukptr) || !up(ctx, &I->d_usrc, usrc) || !up(ctx, &I->d_udst, udst) ||
      !up(ctx, &I->d_flev_ptr, fptr) || !up(ctx, &I->d_flev_row, frow) ||
      !up(ctx, &I->d_blev_ptr, bptr) || !up(ctx, &I->d_blev_row, brow))
    return pfc_fail(ctx, PFC_ENOMEM, "ILU structures");
  if (mirror) {
    if (!up(ctx, &I->d_eccnt, eccnt) ||
        cudaMalloc(&I->d_elin, std::max<size_t>(nnz, 1) * sizeof(double)) != cudaSuccess ||
        cudaMemcpy(I->d_elin, elin.data(), (size_t)nnz * sizeof(double),
                   cudaMemcpyHostToDevice) != cudaSuccess)
      return pfc_fail(ctx, PFC_ENOMEM, "ILU structures");
  }
  if ((size_t)(2 * I->maxrow + I->maxupd) * 8 + (I->maxrow + 1 + I->maxupd) * 4 > kSmemPlan)
    return pfc_fail(ctx, PFC_EINVAL, "ILU: rows too large for the shared-memory plan");
  return PFC_OK;
}

pfc_status ilu_setup(pfc_ctx* ctx) {
  const pfc_config& c = ctx->cfg;
  const int nd = c.ndim;
  const bool mirror = c.bc == PFC_BC_MIRROR;
  int E[3] = {1, 1, 1};
  for (int d = 0; d < nd; ++d) E[d] = c.ras_box[d] + 2 * c.ras_overlap;
  const int n = E[0] * E[1] * E[2];
  // cheap early rejection (before the symbolic factorisation, whose lists grow like band^2):
  // the ext box must fit the factor kernel's shared-memory plan, and so must the complete fill
  // of the natural-order LU, whose rows span the band b = 3 E0 (2D) / 3 E0 E1 (3D) on both
  // sides of the diagonal (row length <= 2b+1) with up to b^2 IKJ updates per row
  if ((size_t)n * sizeof(double) > kSmemPlan)
    return pfc_fail(ctx, PFC_EINVAL, "ILU: ext box too large for the shared-memory plan");
  if (c.ras_local_solver == PFC_LOCAL_LU) {
    const size_t b = (size_t)3 * E[0] * (nd == 3 ? E[1] : 1);
    const size_t mr = 2 * b + 1, mu = b * b;
    if ((2 * mr + mu) * 8 + (mr + 1 + mu) * 4 > kSmemPlan)
      return pfc_fail(ctx, PFC_EINVAL,
                      "LU: complete fill of this ext box exceeds the shared-memory plan "
                      "(every 3D box of the configs; use PFC_LOCAL_ILU or PFC_LOCAL_GMRES)");
  }
  pfc_ilu* I = new pfc_ilu();
  ctx->ilu = I;
  I->n = n;
  int nb[3] = {1, 1, 1};
  for (int d = 0; d < nd; ++d) nb[d] = c.n[d] / c.ras_box[d];
  I->nbox = (size_t)nb[0] * nb[1] * nb[2];
  // classes of boxes.  Periodic: one.  Mirror walls: per axis the position of the ext box
  // relative to either wall, capped at the stencil radius (beyond it no stencil point of the
  // box reaches the wall); negative = clipped layers
  std::map<std::vector<int>, int> index;
  std::vector<std::vector<int>> members;      // global box ids per class
  std::vector<std::vector<int>> origin;       // g0 of the class's first box
  for (int bz = 0; bz < nb[2]; ++bz)
    for (int by = 0; by < nb[1]; ++by)
      for (int bx = 0; bx < nb[0]; ++bx) {
        const int ib[3] = {bx, by, bz};
        std::vector<int> key, g0(3, 0);
        for (int d = 0; d < nd; ++d) {
          g0[d] = ib[d] * c.ras_box[d] - c.ras_overlap;
          if (mirror) {
            key.push_back(std::min(g0[d], 3));
            key.push_back(std::min(c.n[d] - g0[d] - E[d], 3));
          }
        }
        auto it = index.find(key);
        if (it == index.end()) {
          it = index.emplace(key, (int)members.size()).first;
          members.emplace_back();
          origin.push_back(g0);
        }
        members[it->second].push_back(bx + nb[0] * (by + nb[1] * bz));
      }
  I->cls.resize(members.size());
  for (size_t k = 0; k < members.size(); ++k) {
    IluClass* C = &I->cls[k];
    C->nbox = members[k].size();
    pfc_status st = build_class(ctx, E, origin[k].data(), mirror, C);
    if (st) return st;
    if (mirror && !up(ctx, &C->d_boxes, members[k]))
      return pfc_fail(ctx, PFC_ENOMEM, "ILU box lists");
    I->nnz_total += C->nbox * (size_t)C->nnz;
  }
  for (auto& C : I->cls)   // after every check
    if (cudaMalloc(&C.d_vals, C.nbox * (size_t)C.nnz * sizeof(double)) != cudaSuccess)
      return pfc_fail(ctx, PFC_ENOMEM, "ILU factor values");
  return PFC_OK;
}

void ilu_free(pfc_ctx* ctx) {
  pfc_ilu* I = ctx->ilu;
  if (!I) return;
  for (auto& C : I->cls) {
    int* a[] = {C.d_lptr, C.d_lcol, C.d_uptr, C.d_ucol, C.d_ecls, C.d_ectype, C.d_eccnt,
                C.d_ukptr, C.d_usrc, C.d_udst, C.d_flev_ptr, C.d_flev_row, C.d_blev_ptr,
                C.d_blev_row, C.d_boxes};
    for (int* p : a)
      if (p) cudaFree(p);
    if (C.d_elin) cudaFree(C.d_elin);
    if (C.d_vals) cudaFree(C.d_vals);
  }
  delete I;
  ctx->ilu = nullptr;
}

static IluArgs ilu_args(pfc_ctx* ctx, const IluClass& C, double dt) {
  const pfc_config& cf = ctx->cfg;
  IluArgs p{};
  p.vals = C.d_vals; p.lptr = C.d_lptr; p.lcol = C.d_lcol; p.uptr = C.d_uptr;
  p.ucol = C.d_ucol; p.nL = C.nL; p.nU = C.nU;
  p.ecls = C.d_ecls; p.ectype = C.d_ectype; p.ukptr = C.d_ukptr; p.usrc = C.d_usrc;
  p.elin = C.d_elin; p.eccnt = C.d_eccnt; p.boxes = C.d_boxes;
  p.mirror = cf.bc == PFC_BC_MIRROR;
  p.idt = 1.0 / dt;
  p.udst = C.d_udst; p.maxrow = C.maxrow; p.maxupd = C.maxupd;
  p.flev_ptr = C.d_flev_ptr; p.flev_row = C.d_flev_row;
  p.blev_ptr = C.d_blev_ptr; p.blev_row = C.d_blev_row;
  p.nflev = C.nflev; p.nblev = C.nblev; p.n = ctx->ilu->n; p.nnz = C.nnz;
  p.nx = cf.n[0]; p.ny = cf.n[1]; p.nz = cf.ndim == 3 ? cf.n[2] : 1;
  p.bx = cf.ras_box[0]; p.by = cf.ras_box[1]; p.bz = cf.ndim == 3 ? cf.ras_box[2] : 1;
  p.o = cf.ras_overlap; p.nd = cf.ndim;
  const double ih2 = ctx->ih2, ih4 = ih2 * ih2, ih6 = ih4 * ih2, al = 0.5 * (1.0 - cf.gamma);
  if (cf.ndim == 2) {   // class weights of the linear part (as in ras2d.cu)
    p.W[0] = 1.0 / dt + 4.0 * al * ih2 - 20.0 * ih4 + 56.0 * ih6;
    p.W[1] = -al * ih2 + 8.0 * ih4 - 28.5 * ih6;
    p.W[2] = -ih4 + 6.0 * ih6;
    p.W[3] = -2.0 * ih4 + 12.0 * ih6;
    p.W[4] = -0.5 * ih6;
    p.W[5] = -1.5 * ih6;
    p.W[6] = 0.0;
  } else {              // as in ras3d_col.cu
    p.W[0] = 1.0 / dt + 6.0 * al * ih2 - 42.0 * ih4 + 162.0 * ih6;
    p.W[1] = -al * ih2 + 12.0 * ih4 - 61.5 * ih6;
    p.W[2] = -ih4 + 9.0 * ih6;
    p.W[3] = -2.0 * ih4 + 18.0 * ih6;
    p.W[4] = -0.5 * ih6;
    p.W[5] = -1.5 * ih6;
    p.W[6] = -3.0 * ih6;
  }
  p.ih2 = ih2;
  p.restrict_owned = cf.ras_variant == PFC_RAS_RIGHT;
  return p;
}

cudaError_t launch_ilu_factor(pfc_ctx* ctx, const double* c, double dt) {
  static size_t attr = 0;
  for (const IluClass& C : ctx->ilu->cls) {
    IluArgs p = ilu_args(ctx, C, dt);
    p.c = c;
    const size_t per_warp = (2 * p.maxrow + p.maxupd) * sizeof(double) +
                            (p.maxrow + 1 + p.maxupd) * sizeof(int);
    // one warp per row of the widest level (12 for 36^2 boxes): more warps only wait at the
    // level barriers and cost resident CTAs (measured: 16 warps 3.10 ms, 12 warps 2.35 ms at
    // cfg2)
    int nw = (int)std::max<size_t>(1, std::min<size_t>(NT / 32, kSmemPlan / per_warp));
    nw = std::max(1, std::min(nw, C.maxlev));
    const size_t sm = (size_t)nw * per_warp;
    if (sm > 48 * 1024 && sm > attr) {
      cudaError_t e = cudaFuncSetAttribute(
          k_ilu_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      attr = sm;
    }
    k_ilu_factor<<<(int)C.nbox, nw * 32, sm, ctx->stream>>>(p);
    ctx->launches++;
  }
  ctx->ilu_dt = dt;
  pfc_account(ctx, PFC_K_RAS, 8.0 * ctx->N + 8.0 * ctx->ilu->nnz_total,
              2.0 * ctx->ilu->nnz_total);
  return cudaGetLastError();
}

cudaError_t launch_ras_ilu(pfc_ctx* ctx, const double* v, double* z) {
  const pfc_config& cf = ctx->cfg;
  static size_t attr = 0;
  for (const IluClass& C : ctx->ilu->cls) {
    IluArgs p = ilu_args(ctx, C, ctx->ilu_dt);
    p.v = v;
    p.z = z;
    p.y_ext = cf.ras_variant == PFC_RAS_LEFT ? nullptr : ctx->ras_y;
    p.gate = ctx->gate;
    const int aw = std::max(1, std::min<int>(AWMAX, (int)(kSmemPlan / ((size_t)p.n * 8))));
    const size_t sm = (size_t)aw * p.n * sizeof(double);
    if (sm > 48 * 1024 && sm > attr) {
      cudaError_t e = cudaFuncSetAttribute(
          k_ilu_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      attr = sm;
    }
    const int nbox = (int)C.nbox;
    k_ilu_apply<<<(nbox + aw - 1) / aw, aw * 32, sm, ctx->stream>>>(p, nbox);
    ctx->launches++;
  }
  {
    const double next = (double)ctx->ilu->nbox * ctx->ilu->n;
    pfc_account(ctx, PFC_K_RAS, 8.0 * (next + ctx->N) + 8.0 * ctx->ilu->nnz_total,
                4.0 * ctx->ilu->nnz_total);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || cf.ras_variant == PFC_RAS_LEFT) return e;
  return launch_ras_extend(ctx, z);
}
