// ras2d.cu -- left restricted additive Schwarz apply (K4), 2D, sm_100a.
//
//   z = sum_k (R_k^0)^T inv(A_k) R_k^delta v          Eq. (eq:ras) P:398-409
//
// One CTA per subdomain box Omega_k (b_x x b_y owned nodes).  The CTA gathers v and the
// Jacobian coefficient c on the extended box Omega_k^delta (E = b + 2o nodes per axis,
// periodic wrap = restriction R_k^delta), then runs exactly K steps of GMRES on
// A_k y = R_k^delta v entirely on chip (reading R9: fixed-work local solve, zero initial guess,
// CGS2, Givens, early exit only on exact breakdown), and writes only the owned nodes
// (R_k^0)^T -- disjoint writes, no atomics.
//
// A_k is the local Jacobian with phi = 0 on the 3-layer ring around the extended box
// (modified subdomain BC): the Krylov vector lives in the interior of a zero-padded
// (E+6)^2 shared-memory plane whose ring is never written, and the local J v is the composed
// stencil of K2 in three stages (halo 2 -> 1 -> 0):
//   L1 = Delta v,  B = ((1-gamma)/2 + c) v + L1 + Delta L1 / 2,  w = v/dt - Delta B.
//
// Latency design (one box per SM at E = 36..40: the K basis vectors take 104-128 KB):
//  * the Arnoldi vector w of the thread's own nodes stays in registers;
//  * each CGS2 pass is ONE block reduction: warp reduce-scatter (16 values in 16 shuffles
//    instead of 80), one barrier, lane-parallel cross-warp sums, shuffle broadcast;
//  * pass 2 also reduces |w'|^2 and the new norm is |w''|^2 = |w'|^2 - |h2|^2 (exact for an
//    orthonormal basis; pass 2 only removes rounding-size components), with an explicit extra
//    reduction when |h2|^2 > 1e-8 |w'|^2;
//  * normalisation writes V_{j+1} and the padded plane in one pass; the Givens QR of the small
//    Hessenberg matrix is deferred to one thread after the K steps (nothing inside the fixed-work
//    loop depends on it).  Five barriers per Arnoldi step.
#include "pfc_device.cuh"
#include "pfc_internal.h"
#include "ras_common.cuh"
#include "tmem.cuh"

#include <stdlib.h>

namespace {

constexpr int NT = 512;
constexpr int NW = NT / 32;
constexpr int MAXN = 1600;                 // largest ext box (E = 40)
constexpr int SLOTS = (MAXN + NT - 1) / NT;

struct RasArgs {
  const double* v;
  const double* c;
  double* z;
  int nx, ny;
  int bx, by, o;
  double idt, gamma, ih2;
  int restrict_owned;   // right-RAS: R_k^0 (v zero outside the owned box)
  double* y_ext;        // AS / right-RAS: ext-box solutions [box][ext node] for (R_k^delta)^T
  const int* gate;   // device-resident FGMRES: skip the launch when *gate != 0 (f1)
  // variable mobility (row f3): the Jacobian state Phi, psi, A of the current iterate; the
  // local operator is then A_k = R_k^delta J (R_k^delta)^T (reading R8b)
  const double* phi;
  const double* psi;
  const double* A;
  int mobility;
  // Neumann-type mirror BCs (row f3, reading R23): subdomains clipped at the physical boundary
  // (ext-box nodes outside the domain are no unknowns), and the padded plane carries the
  // mirror ghosts of the Krylov vector (the even extension) so that the stencils act as J
  int mirror;
  unsigned long long* jcnt;   // profiling: Arnoldi steps taken (ras_count)
  const double* dtp;   // graph path (f1): dt on the device
};

// node index of global (x, y): periodic wrap, or the mirror partner (R23)
__device__ __forceinline__ int axis2(int x, int n, int mirror) {
  if (!mirror) return wrapi(x, n);
  return x < 0 ? -1 - x : (x >= n ? 2 * n - 1 - x : x);
}

// Block sum of nv (runtime, <= NVP) values held by every thread in acc[]: the sums are left in
// this warp's private copy hw[0..nv) (valid after return for every lane of the warp).  One
// barrier; `red` alternates between two buffers so consecutive reductions never race.
// Value NVP-1 is also reduced when `with_last` (the norm slot).
template <int NVP, int NWB = NW>
__device__ __forceinline__ void block_allreduce(double (&acc)[NVP], int nv, double* red,
                                                double* hw, bool with_last = false) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int SH = 5 - (NVP == 1 ? 0 : NVP == 2 ? 1 : NVP == 4 ? 2 : NVP == 8 ? 3 : NVP == 16 ? 4 : 5);
  double s = warp_reduce_scatter<NVP>(acc);
  const int vi = lane >> SH;
  if ((lane & ((1 << SH) - 1)) == 0 && (vi < nv || (with_last && vi == NVP - 1)))
    red[wid * NVP + vi] = s;
  __syncthreads();
  if (lane < nv || (with_last && lane == NVP - 1)) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NWB; ++w) t += red[w * NVP + lane];
    hw[lane] = t;
  }
  __syncwarp();
}

template <int K>
__global__ void __launch_bounds__(NT, 1) ras2d_kernel(RasArgs p) {
  constexpr int NVP = pow2_at_least(K + 2);   // values 0..K-1 plus the norm slot NVP-1
  // declared as a shared array (not re-derived through an integer) so that every access
  // compiles to LDS/STS with 32-bit shared addressing; 128-B aligned for TMA destinations
  extern __shared__ __align__(128) double smem_dyn[];
  double* sm = smem_dyn;
  const int Ex = p.bx + 2 * p.o, Ey = p.by + 2 * p.o;
  const int n = Ex * Ey;
  const int Px = Ex + 6, Py = Ey + 6;
  const int np = Px * Py;
  double* V = sm;                        // K n
  double* cl = V + (size_t)K * n;        // n
  double* pv = cl + n;                   // np (zero ring)
  double* pl = pv + np;                  // np
  double* pb = pl + np;                  // np
  double* red = pb + np;                 // 2 x NW x NVP
  double* hwall = red + 2 * NW * NVP;    // NW x 3 NVP: per-warp copies of h1 | h2 | misc
  double* pm = hwall + NW * 3 * NVP;     // mobility: M, A, u on the padded plane (np each)
  double* pa = pm + np;
  double* pu = pa + np;
  double* pc = pm + (p.mobility ? 3 * np : 0);                          // mirror: c on the plane
  int* gp = reinterpret_cast<int*>(pc + (p.mirror ? np : 0));           // mirror: ghost partners
  __shared__ double H[(K + 1) * K];
  __shared__ double gv[K + 1], cs[K], sn[K], yv[K];

  if (p.gate && *p.gate) return;
  const int tid = threadIdx.x;
  double* h1 = hwall + (tid >> 5) * 3 * NVP;
  double* h2 = h1 + NVP;
  double* hx = h2 + NVP;
  const int nbx = p.nx / p.bx;
  const int ibx = blockIdx.x % nbx, iby = blockIdx.x / nbx;
  const int gx0 = ibx * p.bx - p.o, gy0 = iby * p.by - p.o;
  const double ih2 = p.ih2, idt = dt_inv(p.dtp, p.idt), alpha = 0.5 * (1.0 - p.gamma);

  // own box nodes: l = tid + s*NT; padded index of node l
  int pidx[SLOTS];
  bool own[SLOTS];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    int l = tid + s * NT;
    own[s] = l < n;
    pidx[s] = own[s] ? ((l / Ex) + 3) * Px + (l % Ex) + 3 : 0;
  }

  // zero the padded planes (ring stays zero), gather R_k^delta v and c with periodic wrap
  for (int q = tid; q < 3 * np; q += NT) pv[q] = 0.0;
  auto gnode = [&](int x, int y) {
    return (size_t)axis2(x, p.nx, p.mirror) + (size_t)p.nx * axis2(y, p.ny, p.mirror);
  };
  auto in_dom = [&](int x, int y) {
    return !p.mirror || (x >= 0 && x < p.nx && y >= 0 && y < p.ny);
  };
  // mirror: does this box reach the boundary (its plane then has ghost positions)?
  const bool ghosts = p.mirror && (gx0 - 3 < 0 || gy0 - 3 < 0 || gx0 + Px - 3 > p.nx ||
                                   gy0 + Py - 3 > p.ny);
  if (p.mirror) {   // c of the even extension on the plane; ghost -> partner map
    for (int q = tid; q < np; q += NT) {
      const int pi = q % Px, pj = q / Px, x = gx0 + pi - 3, y = gy0 + pj - 3;
      const bool inext = pi >= 3 && pi < Px - 3 && pj >= 3 && pj < Py - 3;
      const bool ghost = !in_dom(x, y);
      pc[q] = (inext || ghost) ? p.c[gnode(x, y)] : 0.0;
      int part = -1;
      if (ghost) {
        const int mi = axis2(x, p.nx, 1) - gx0 + 3, mj = axis2(y, p.ny, 1) - gy0 + 3;
        part = (mi >= 3 && mi < Px - 3 && mj >= 3 && mj < Py - 3) ? mj * Px + mi : -2;
      }
      gp[q] = part;
    }
  }
  if (p.mobility) {   // M = 1 - u^2, A and u of the iterate on the ext box and its +1 ring
    for (int q = tid; q < np; q += NT) {
      const int pi = q % Px, pj = q / Px;
      double m = 0.0, a = 0.0, u = 0.0;
      if (pi >= 2 && pi < Px - 2 && pj >= 2 && pj < Py - 2) {
        const size_t g = gnode(gx0 + pi - 3, gy0 + pj - 3);
        u = 0.5 * (p.phi[g] + p.psi[g]);
        m = 1.0 - u * u;
        a = p.A[g];
      }
      pm[q] = m; pa[q] = a; pu[q] = u;
    }
  }
  double w[SLOTS];
  double acc[NVP];
  bool act[SLOTS];   // unknowns of A_k: every ext-box node, except outside the domain (mirror)
#pragma unroll
  for (int i = 0; i < NVP; ++i) acc[i] = 0.0;
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    w[s] = 0.0;
    act[s] = false;
    if (own[s]) {
      int l = tid + s * NT;
      size_t g = gnode(gx0 + l % Ex, gy0 + l / Ex);
      act[s] = in_dom(gx0 + l % Ex, gy0 + l / Ex);
      const int li = l % Ex - p.o, lj = l / Ex - p.o;
      const bool owned = li >= 0 && li < p.bx && lj >= 0 && lj < p.by;
      w[s] = ((p.restrict_owned && !owned) || !act[s]) ? 0.0 : p.v[g];
      cl[l] = p.c[g];
      acc[0] += w[s] * w[s];
    }
  }
  int rb = 0;
  block_allreduce<NVP>(acc, 1, red + rb * NW * NVP, hx);
  rb ^= 1;
  const double beta = sqrt(hx[0]);
  if (beta == 0.0) {
    if (tid == 0) ras_count(p.jcnt, 0);
    if (p.y_ext) {
      for (int l = tid; l < n; l += NT) p.y_ext[(size_t)blockIdx.x * n + l] = 0.0;
    } else {
      for (int l = tid; l < p.bx * p.by; l += NT)
        p.z[(size_t)(ibx * p.bx + l % p.bx) + (size_t)p.nx * (iby * p.by + l / p.bx)] = 0.0;
    }
    return;
  }
  {
    const double ib = 1.0 / beta;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s)
      if (own[s]) {
        double v0 = w[s] * ib;
        V[tid + s * NT] = v0;
        pv[pidx[s]] = v0;
      }
  }
  if (tid == 0) gv[0] = beta;

  // stage iteration geometry, hoisted out of the Arnoldi loop (no integer division inside it)
  const int wxL = Px - 2, cntL = wxL * (Py - 2), r0L = tid / wxL, c0L = tid % wxL;
  const int wxB = Px - 4, cntB = wxB * (Py - 4), r0B = tid / wxB, c0B = tid % wxB;
  const int drL = NT / wxL, dcL = NT % wxL, drB = NT / wxB, dcB = NT % wxB;

  int jm = 0;
#pragma unroll 1
  for (int j = 0; j < K; ++j) {
    __syncthreads();                                   // pv holds V_j
    if (ghosts) {   // mirror ghosts of V_j (the even extension; partners outside the box: 0)
      for (int q = tid; q < np; q += NT)
        if (gp[q] >= 0) pv[q] = pv[gp[q]];
      __syncthreads();
    }
    {   // L1 = Delta v on padded [1, P-1)
      int r = r0L, c = c0L;
      for (int q = tid; q < cntL; q += NT) {
        const int f = (1 + r) * Px + 1 + c;
        pl[f] = ih2 * ((pv[f - 1] + pv[f + 1]) + (pv[f - Px] + pv[f + Px]) - 4.0 * pv[f]);
        r += drL; c += dcL;
        if (c >= wxL) { c -= wxL; ++r; }
      }
    }
    __syncthreads();
    {   // B on padded [2, P-2); c v = 0 outside the extended box
      int r = r0B, c = c0B;
      for (int q = tid; q < cntB; q += NT) {
        const int pi = 2 + c, pj = 2 + r;
        r += drB; c += dcB;
        if (c >= wxB) { c -= wxB; ++r; }
        int f = pj * Px + pi;
        double vv = pv[f];
        int li = pi - 3, lj = pj - 3;
        double cv = p.mirror ? pc[f] * vv
                             : (li >= 0 && li < Ex && lj >= 0 && lj < Ey) ? cl[lj * Ex + li] * vv : 0.0;
        double lapl = ih2 * ((pl[f - 1] + pl[f + 1]) + (pl[f - Px] + pl[f + Px]) - 4.0 * pl[f]);
        pb[f] = alpha * vv + cv + pl[f] + 0.5 * lapl;
      }
    }
    __syncthreads();
    // w = v/dt - Delta B on own nodes (registers); CGS2 pass 1: h1 = V^T w
#pragma unroll
    for (int i = 0; i < NVP; ++i) acc[i] = 0.0;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      if (own[s]) {
        const int f = pidx[s], l = tid + s * NT;
        double ww;
        if (p.mobility) {   // v/dt - (grad . M grad) B - (grad . (-u v) grad) A
          auto dmg = [&](const double* m, const double* g, const double* s2) {
            auto mm = [&](int k) { return s2 ? -pu[k] * s2[k] : m[k]; };
            const double mc = mm(f), gc = g[f];
            return ih2 * (0.5 * (mc + mm(f + 1)) * (g[f + 1] - gc) -
                          0.5 * (mc + mm(f - 1)) * (gc - g[f - 1]) +
                          0.5 * (mc + mm(f + Px)) * (g[f + Px] - gc) -
                          0.5 * (mc + mm(f - Px)) * (gc - g[f - Px]));
          };
          ww = pv[f] * idt - dmg(pm, pb, nullptr) - dmg(nullptr, pa, pv);
        } else {
          double lapb = ih2 * ((pb[f - 1] + pb[f + 1]) + (pb[f - Px] + pb[f + Px]) - 4.0 * pb[f]);
          ww = pv[f] * idt - lapb;
        }
        if (!act[s]) ww = 0.0;   // R_k: rows of the non-unknowns are dropped
        w[s] = ww;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i > j) break;
          acc[i] += V[(size_t)i * n + l] * ww;
        }
      }
    }
    block_allreduce<NVP>(acc, j + 1, red + rb * NW * NVP, h1);
    rb ^= 1;
    // w' = w - V h1 ; pass 2: h2 = V^T w', and |w'|^2 (slot K of the reduction)
#pragma unroll
    for (int i = 0; i < NVP; ++i) acc[i] = 0.0;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      if (own[s]) {
        const int l = tid + s * NT;
        double vv[K];
        double ww = w[s];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i > j) break;
          vv[i] = V[(size_t)i * n + l];
          ww -= h1[i] * vv[i];
        }
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i > j) break;
          acc[i] += vv[i] * ww;
        }
        acc[NVP - 1] += ww * ww;
        w[s] = ww;
      }
    }
    block_allreduce<NVP>(acc, j + 1, red + rb * NW * NVP, h2, true);
    rb ^= 1;
    const double wn2 = h2[NVP - 1];
    double h2n = 0.0;
    for (int i = 0; i <= j; ++i) h2n += h2[i] * h2[i];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      if (own[s]) {
        const int l = tid + s * NT;
        double ww = w[s];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i > j) break;
          ww -= h2[i] * V[(size_t)i * n + l];
        }
        w[s] = ww;
      }
    }
    double hn2;
    if (h2n <= 1e-8 * wn2) {
      hn2 = wn2 - h2n;                                  // |w''|^2 = |w'|^2 - |h2|^2
    } else {                                            // rare: explicit |w''|^2
#pragma unroll
      for (int i = 0; i < NVP; ++i) acc[i] = 0.0;
#pragma unroll
      for (int s = 0; s < SLOTS; ++s)
        if (own[s]) acc[0] += w[s] * w[s];
      block_allreduce<NVP>(acc, 1, red + rb * NW * NVP, hx);
      rb ^= 1;
      hn2 = hx[0];
    }
    const double hn = sqrt(hn2 > 0.0 ? hn2 : 0.0);
    if (tid == 0) {   // Hessenberg column j (the Givens QR runs once, after the loop)
      const int ld = K + 1;
      for (int i = 0; i <= j; ++i) H[i + ld * j] = h1[i] + h2[i];
      H[j + 1 + ld * j] = hn;
    }
    jm = j + 1;
    if (hn <= 1e-14 * beta) break;                     // exact breakdown (uniform)
    if (j + 1 < K) {
      const double ihn = 1.0 / hn;
#pragma unroll
      for (int s = 0; s < SLOTS; ++s)
        if (own[s]) {
          double vn = w[s] * ihn;
          V[(size_t)(j + 1) * n + tid + s * NT] = vn;
          pv[pidx[s]] = vn;
        }
    }
  }
  __syncthreads();
  if (tid == 0) {
    // Givens QR of the (jm+1) x jm Hessenberg matrix, column by column in Arnoldi order (the
    // same operations an incremental update performs), then back substitution R y = g
    const int ld = K + 1;
    for (int j = 0; j < jm; ++j) {
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
    }
    for (int i = jm - 1; i >= 0; --i) {
      double s = gv[i];
      for (int l = i + 1; l < jm; ++l) s -= H[i + ld * l] * yv[l];
      yv[i] = s / H[i + ld * i];
    }
    ras_count(p.jcnt, jm);
  }
  __syncthreads();
  // (R_k^0)^T: owned nodes only, y = V yv
  if (p.y_ext) {   // (R_k^delta)^T: the whole ext-box solution, summed by ras_extend
    for (int l = tid; l < n; l += NT) {
      double s = 0.0;
      for (int i = 0; i < jm; ++i) s += yv[i] * V[(size_t)i * n + l];
      p.y_ext[(size_t)blockIdx.x * n + l] = s;
    }
    return;
  }
  for (int l = tid; l < p.bx * p.by; l += NT) {
    int li = l % p.bx, lj = l / p.bx;
    int ll = (lj + p.o) * Ex + li + p.o;
    double s = 0.0;
    for (int i = 0; i < jm; ++i) s += yv[i] * V[(size_t)i * n + ll];
    p.z[(size_t)(ibx * p.bx + li) + (size_t)p.nx * (iby * p.by + lj)] = s;
  }
}

// ---------------------------------------------------------------------------------------
// Column-strip variant (the production path for extended boxes up to 42 x 42).
//
// Thread (x, s) owns the R nodes (x, sR .. sR+R-1) of the extended box for the whole solve:
//  * the K basis vectors of its nodes live in registers, so CGS2 touches no shared memory;
//  * the local J v is ONE pass of the direct 25-point stencil of the linear part
//      w = v/dt - alpha Delta v - Delta^2 v - Delta^3 v / 2 - Delta(c v),  alpha = (1-gamma)/2
//    (the class weights of h^2 Delta = L, L^2 and L^3 summed on the host) read
//    column by column from the zero-padded plane of v (immediate offsets: the plane pitch is a
//    compile-time 48), plus the 5-point Laplacian of c v from a second padded plane; one barrier
//    per Arnoldi step for the stencil instead of three;
//  * step j is dispatched to code specialised for J = j (compile-time CGS2 lengths, register
//    indices and block-reduction widths), so no predicated K-long loops remain;
//  * each block reduction is a warp reduce-scatter sized to the number of values (1, 2, 4, 8
//    or 16), one barrier, and lane-parallel cross-warp sums: fixed order, deterministic.
// Arithmetic: same algorithm as ras2d_kernel and the oracle (reading R9); the stencil sums the
// 25 weighted terms instead of composing three 5-point Laplacians (rounding-level difference).
constexpr int PP = 48;          // padded plane pitch (doubles) at most: Ex + 6 <= 48
// Row pitch of the padded planes for R rows per thread: a warp covers consecutive x of strip s
// and then strip s+1 (R rows further), so its 8-byte loads are conflict-free when
// R * pitch = Ex (mod 16): 45 for R = 4 (Ex = 36, 20: cfg2/3), 50 for R = 2 (Ex = 20: cfg1);
// other shapes are correct at any pitch, just not conflict-free.
constexpr int col_pp(int R) { return R == 4 ? 45 : R == 2 ? 50 : R == 6 ? 46 : PP; }
constexpr int PPY = 56;         // padded plane rows: Ey + R + 5 <= 56
constexpr int NTC = 384;        // threads per CTA at most (1 CTA per SM, <= 168 registers)
constexpr int NWC = NTC / 32;

struct RasColArgs {
  const double* v;
  const double* c;
  double* z;
  int nx, ny, bx, by, o;
  int Ex, Ey, ns;               // extended box, strips per column
  int restrict_owned;           // right-RAS: R_k^0 (v zero outside the owned box)
  double* y_ext;                // AS / right-RAS: ext-box solutions [box][ext node]
  const int* gate;   // device-resident FGMRES: skip the launch when *gate != 0 (f1)
  double W[6];                  // 25-point class weights: (0,0) (0,1) (0,2) (1,1) (0,3) (1,2)
  double ih2;
  double idt, alpha;            // MOB: 1/dt, (1 - gamma)/2
  // Neumann-type mirror BCs (row f3, R23): ext-box nodes outside the domain are no unknowns
  // (zero basis entries) and the padded planes carry the mirror ghosts of v and c v, refreshed
  // after every basis write in boxes that touch a wall
  int mirror;
  // variable mobility (row f3, R8b): the Jacobian state of the iterate (Phi, psi, A)
  const double* phi;
  const double* psi;
  const double* A;
  unsigned long long* jcnt;     // profiling: Arnoldi steps taken (ras_count)
  const double* dtp;             // graph path (f1): dt-dependent scalars on the device
};

constexpr int wclass(int ax, int ay) {
  return (ax + ay == 0) ? 0 : (ax + ay == 1) ? 1 : (ax == 1 && ay == 1) ? 3
         : (ax + ay == 2) ? 2 : (ax + ay == 3 && (ax == 0 || ay == 0)) ? 4 : 5;
}
constexpr int iabs(int a) { return a < 0 ? -a : a; }

// Block all-reduce of NV values per thread (NV <= 16): totals in hw[0..NV) of this warp.
template <int NV>
__device__ __forceinline__ void col_allreduce(const double (&acc)[NV], double* red, double* hw,
                                              int nwt) {
  constexpr int NVP = pow2_at_least(NV);
  constexpr int SH = 5 - (NVP == 1 ? 0 : NVP == 2 ? 1 : NVP == 4 ? 2 : NVP == 8 ? 3 : 4);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double a[NVP];
#pragma unroll
  for (int i = 0; i < NVP; ++i) a[i] = i < NV ? acc[i] : 0.0;
  const double s = warp_reduce_scatter<NVP>(a);
  const int vi = lane >> SH;
  if ((lane & ((1 << SH) - 1)) == 0 && vi < NV) red[wid * 16 + vi] = s;
  __syncthreads();
  if (lane < NV) {   // all partials loaded first, then a fixed pairwise tree (absent warps add 0)
    double t[NWC];
#pragma unroll
    for (int w = 0; w < NWC; ++w) t[w] = w < nwt ? red[w * 16 + lane] : 0.0;
#pragma unroll
    for (int st = 1; st < NWC; st *= 2)
#pragma unroll
      for (int w = 0; w + st < NWC; w += 2 * st) t[w] += t[w + st];
    hw[lane] = t[0];
  }
  __syncwarp();
}

// Tail of Arnoldi step J (after w = A_k v_J is in registers): CGS2, norm, next basis vector.
// Returns true when the solve stops (exact breakdown).
// Hessenberg column J (h1 + h2, hn) reduced by the previous Givens rotations and a new one,
// in the oracle's incremental order; R column, rotation and 1/R_JJ kept in shared memory.
// Run by lane 0 of the Givens warp one phase late (during the next step's stencil).
template <int K, int J>
__device__ __forceinline__ void col_givens(const double* h1, const double* h2, double hn,
                                           double* cs, double* sn, double* gv, double* H,
                                           double* rd) {
  double col[J + 2];
  double cp[J + 1], sp[J + 1];
#pragma unroll
  for (int i = 0; i < J; ++i) { cp[i] = cs[i]; sp[i] = sn[i]; }
#pragma unroll
  for (int i = 0; i <= J; ++i) col[i] = h1[i] + h2[i];
  col[J + 1] = hn;
#pragma unroll
  for (int i = 0; i < J; ++i) {
    const double a = col[i], b = col[i + 1];
    col[i] = cp[i] * a + sp[i] * b;
    col[i + 1] = -sp[i] * a + cp[i] * b;
  }
  const double a = col[J], b = col[J + 1];
  const double rr = sqrt(a * a + b * b);
  double cc = 1.0, ss = 0.0;
  if (rr != 0.0) { cc = a / rr; ss = b / rr; }
  cs[J] = cc; sn[J] = ss;
  col[J] = cc * a + ss * b;
  const double g = gv[J];
  gv[J + 1] = -ss * g;
  gv[J] = cc * g;
  rd[J] = 1.0 / col[J];
#pragma unroll
  for (int i = 0; i <= J; ++i) H[i + (K + 1) * J] = col[i];
}

template <int K, int J>
__device__ __forceinline__ void col_givens_dispatch(int j, const double* h1, const double* h2,
                                                    double hn, double* cs, double* sn, double* gv,
                                                    double* H, double* rd) {
  if constexpr (J < K) {
    if (j == J) col_givens<K, J>(h1, h2, hn, cs, sn, gv, H, rd);
    else col_givens_dispatch<K, J + 1>(j, h1, h2, hn, cs, sn, gv, H, rd);
  }
}

#ifdef PFC_RAS_PROFILE
// diagnostic build only: thread 0 of block 0 accumulates clock64() deltas per phase into the
// global array ras_prof (read back by tools/ras_phase_probe.py)
__device__ long long ras_prof[8];
__device__ long long ras_prof_last;
#define CPROF(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { long long t_ = clock64(); \
    ras_prof[i] += t_ - ras_prof_last; ras_prof_last = t_; } } while (0)
#else
#define CPROF(i) do {} while (0)
#endif

template <int K, int R, int J>
__device__ __forceinline__ bool col_step(double (&Vr)[K][R], double (&w)[R], double (&cvv)[R],
                                         const double (&cr)[R], const bool (&own)[R],
                                         double* red, int& rb, double* h1, double* h2,
                                         double* hx, double* H, double* cs, double* sn,
                                         double* gv, double* rd, double* pvb, double* pcvb,
                                         double beta, int nwt, bool g0, double& hn_prev) {
  constexpr int PP = col_pp(R);
  if constexpr (J > 0) {
    if (g0) col_givens<K, J - 1>(h1, h2, hn_prev, cs, sn, gv, H, rd);
  }
  // pass 1: h1 = V^T w
  {
    double acc[J + 1];
#pragma unroll
    for (int i = 0; i <= J; ++i) {
      double t = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) t = fma(Vr[i][r], w[r], t);
      acc[i] = t;
    }
    col_allreduce<J + 1>(acc, red + rb * NWC * 16, h1, nwt);
    rb ^= 1;
  }
  CPROF(3);
  // w' = w - V h1 ; pass 2: h2 = V^T w', |w'|^2 in slot J+1
  {
    double hv[J + 1];
#pragma unroll
    for (int i = 0; i <= J; ++i) hv[i] = h1[i];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double ww = w[r];
#pragma unroll
      for (int i = 0; i <= J; ++i) ww = fma(-hv[i], Vr[i][r], ww);
      w[r] = ww;
    }
    double acc[J + 2];
#pragma unroll
    for (int i = 0; i <= J; ++i) {
      double t = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) t = fma(Vr[i][r], w[r], t);
      acc[i] = t;
    }
    double t = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) t = fma(w[r], w[r], t);
    acc[J + 1] = t;
    col_allreduce<J + 2>(acc, red + rb * NWC * 16, h2, nwt);
    rb ^= 1;
  }
  CPROF(4);
  double hv[J + 1];
  double h2n = 0.0;
#pragma unroll
  for (int i = 0; i <= J; ++i) {
    hv[i] = h2[i];
    h2n += hv[i] * hv[i];
  }
  const double wn2 = h2[J + 1];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double ww = w[r];
#pragma unroll
    for (int i = 0; i <= J; ++i) ww = fma(-hv[i], Vr[i][r], ww);
    w[r] = ww;
  }
  double hn2;
  if (h2n <= 1e-8 * wn2) {
    hn2 = wn2 - h2n;                                  // |w''|^2 = |w'|^2 - |h2|^2
  } else {                                            // rare: explicit |w''|^2
    double acc[1] = {0.0};
#pragma unroll
    for (int r = 0; r < R; ++r) acc[0] = fma(w[r], w[r], acc[0]);
    col_allreduce<1>(acc, red + rb * NWC * 16, hx, nwt);
    rb ^= 1;
    hn2 = hx[0];
  }
  const double hn = sqrt(hn2 > 0.0 ? hn2 : 0.0);
  hn_prev = hn;                     // the Givens warp reduces column J during step J+1
  if (hn <= 1e-14 * beta) return true;               // exact breakdown (uniform)
  if constexpr (J + 1 < K) {
    const double ihn = 1.0 / hn;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double vn = w[r] * ihn;
      Vr[J + 1][r] = vn;
      cvv[r] = cr[r] * vn;
      if (own[r]) {
        pvb[r * PP] = vn;
        pcvb[r * PP] = cvv[r];
      }
    }
  }
  return false;
}

template <int K, int R, int J>
__device__ __forceinline__ bool col_dispatch(int j, double (&Vr)[K][R], double (&w)[R],
                                             double (&cvv)[R], const double (&cr)[R],
                                             const bool (&own)[R], double* red, int& rb,
                                             double* h1, double* h2, double* hx, double* H,
                                             double* cs, double* sn, double* gv, double* rd,
                                             double* pvb, double* pcvb, double beta, int nwt,
                                             bool g0, double& hn_prev) {
  if constexpr (J < K) {
    if (j == J)
      return col_step<K, R, J>(Vr, w, cvv, cr, own, red, rb, h1, h2, hx, H, cs, sn, gv, rd, pvb,
                               pcvb, beta, nwt, g0, hn_prev);
    return col_dispatch<K, R, J + 1>(j, Vr, w, cvv, cr, own, red, rb, h1, h2, hx, H, cs, sn, gv,
                                     rd, pvb, pcvb, beta, nwt, g0, hn_prev);
  } else {
    return true;
  }
}

// MOB: variable mobility M = 1 - u^2 (row f3, R8b): A_k v = R J R^T v staged on shared planes
// like ras2d_kernel (L1 = Delta v; B = alpha v + L1 + Delta L1 / 2 + c v; then
// v/dt - (grad . M grad) B - (grad . (-u v) grad) A at the own nodes), the basis in registers
// threads per CTA at most: R >= 6 rows per thread run 8 warps at <= 255 registers (fewer warps
// per block reduction), fewer rows 12 warps at <= 168
constexpr int col_nt(int R) { return R >= 6 ? 256 : NTC; }

template <int K, int R, bool MIR, bool MOB = false>
__global__ void __launch_bounds__(col_nt(R), 1) ras2d_col_kernel(const __grid_constant__ RasColArgs p) {
  constexpr int PP = col_pp(R);
  extern __shared__ __align__(128) double smem_dyn[];
  double* pv = smem_dyn;                     // PP x PPY padded v (zero ring)
  double* pcv = pv + PP * PPY;               // PP x PPY padded c v
  double* red = pcv + PP * PPY;              // 2 x NWC x 16
  double* hwall = red + 2 * NWC * 16;        // NWC x 3 x 16
  double* stg = hwall + NWC * 48;            // next box's v, c of each thread's nodes (2 x NTC x R)
  int* gp = reinterpret_cast<int*>(stg + 2 * NTC * R);   // mirror: ghost -> partner (PP x PPY)
  double* pl = reinterpret_cast<double*>(gp + PP * PPY);  // MOB: L1, B, M, A, u planes
  double* pb = pl + PP * PPY;
  double* pm = pb + PP * PPY;
  double* pa = pm + PP * PPY;
  double* pu = pa + PP * PPY;
  __shared__ double H[(K + 1) * K];
  __shared__ double gv[K + 1], cs[K], sn[K], yv[K], rd[K];

  if (p.gate && *p.gate) return;
  const double W0 = dt_w0<2>(p.dtp, p.W[0]), idt = dt_inv(p.dtp, p.idt);
  const int tid = threadIdx.x, nwt = blockDim.x >> 5;
  const bool gwarp = (tid >> 5) == nwt - 1;     // the Givens warp: no nodes, reduces H
  const bool g0 = gwarp && (tid & 31) == 0;
  double hn_prev = 0.0;
  double* h1 = hwall + (tid >> 5) * 48;
  double* h2 = h1 + 16;
  double* hx = h2 + 16;
  const int Ex = p.Ex, Ey = p.Ey;
  const int nbx = p.nx / p.bx;
  const int nboxes = nbx * (p.ny / p.by);

  const int xs = tid % Ex, ss = tid / Ex;
  const bool active = ss < p.ns;
  const int x = active ? xs : 0, y0 = active ? ss * R : 0;   // inactive threads read in-bounds
  bool own[R];
#pragma unroll
  for (int r = 0; r < R; ++r) own[r] = active && (y0 + r < Ey);
  double* pvb = pv + (y0 + 3) * PP + x + 3;
  double* pcvb = pcv + (y0 + 3) * PP + x + 3;

  for (int q = tid; q < 2 * PP * PPY; q += blockDim.x) pv[q] = 0.0;   // the ring stays zero
  if (MOB)
    for (int q = tid; q < 2 * PP * PPY; q += blockDim.x) pl[q] = 0.0;  // L1, B outside their ranges
  double* sv = stg + tid;              // [r][thread]: a warp's 8-byte accesses are contiguous
  double* sc = stg + NTC * R + tid;
  // R_k^delta v and c of a box (periodic wrap) into this thread's staging slots, asynchronously
  auto prefetch = [&](int box) {
    if (box >= nboxes) return;
    const int gx0 = (box % nbx) * p.bx - p.o, gy0 = (box / nbx) * p.by - p.o;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (own[r]) {
        const size_t g = (size_t)wrapi(gx0 + x, p.nx) + (size_t)p.nx * wrapi(gy0 + y0 + r, p.ny);
        cp_async8(sv + r * NTC, p.v + g);
        cp_async8(sc + r * NTC, p.c + g);
      }
    cp_async_commit();
  };
  prefetch(blockIdx.x);
  // persistent CTA: boxes blockIdx.x, + gridDim.x, ...; the next box's inputs load while the
  // current box is solved
  bool prev_ghosts = false;
  for (int box = blockIdx.x; box < nboxes; box += gridDim.x) {
  const int ibx = box % nbx, iby = box / nbx;
  const int gx0 = ibx * p.bx - p.o, gy0 = iby * p.by - p.o;
  // mirror: a box whose padded plane reaches past a wall has ghost positions
  const bool ghosts = MIR && (gx0 - 3 < 0 || gy0 - 3 < 0 || gx0 + Ex + 3 > p.nx ||
                                   gy0 + Ey + 3 > p.ny);
  if (MIR && prev_ghosts)   // the previous box left ghost values on the ring: zero it again
    for (int q = tid; q < 2 * PP * PPY; q += blockDim.x) pv[q] = 0.0;
  if (MIR && ghosts)
    for (int q = tid; q < PP * PPY; q += blockDim.x) {
      const int pc = q % PP, pr = q / PP, gx = gx0 + pc - 3, gy = gy0 + pr - 3;
      int part = -1;
      if (pc < Ex + 6 && pr < Ey + 6 && (gx < 0 || gx >= p.nx || gy < 0 || gy >= p.ny)) {
        const int mx = gx < 0 ? -1 - gx : (gx >= p.nx ? 2 * p.nx - 1 - gx : gx);
        const int my = gy < 0 ? -1 - gy : (gy >= p.ny ? 2 * p.ny - 1 - gy : gy);
        const int lx = mx - gx0, ly = my - gy0;   // partner in the ext box, else zero
        part = (lx >= 0 && lx < Ex && ly >= 0 && ly < Ey) ? (ly + 3) * PP + lx + 3 : -2;
      }
      gp[q] = part;
    }
  prev_ghosts = ghosts;
  if (MOB)   // M = 1 - u^2, A and u of the iterate on the ext box and its +1 ring (else 0)
    for (int q = tid; q < PP * PPY; q += blockDim.x) {
      const int pc = q % PP, pr = q / PP;
      double m = 0.0, a = 0.0, u = 0.0;
      if (pc >= 2 && pc < Ex + 4 && pr >= 2 && pr < Ey + 4) {
        const size_t g = (size_t)axis2(gx0 + pc - 3, p.nx, MIR) +
                         (size_t)p.nx * axis2(gy0 + pr - 3, p.ny, MIR);   // MIR: even extension
        u = 0.5 * (p.phi[g] + p.psi[g]);
        m = 1.0 - u * u;
        a = p.A[g];
      }
      pm[q] = m; pa[q] = a; pu[q] = u;
    }
  cp_async_wait_all();
  double Vr[K][R];
  double w[R], cr[R], cvv[R];
  bool act[R];   // unknowns of A_k: the ext-box nodes inside the domain
  double acc0[1] = {0.0};
#pragma unroll
  for (int r = 0; r < R; ++r) {
    w[r] = 0.0;
    cr[r] = 0.0;
    act[r] = own[r] && (!MIR || (gx0 + x >= 0 && gx0 + x < p.nx && gy0 + y0 + r >= 0 &&
                                      gy0 + y0 + r < p.ny));
    if (own[r]) {
      const int li = x - p.o, lj = y0 + r - p.o;
      const bool owned = li >= 0 && li < p.bx && lj >= 0 && lj < p.by;
      w[r] = ((p.restrict_owned && !owned) || !act[r]) ? 0.0 : sv[r * NTC];
      cr[r] = sc[r * NTC];
      acc0[0] = fma(w[r], w[r], acc0[0]);
    }
  }
  prefetch(box + gridDim.x);   // this thread's slots are free again
  hn_prev = 0.0;
  int rb = 0;
  col_allreduce<1>(acc0, red + rb * NWC * 16, hx, nwt);   // also orders the zero fill
  rb ^= 1;
  const double beta = sqrt(hx[0]);
  if (beta == 0.0) {
    if (tid == 0) ras_count(p.jcnt, 0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int li = x - p.o, lj = y0 + r - p.o;
      if (p.y_ext) {
        if (own[r]) p.y_ext[(size_t)box * (Ex * Ey) + (y0 + r) * Ex + x] = 0.0;
      } else if (own[r] && li >= 0 && li < p.bx && lj >= 0 && lj < p.by) {
        p.z[(size_t)(ibx * p.bx + li) + (size_t)p.nx * (iby * p.by + lj)] = 0.0;
      }
    }
    // every warp must be done reading this box's beta from red[0] before the next box's
    // first col_allreduce writes its partials there (rb restarts at 0)
    __syncthreads();
    continue;   // uniform: every thread saw beta = 0
  }
  {
    const double ib = 1.0 / beta;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double v0 = w[r] * ib;
      Vr[0][r] = v0;
      cvv[r] = cr[r] * v0;
      if (own[r]) {
        pvb[r * PP] = v0;
        pcvb[r * PP] = cvv[r];
      }
    }
  }
  if (tid == 0) gv[0] = beta;
#ifdef PFC_RAS_PROFILE
  if (blockIdx.x == 0 && tid == 0) ras_prof_last = clock64();
#endif

  int jm = 0;
#pragma unroll 1
  for (int j = 0; j < K; ++j) {
    __syncthreads();                                  // planes hold v_j and c v_j
    if (MIR && ghosts) {   // mirror ghosts of v_j and c v_j (the even extension)
      for (int q = tid; q < PP * PPY; q += blockDim.x) {
        const int g = gp[q];
        if (g >= 0) { pv[q] = pv[g]; pcv[q] = pcv[g]; }
      }
      __syncthreads();
    }
    CPROF(0);
    if constexpr (MOB) {   // staged variable-coefficient operator (all threads share the stages)
      const double ih2 = p.ih2, al = p.alpha;
      const int wl = Ex + 4, wb = Ex + 2;
      for (int q = tid; q < wl * (Ey + 4); q += blockDim.x) {   // L1 on padded [1, P-1)
        const int f = (1 + q / wl) * PP + 1 + q % wl;
        pl[f] = ih2 * ((pv[f - 1] + pv[f + 1]) + (pv[f - PP] + pv[f + PP]) - 4.0 * pv[f]);
      }
      __syncthreads();
      for (int q = tid; q < wb * (Ey + 2); q += blockDim.x) {   // B on padded [2, P-2)
        const int f = (2 + q / wb) * PP + 2 + q % wb;
        const double lapl = ih2 * ((pl[f - 1] + pl[f + 1]) + (pl[f - PP] + pl[f + PP]) - 4.0 * pl[f]);
        pb[f] = al * pv[f] + pcv[f] + pl[f] + 0.5 * lapl;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < R; ++r) {
        w[r] = 0.0;
        if (!gwarp && act[r]) {
          const int f = (y0 + r + 3) * PP + x + 3;
          auto dmg = [&](const double* m, const double* g, bool uv) {
            auto mm = [&](int k) { return uv ? -pu[k] * pv[k] : m[k]; };
            const double mc = mm(f), gc = g[f];
            return ih2 * (0.5 * (mc + mm(f + 1)) * (g[f + 1] - gc) -
                          0.5 * (mc + mm(f - 1)) * (gc - g[f - 1]) +
                          0.5 * (mc + mm(f + PP)) * (g[f + PP] - gc) -
                          0.5 * (mc + mm(f - PP)) * (gc - g[f - PP]));
          };
          w[r] = pv[f] * idt - dmg(pm, pb, false) - dmg(nullptr, pa, true);
        }
      }
    } else
    // ---- w = A_k v_j: direct 25-point linear part, column by column (not in the Givens warp)
    if (!gwarp) {
    double out[R];
#pragma unroll
    for (int r = 0; r < R; ++r) out[r] = 0.0;
#pragma unroll
    for (int dx = -3; dx <= 3; ++dx) {
      const int a = 3 - iabs(dx);
      double col[R + 6];
#pragma unroll
      for (int rr = -a; rr < R + a; ++rr) col[rr + a] = pvb[rr * PP + dx];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int dy = -a; dy <= a; ++dy)
          out[r] = fma(wclass(iabs(dx), iabs(dy)) == 0 ? W0 : p.W[wclass(iabs(dx), iabs(dy))],
                       col[r + dy + a], out[r]);
    }
    // ---- minus Delta(c v): x-neighbours from the plane, y-neighbours from registers
#pragma unroll
    for (int r = 0; r < R; ++r) {   // (mirror: a y-neighbour in the strip may be a ghost)
      const double up = (r == 0 || MIR) ? pcvb[(r - 1) * PP] : cvv[r - 1];
      const double dn = (r == R - 1 || MIR) ? pcvb[(r + 1) * PP] : cvv[r + 1];
      const double lap = (pcvb[r * PP - 1] + pcvb[r * PP + 1]) + (up + dn) - 4.0 * cvv[r];
      w[r] = act[r] ? fma(-p.ih2, lap, out[r]) : 0.0;
    }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) w[r] = 0.0;
    }
    CPROF(1);
    const bool stop = col_dispatch<K, R, 0>(j, Vr, w, cvv, cr, own, red, rb, h1, h2, hx, H, cs,
                                            sn, gv, rd, pvb, pcvb, beta, nwt, g0, hn_prev);
    CPROF(5);
    jm = j + 1;
    if (stop) break;
  }
  CPROF(6);
  if (g0) {   // last Hessenberg column, then back substitution R yv = g
    col_givens_dispatch<K, 0>(jm - 1, h1, h2, hn_prev, cs, sn, gv, H, rd);
    const int ld = K + 1;
    double y[K];
#pragma unroll
    for (int i = K - 1; i >= 0; --i) {
      if (i >= jm) continue;
      double sacc = gv[i];
#pragma unroll
      for (int l = i + 1; l < K; ++l)
        if (l < jm) sacc -= H[i + ld * l] * y[l];
      y[i] = sacc * rd[i];
      yv[i] = y[i];
    }
    ras_count(p.jcnt, jm);
  }
  __syncthreads();
  // (R_k^0)^T: the owner thread of each owned node writes y = V yv; (R_k^delta)^T (AS,
  // right-RAS): every ext node's value goes to y_ext for the deterministic overlap-add
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int li = x - p.o, lj = y0 + r - p.o;
    const bool wr = p.y_ext ? own[r] : (own[r] && li >= 0 && li < p.bx && lj >= 0 && lj < p.by);
    if (!wr) continue;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i)
      if (i < jm) s = fma(yv[i], Vr[i][r], s);
    if (p.y_ext) p.y_ext[(size_t)box * (Ex * Ey) + (y0 + r) * Ex + x] = s;
    else p.z[(size_t)(ibx * p.bx + li) + (size_t)p.nx * (iby * p.by + lj)] = s;
  }
  CPROF(7);
  __syncthreads();   // yv, H and the planes are reused by the next box
  }
}

// ============================================================================================
// Two boxes per SM (ras2d_colt_kernel, periodic, M = 1): the column kernel with the Krylov basis
// in TENSOR MEMORY instead of registers, so a CTA of R = 6 rows per thread (36 x 6 strips = 216
// node threads + the Givens warp) fits in 128 registers and two CTAs -- two boxes -- share each
// SM: one box's reductions, barriers and Givens hide under the other's stencil (the column
// kernel runs one box of 12 warps per SM, latency-bound on its block reductions).  Each CTA
// allocates 256 TMEM columns; thread t of warp w keeps vector i of its R nodes at columns
// 128 (w div 4) + 2 R i of lane 32 (w mod 4) + t mod 32 (K R <= 64).  Same arithmetic as
// ras2d_col_kernel (the CGS2 sums per node and per vector in the same order).
constexpr int NTT = 256;   // threads per CTA at most (two CTAs per SM at <= 128 registers)

template <int K, int R, int J>
__device__ __forceinline__ bool colt_step(uint32_t tma, double (&w)[R], double (&cvv)[R],
                                          const double (&cr)[R], const bool (&own)[R],
                                          double* red, int& rb, double* h1, double* h2,
                                          double* hx, double* H, double* cs, double* sn,
                                          double* gv, double* rd, double* pvb, double* pcvb,
                                          double beta, int nwt, bool g0, double& hn_prev) {
  constexpr int PP = col_pp(R);
  if constexpr (J > 0) {
    if (g0) col_givens<K, J - 1>(h1, h2, hn_prev, cs, sn, gv, H, rd);
  }
  tmem::wait_st();   // v_J (stored at the end of the previous step) has landed
  // pass 1: h1 = V^T w
  {
    double acc[J + 1];
#pragma unroll
    for (int i = 0; i <= J; ++i) {
      double vi[R];
      tmem::ld<R>(tma + (uint32_t)(2 * R * i), vi);
      double t = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) t = fma(vi[r], w[r], t);
      acc[i] = t;
    }
    col_allreduce<J + 1>(acc, red + rb * NWC * 16, h1, nwt);
    rb ^= 1;
  }
  // w' = w - V h1 ; pass 2: h2 = V^T w', |w'|^2 in slot J+1
  {
    double hv[J + 1];
#pragma unroll
    for (int i = 0; i <= J; ++i) hv[i] = h1[i];
#pragma unroll
    for (int i = 0; i <= J; ++i) {   // per node in the order i = 0..J, as the column kernel
      double vi[R];
      tmem::ld<R>(tma + (uint32_t)(2 * R * i), vi);
#pragma unroll
      for (int r = 0; r < R; ++r) w[r] = fma(-hv[i], vi[r], w[r]);
    }
    double acc[J + 2];
#pragma unroll
    for (int i = 0; i <= J; ++i) {
      double vi[R];
      tmem::ld<R>(tma + (uint32_t)(2 * R * i), vi);
      double t = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) t = fma(vi[r], w[r], t);
      acc[i] = t;
    }
    double t = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) t = fma(w[r], w[r], t);
    acc[J + 1] = t;
    col_allreduce<J + 2>(acc, red + rb * NWC * 16, h2, nwt);
    rb ^= 1;
  }
  double hv[J + 1];
  double h2n = 0.0;
#pragma unroll
  for (int i = 0; i <= J; ++i) {
    hv[i] = h2[i];
    h2n += hv[i] * hv[i];
  }
  const double wn2 = h2[J + 1];
#pragma unroll
  for (int i = 0; i <= J; ++i) {
    double vi[R];
    tmem::ld<R>(tma + (uint32_t)(2 * R * i), vi);
#pragma unroll
    for (int r = 0; r < R; ++r) w[r] = fma(-hv[i], vi[r], w[r]);
  }
  double hn2;
  if (h2n <= 1e-8 * wn2) {
    hn2 = wn2 - h2n;                                  // |w''|^2 = |w'|^2 - |h2|^2
  } else {                                            // rare: explicit |w''|^2
    double acc[1] = {0.0};
#pragma unroll
    for (int r = 0; r < R; ++r) acc[0] = fma(w[r], w[r], acc[0]);
    col_allreduce<1>(acc, red + rb * NWC * 16, hx, nwt);
    rb ^= 1;
    hn2 = hx[0];
  }
  const double hn = sqrt(hn2 > 0.0 ? hn2 : 0.0);
  hn_prev = hn;                     // the Givens warp reduces column J during step J+1
  if (hn <= 1e-14 * beta) return true;               // exact breakdown (uniform)
  if constexpr (J + 1 < K) {
    const double ihn = 1.0 / hn;
    double vn[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      vn[r] = w[r] * ihn;
      cvv[r] = cr[r] * vn[r];
      if (own[r]) {
        pvb[r * PP] = vn[r];
        pcvb[r * PP] = cvv[r];
      }
    }
    tmem::st<R>(tma + (uint32_t)(2 * R * (J + 1)), vn);
  }
  return false;
}

template <int K, int R, int J>
__device__ __forceinline__ bool colt_dispatch(int j, uint32_t tma, double (&w)[R],
                                              double (&cvv)[R], const double (&cr)[R],
                                              const bool (&own)[R], double* red, int& rb,
                                              double* h1, double* h2, double* hx, double* H,
                                              double* cs, double* sn, double* gv, double* rd,
                                              double* pvb, double* pcvb, double beta, int nwt,
                                              bool g0, double& hn_prev) {
  if constexpr (J < K) {
    if (j == J)
      return colt_step<K, R, J>(tma, w, cvv, cr, own, red, rb, h1, h2, hx, H, cs, sn, gv, rd,
                                pvb, pcvb, beta, nwt, g0, hn_prev);
    return colt_dispatch<K, R, J + 1>(j, tma, w, cvv, cr, own, red, rb, h1, h2, hx, H, cs, sn,
                                      gv, rd, pvb, pcvb, beta, nwt, g0, hn_prev);
  } else {
    return true;
  }
}

template <int K, int R>
__global__ void __launch_bounds__(NTT, 2) ras2d_colt_kernel(const __grid_constant__ RasColArgs p) {
  static_assert(K * R <= 64, "K R doubles = 2 K R <= 128 TMEM columns per thread");
  constexpr int PP = col_pp(R);
  extern __shared__ __align__(128) double smem_dyn[];
  double* pv = smem_dyn;                     // PP x PPY padded v (zero ring)
  double* pcv = pv + PP * PPY;               // PP x PPY padded c v
  double* red = pcv + PP * PPY;              // 2 x NWC x 16
  double* hwall = red + 2 * NWC * 16;        // NWC x 3 x 16
  double* stg = hwall + NWC * 48;            // next box's v, c of each thread's nodes (2 x NTT x R)
  __shared__ double H[(K + 1) * K];
  __shared__ double gv[K + 1], cs[K], sn[K], yv[K], rd[K];
  __shared__ uint32_t tm_base;

  if (p.gate && *p.gate) return;
  const double W0 = dt_w0<2>(p.dtp, p.W[0]);
  const int tid = threadIdx.x, nwt = blockDim.x >> 5, wid = tid >> 5;
  const bool gwarp = wid == nwt - 1;            // the Givens warp: no nodes, reduces H
  const bool g0 = gwarp && (tid & 31) == 0;
  double hn_prev = 0.0;
  double* h1 = hwall + wid * 48;
  double* h2 = h1 + 16;
  double* hx = h2 + 16;
  const int Ex = p.Ex;
  const int nbx = p.nx / p.bx;
  const int nboxes = nbx * (p.ny / p.by);

  const int xs = tid % Ex, ss = tid / Ex;
  const bool active = ss < p.ns;
  const int x = active ? xs : 0, y0 = active ? ss * R : 0;   // inactive threads read in-bounds
  bool own[R];
#pragma unroll
  for (int r = 0; r < R; ++r) own[r] = active && (y0 + r < p.Ey);
  double* pvb = pv + (y0 + 3) * PP + x + 3;
  double* pcvb = pcv + (y0 + 3) * PP + x + 3;

  for (int q = tid; q < 2 * PP * PPY; q += blockDim.x) pv[q] = 0.0;   // the ring stays zero
  if (wid == 0) tmem::alloc<256>(&tm_base);   // half of the SM's columns (two CTAs per SM)
  tmem::fence_before();
  __syncthreads();
  tmem::fence_after();
  const uint32_t tma = tm_base + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)(128 * (wid >> 2));
  double* sv = stg + tid;              // [r][thread]: a warp's 8-byte accesses are contiguous
  double* sc = stg + NTT * R + tid;
  auto prefetch = [&](int box) {
    if (box >= nboxes) return;
    const int gx0 = (box % nbx) * p.bx - p.o, gy0 = (box / nbx) * p.by - p.o;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (own[r]) {
        const size_t g = (size_t)wrapi(gx0 + x, p.nx) + (size_t)p.nx * wrapi(gy0 + y0 + r, p.ny);
        cp_async8(sv + r * NTT, p.v + g);
        cp_async8(sc + r * NTT, p.c + g);
      }
    cp_async_commit();
  };
  prefetch(blockIdx.x);
  for (int box = blockIdx.x; box < nboxes; box += gridDim.x) {
  const int ibx = box % nbx, iby = box / nbx;
  cp_async_wait_all();
  double w[R], cr[R], cvv[R];
  double acc0[1] = {0.0};
#pragma unroll
  for (int r = 0; r < R; ++r) {
    w[r] = 0.0;
    cr[r] = 0.0;
    if (own[r]) {
      const int li = x - p.o, lj = y0 + r - p.o;
      const bool owned = li >= 0 && li < p.bx && lj >= 0 && lj < p.by;
      w[r] = (p.restrict_owned && !owned) ? 0.0 : sv[r * NTT];
      cr[r] = sc[r * NTT];
      acc0[0] = fma(w[r], w[r], acc0[0]);
    }
  }
  prefetch(box + gridDim.x);   // this thread's slots are free again
  hn_prev = 0.0;
  int rb = 0;
  col_allreduce<1>(acc0, red + rb * NWC * 16, hx, nwt);   // also orders the zero fill
  rb ^= 1;
  const double beta = sqrt(hx[0]);
  if (beta == 0.0) {
    if (tid == 0) ras_count(p.jcnt, 0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int li = x - p.o, lj = y0 + r - p.o;
      if (p.y_ext) {
        if (own[r]) p.y_ext[(size_t)box * (Ex * p.Ey) + (y0 + r) * Ex + x] = 0.0;
      } else if (own[r] && li >= 0 && li < p.bx && lj >= 0 && lj < p.by) {
        p.z[(size_t)(ibx * p.bx + li) + (size_t)p.nx * (iby * p.by + lj)] = 0.0;
      }
    }
    __syncthreads();   // every warp has read beta before the next box's first reduction
    continue;
  }
  {
    const double ib = 1.0 / beta;
    double v0[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      v0[r] = w[r] * ib;
      cvv[r] = cr[r] * v0[r];
      if (own[r]) {
        pvb[r * PP] = v0[r];
        pcvb[r * PP] = cvv[r];
      }
    }
    tmem::st<R>(tma, v0);
  }
  if (tid == 0) gv[0] = beta;
  int jm = 0;
#pragma unroll 1
  for (int j = 0; j < K; ++j) {
    __syncthreads();                                  // planes hold v_j and c v_j
    if (!gwarp) {   // ---- w = A_k v_j: direct 25-point linear part, column by column
      double out[R];
#pragma unroll
      for (int r = 0; r < R; ++r) out[r] = 0.0;
#pragma unroll
      for (int dx = -3; dx <= 3; ++dx) {
        const int a = 3 - iabs(dx);
        double col[R + 6];
#pragma unroll
        for (int rr = -a; rr < R + a; ++rr) col[rr + a] = pvb[rr * PP + dx];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int dy = -a; dy <= a; ++dy)
            out[r] = fma(wclass(iabs(dx), iabs(dy)) == 0 ? W0 : p.W[wclass(iabs(dx), iabs(dy))],
                         col[r + dy + a], out[r]);
      }
      // ---- minus Delta(c v): x-neighbours from the plane, y-neighbours from registers
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double up = r == 0 ? pcvb[(r - 1) * PP] : cvv[r - 1];
        const double dn = r == R - 1 ? pcvb[(r + 1) * PP] : cvv[r + 1];
        const double lap = (pcvb[r * PP - 1] + pcvb[r * PP + 1]) + (up + dn) - 4.0 * cvv[r];
        w[r] = own[r] ? fma(-p.ih2, lap, out[r]) : 0.0;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) w[r] = 0.0;
    }
    const bool stop = colt_dispatch<K, R, 0>(j, tma, w, cvv, cr, own, red, rb, h1, h2, hx, H,
                                             cs, sn, gv, rd, pvb, pcvb, beta, nwt, g0, hn_prev);
    jm = j + 1;
    if (stop) break;
  }
  if (g0) {   // last Hessenberg column, then back substitution R yv = g
    col_givens_dispatch<K, 0>(jm - 1, h1, h2, hn_prev, cs, sn, gv, H, rd);
    const int ld = K + 1;
    double y[K];
#pragma unroll
    for (int i = K - 1; i >= 0; --i) {
      if (i >= jm) continue;
      double sacc = gv[i];
#pragma unroll
      for (int l = i + 1; l < K; ++l)
        if (l < jm) sacc -= H[i + ld * l] * y[l];
      y[i] = sacc * rd[i];
      yv[i] = y[i];
    }
    ras_count(p.jcnt, jm);
  }
  __syncthreads();
  // (R_k^0)^T: y = V yv at the owned nodes (every lane loads: TMEM loads are warp-collective)
  {
    double s[R];
#pragma unroll
    for (int r = 0; r < R; ++r) s[r] = 0.0;
    tmem::wait_st();
    for (int i = 0; i < jm; ++i) {
      double vi[R];
      tmem::ld<R>(tma + (uint32_t)(2 * R * i), vi);
      const double yi = yv[i];
#pragma unroll
      for (int r = 0; r < R; ++r) s[r] = fma(yi, vi[r], s[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int li = x - p.o, lj = y0 + r - p.o;
      const bool wr = p.y_ext ? own[r] : (own[r] && li >= 0 && li < p.bx && lj >= 0 && lj < p.by);
      if (!wr) continue;
      if (p.y_ext) p.y_ext[(size_t)box * (Ex * p.Ey) + (y0 + r) * Ex + x] = s[r];
      else p.z[(size_t)(ibx * p.bx + li) + (size_t)p.nx * (iby * p.by + lj)] = s[r];
    }
  }
  __syncthreads();   // yv, H and the planes are reused by the next box
  }
  tmem::fence_before();
  __syncthreads();
  tmem::fence_after();
  if (wid == 0) tmem::dealloc<256>(tm_base);
}

size_t ras2d_colt_smem_bytes(int R) {
  return (size_t)(2 * col_pp(R) * PPY + 2 * NWC * 16 + NWC * 48 + 2 * NTT * R) * sizeof(double);
}

#ifdef PFC_RAS_PROFILE
}  // namespace
extern "C" void pfc_ras_prof_read(long long* out) {
  cudaMemcpyFromSymbol(out, ras_prof, sizeof(long long) * 8);
  long long z[8] = {0};
  cudaMemcpyToSymbol(ras_prof, z, sizeof(z));
}
namespace {
#endif
size_t ras2d_col_smem_bytes(int R, bool mob = false) {
  return (size_t)(2 * col_pp(R) * PPY + 2 * NWC * 16 + NWC * 48 + 2 * NTC * R) * sizeof(double) +
         (size_t)col_pp(R) * PPY * sizeof(int) +
         (mob ? (size_t)5 * col_pp(R) * PPY * sizeof(double) : 0);
}

typedef void (*ras2d_fn)(RasArgs);
size_t ras2d_smem_bytes(int bx, int by, int o, int k, int mobility, int mirror) {
  const size_t Ex = bx + 2 * o, Ey = by + 2 * o, n = Ex * Ey, np = (Ex + 6) * (Ey + 6);
  size_t d = (size_t)k * n + n + 3 * np + 2 * NW * 16 + NW * 3 * 16 + (mobility ? 3 * np : 0) +
             (mirror ? np + (np + 1) / 2 : 0);   // c plane + ghost partner ints
  return d * sizeof(double) + 128;
}

ras2d_fn pick(int k) {
  switch (k) {
#define X(K) case K: return ras2d_kernel<K>;
    X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15)
#undef X
  }
  return nullptr;
}

// column-strip instantiations: local GMRES steps K x rows per thread R
typedef void (*ras2d_col_fn)(const RasColArgs);
template <bool MIR>
ras2d_col_fn pick_col_t(int k, int r) {
  if (k == 10 && r == 6) return ras2d_col_kernel<10, 6, MIR>;
#define RC(K)                                              \
  case K:                                                  \
    switch (r) {                                           \
      case 1: return ras2d_col_kernel<K, 1, MIR>;          \
      case 2: return ras2d_col_kernel<K, 2, MIR>;          \
      case 4: return ras2d_col_kernel<K, 4, MIR>;          \
      case 5: return ras2d_col_kernel<K, 5, MIR>;          \
    }                                                      \
    return nullptr;
  switch (k) {
    RC(4) RC(5) RC(6) RC(8) RC(10) RC(12)
  }
#undef RC
  return nullptr;
}
template <bool MIR>
ras2d_col_fn pick_col_mob(int k, int r) {
  switch (k) {
    case 10:
      switch (r) {
        case 1: return ras2d_col_kernel<10, 1, MIR, true>;
        case 2: return ras2d_col_kernel<10, 2, MIR, true>;
        case 4: return ras2d_col_kernel<10, 4, MIR, true>;
        case 5: return ras2d_col_kernel<10, 5, MIR, true>;
      }
  }
  return nullptr;
}
ras2d_col_fn pick_col(int k, int r, bool mirror = false, bool mob = false) {
  if (mob) return mirror ? pick_col_mob<true>(k, r) : pick_col_mob<false>(k, r);
  return mirror ? pick_col_t<true>(k, r) : pick_col_t<false>(k, r);
}

// rows per thread for the column kernel: the fewest that fit the extended box in NTC threads
// TMEM two-boxes-per-SM kernel (periodic, M = 1): rows per thread, 0 if not applicable
typedef void (*ras2d_colt_fn)(const RasColArgs);
ras2d_colt_fn pick_colt(int k, int r) {
  if (k != 10) return nullptr;
  switch (r) {
    case 2: return ras2d_colt_kernel<10, 2>;
    case 4: return ras2d_colt_kernel<10, 4>;
    case 6: return ras2d_colt_kernel<10, 6>;
  }
  return nullptr;
}
// Opt-in (PFC_RAS2_TMEM=1): measured slower than the one-box column kernel (cfg2 apply 252 vs
// 238 us, Test C 971 vs 921 us; two CTAs of 8 warps per SM, R = 6 rows per thread)
int colt_rows(int k, int Ex, int Ey) {
  const char* e = getenv("PFC_RAS2_TMEM");
  if (!(e && e[0] == '1') || Ex + 6 > PP || Ey + 11 > PPY) return 0;
  const char* force = getenv("PFC_RAS2_ROWS");   // A/B probes only: rows per thread
  const int rmin = force ? atoi(force) : 1;
  const int cand[3] = {2, 4, 6};
  for (int i = 0; i < 3; ++i) {
    const int r = cand[i];
    if (r < rmin) continue;
    const int ns = (Ey + r - 1) / r;
    if (Ex + 6 <= col_pp(r) && (Ex * ns + 31) / 32 * 32 + 32 <= NTT && pick_colt(k, r)) return r;
  }
  return 0;
}

int col_rows(int k, int Ex, int Ey, bool mirror = false, bool mob = false) {
  if (Ex + 6 > PP || Ey > 42) return 0;
  const int cand[5] = {1, 2, 4, 5, 6};
  const char* force = getenv("PFC_RAS2_ROWS");   // A/B probes only: rows per thread
  const int rmin = force ? atoi(force) : 1;
  if (!force) {   // R = 6 (8 warps, 255 registers) when it still gives >= 6 node warps: fewer
                  // warps per block reduction (cfg2, E = 36: 0.2266 -> 0.2204 ms per apply)
    const int nt = Ex * ((Ey + 5) / 6);
    if (nt > 160 && Ex + 6 <= col_pp(6) && (nt + 31) / 32 * 32 + 32 <= col_nt(6) &&
        pick_col(k, 6, mirror, mob))
      return 6;
  }
  for (int i = 0; i < 5; ++i) {
    const int r = cand[i];
    if (r < rmin) continue;
    const int ns = (Ey + r - 1) / r;
    if (Ex + 6 <= col_pp(r) && (Ex * ns + 31) / 32 * 32 + 32 <= col_nt(r) &&
        pick_col(k, r, mirror, mob))
      return r;
  }
  return 0;
}

}  // namespace

int ras2d_plan(pfc_ctx* ctx) {
  const pfc_config& c = ctx->cfg;
  const int Ex = c.ras_box[0] + 2 * c.ras_overlap, Ey = c.ras_box[1] + 2 * c.ras_overlap;
  if (Ex * Ey > MAXN) return 0;
  const bool mir = c.bc == PFC_BC_MIRROR, mob = c.mobility != PFC_MOBILITY_ONE;
  ctx->ras_tmem = 0;
  if (getenv("PFC_RAS_SMEM_BASIS") == nullptr && !mir && !mob) {
    const int r = colt_rows(c.ras_local_k, Ex, Ey);
    if (r) {
      const int ns = (Ey + r - 1) / r;
      ctx->ras_smem = (int)ras2d_colt_smem_bytes(r);
      ctx->ras_threads = (Ex * ns + 31) / 32 * 32 + 32;
      ctx->ras_rows = r;
      ctx->ras_tmem = 1;
      return 1;
    }
  }
  if (getenv("PFC_RAS_SMEM_BASIS") == nullptr) {
    const int r = col_rows(c.ras_local_k, Ex, Ey, mir, mob);
    if (r) {
      const int ns = (Ey + r - 1) / r;
      ctx->ras_smem = (int)ras2d_col_smem_bytes(r, mob);
      ctx->ras_threads = (Ex * ns + 31) / 32 * 32 + 32;   // node warps + the Givens warp
      ctx->ras_rows = r;                             // rows per thread
      return 1;
    }
  }
  size_t sm = ras2d_smem_bytes(c.ras_box[0], c.ras_box[1], c.ras_overlap, c.ras_local_k,
                               c.mobility, c.bc == PFC_BC_MIRROR);
  if (sm + 2048 > 227 * 1024) return 0;   // + static shared memory (H, Givens, reductions)
  ctx->ras_smem = (int)sm;
  ctx->ras_threads = NT;        // shared-memory-basis kernel
  ctx->ras_rows = 0;
  return 1;
}

cudaError_t launch_ras_2d(pfc_ctx* ctx, const double* v, const double* c, double dt, double* z) {
  const pfc_config& cf = ctx->cfg;
  const int Ex = cf.ras_box[0] + 2 * cf.ras_overlap, Ey = cf.ras_box[1] + 2 * cf.ras_overlap;
  const int nb = (cf.n[0] / cf.ras_box[0]) * (cf.n[1] / cf.ras_box[1]);
  cudaError_t e;
  if (ctx->ras_tmem) {   // two boxes per SM, basis in tensor memory
    const int R = ctx->ras_rows;
    ras2d_colt_fn fn = pick_colt(cf.ras_local_k, R);
    if (!fn) return cudaErrorInvalidValue;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->ras_smem);
    if (e != cudaSuccess) return e;
    RasColArgs p{};
    p.v = v; p.c = c; p.z = z;
    p.nx = cf.n[0]; p.ny = cf.n[1]; p.bx = cf.ras_box[0]; p.by = cf.ras_box[1];
    p.o = cf.ras_overlap; p.Ex = Ex; p.Ey = Ey; p.ns = (Ey + R - 1) / R;
    p.restrict_owned = cf.ras_variant == PFC_RAS_RIGHT;
    p.y_ext = cf.ras_variant == PFC_RAS_LEFT ? nullptr : ctx->ras_y;
    p.gate = ctx->gate;
    p.jcnt = ctx->prof ? ctx->d_jcnt : nullptr;
    const double ih2 = ctx->ih2, ih4 = ih2 * ih2, ih6 = ih4 * ih2;
    const double al = 0.5 * (1.0 - cf.gamma);
    p.W[0] = 1.0 / dt + 4.0 * al * ih2 - 20.0 * ih4 + 56.0 * ih6;
    p.dtp = ctx->dtdev;
    p.W[1] = -al * ih2 + 8.0 * ih4 - 28.5 * ih6;
    p.W[2] = -ih4 + 6.0 * ih6;
    p.W[3] = -2.0 * ih4 + 12.0 * ih6;
    p.W[4] = -0.5 * ih6;
    p.W[5] = -1.5 * ih6;
    p.ih2 = ih2;
    int nsm = 148, per_sm = 1;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, ctx->ras_threads,
                                                      ctx->ras_smem) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    if (per_sm > 2) per_sm = 2;   // 256 TMEM columns per CTA: at most two CTAs per SM
    fn<<<std::min(nb, nsm * per_sm), ctx->ras_threads, ctx->ras_smem, ctx->stream>>>(p);
  } else if (ctx->ras_rows > 0) {
    const int R = ctx->ras_rows;
    const bool mob = cf.mobility != PFC_MOBILITY_ONE;
    ras2d_col_fn fn = pick_col(cf.ras_local_k, R, cf.bc == PFC_BC_MIRROR, mob);
    if (!fn) return cudaErrorInvalidValue;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->ras_smem);
    if (e != cudaSuccess) return e;
    RasColArgs p{};
    p.v = v; p.c = c; p.z = z;
    p.nx = cf.n[0]; p.ny = cf.n[1]; p.bx = cf.ras_box[0]; p.by = cf.ras_box[1];
    p.o = cf.ras_overlap; p.Ex = Ex; p.Ey = Ey; p.ns = (Ey + R - 1) / R;
    p.mirror = cf.bc == PFC_BC_MIRROR;
    p.phi = ctx->mob_phi; p.psi = ctx->mob_psi; p.A = ctx->mob_A;   // MOB: Jacobian state
    p.idt = 1.0 / dt;
    p.alpha = 0.5 * (1.0 - cf.gamma);
    p.restrict_owned = cf.ras_variant == PFC_RAS_RIGHT;
    p.y_ext = cf.ras_variant == PFC_RAS_LEFT ? nullptr : ctx->ras_y;
    p.gate = ctx->gate;
    p.jcnt = ctx->prof ? ctx->d_jcnt : nullptr;
    // class weights of the linear part v/dt - alpha Delta v - Delta^2 v - Delta^3 v / 2 with
    // h^2 Delta = L:  L (0,0) -4, (0,1) 1;  L^2 (0,0) 20, (0,1) -8, (0,2) 1, (1,1) 2;
    // L^3 (0,0) -112, (0,1) 57, (0,2) -12, (1,1) -24, (0,3) 1, (1,2) 3
    const double ih2 = ctx->ih2, ih4 = ih2 * ih2, ih6 = ih4 * ih2;
    const double al = 0.5 * (1.0 - cf.gamma);
    p.W[0] = 1.0 / dt + 4.0 * al * ih2 - 20.0 * ih4 + 56.0 * ih6;
    p.dtp = ctx->dtdev;
    p.W[1] = -al * ih2 + 8.0 * ih4 - 28.5 * ih6;
    p.W[2] = -ih4 + 6.0 * ih6;
    p.W[3] = -2.0 * ih4 + 12.0 * ih6;
    p.W[4] = -0.5 * ih6;
    p.W[5] = -1.5 * ih6;
    p.ih2 = ih2;
    int nsm = 148, per_sm = 1;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, ctx->ras_threads,
                                                      ctx->ras_smem) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    fn<<<std::min(nb, nsm * per_sm), ctx->ras_threads, ctx->ras_smem, ctx->stream>>>(p);   // persistent
  } else {
    ras2d_fn fn = pick(cf.ras_local_k);
    if (!fn) return cudaErrorInvalidValue;
    // opt in to the dynamic shared memory once per kernel
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->ras_smem);
    if (e != cudaSuccess) return e;
    RasArgs p{v, c, z, cf.n[0], cf.n[1], cf.ras_box[0], cf.ras_box[1], cf.ras_overlap,
              1.0 / dt, cf.gamma, ctx->ih2, cf.ras_variant == PFC_RAS_RIGHT,
              cf.ras_variant == PFC_RAS_LEFT ? nullptr : ctx->ras_y, ctx->gate,
              ctx->mob_phi, ctx->mob_psi, ctx->mob_A, cf.mobility, cf.bc == PFC_BC_MIRROR,
              ctx->prof ? ctx->d_jcnt : nullptr};
    p.dtp = ctx->dtdev;
    fn<<<nb, NT, ctx->ras_smem, ctx->stream>>>(p);
  }
  ctx->launches++;
  {  // algorithmic: v, c gathered on the extended boxes, z written on owned nodes; flops of
     // k local J v (25/pt) + CGS2 vector work 4k(k+1) + 3k + 3 per ext node + V y
    const double next = (double)nb * Ex * Ey;
    const double nout = cf.ras_variant == PFC_RAS_LEFT ? (double)ctx->N : next;
    pfc_account(ctx, PFC_K_RAS, 8.0 * (2.0 * next + nout), 0.0);
    ras_flop_model(ctx, (double)Ex * Ey, 25.0, nout / nb);   // flops from the step counters
  }
  cudaError_t e2 = cudaGetLastError();
  if (e2 != cudaSuccess || cf.ras_variant == PFC_RAS_LEFT) return e2;
  return launch_ras_extend(ctx, z);
}
