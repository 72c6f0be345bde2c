// ras3d_col.cu -- Schwarz subdomain solves in 3D with the Krylov vector on chip (K4, sm_100a).
//
// Same algorithm as ras3d.cu / ras2d.cu and the oracle: Eq. (eq:ras) P:398-409 (and the AS /
// right-RAS variants), the modified subdomain BC phi = 0 on the 3-layer ring
// as zero padding, and exactly K steps of GMRES with CGS2 and Givens (reading R9).
//
// One CTA per extended box of E^3 nodes (E = b + 2o, e.g. 20^3 for the configs' 16^3 boxes with
// overlap 2), persistent over the boxes.  Thread (x, y) owns the z-column of its E nodes:
//  * the current Krylov vector v_j lives zero-padded in x and y in shared memory (E planes of
//    (E+6) rows at a row pitch PXR >= E+6 with PXR = E (mod 16), 146 KB at E = 20) next to c on
//    the box (E^3, 64 KB).  A warp covers 32 consecutive (x, y) of rows of E nodes, so with
//    PXR = E (mod 16) its 8-byte loads hit every bank pair exactly twice (conflict-free; the
//    plain (E+6) pitch cost 3.1 wavefronts per load instead of 2).  The z-direction needs no
//    zero planes: the unrolled z loop skips the out-of-box planes at compile time;
//  * the local J v is ONE pass of the direct 63-point stencil of the linear part
//      w = v/dt - alpha Delta v - Delta^2 v - Delta^3 v / 2 - Delta(c v),  alpha = (1-gamma)/2
//    (class weights of h^2 Delta = L, L^2, L^3 summed on the host), read column by column with
//    compile-time offsets: 25 xy offsets, each a z-segment of E + 2(3 - |dx| - |dy|) values
//    accumulated into the thread's E outputs in registers;
//  * the K basis vectors (E^3 each) are too large for one SM: they stay in a per-CTA global
//    scratch region that is L2-resident (148 CTAs x K x 64 KB), and every thread only ever
//    reads back its own column of them (coalesced across the warp);
//  * step j is dispatched to code specialised for J = j (CGS2 lengths and reduction widths),
//    block reductions are sized reduce-scatters with one barrier (ras_common.cuh);
//  * the Givens update of column j runs on thread 0 right after the reductions (a few hundred
//    cycles against ~10^4 per step).
#include "pfc_device.cuh"
#include "pfc_internal.h"
#include "ras_common.cuh"

namespace {

constexpr int NW3MAX = 16;     // warps per CTA at most (E <= 22)

struct Ras3ColArgs {
  const double* v;
  const double* c;
  double* z;
  double* basis;         // per-CTA scratch: K x E^3 doubles per CTA
  int nx, ny, nz, bx, by, bz, o;
  int restrict_owned;    // right-RAS: R_k^0
  double* y_ext;         // AS / right-RAS: ext-box solutions [box][ext node]
  const int* gate;       // device-resident FGMRES: skip when *gate != 0
  double W[7];           // classes (0,0,0) (0,0,1) (0,0,2) (0,1,1) (0,0,3) (0,1,2) (1,1,1)
  double ih2;
  unsigned long long* jcnt;   // profiling: Arnoldi steps taken (ras_count)
  const double* dtp;     // graph path (f1): dt-dependent scalars on the device
};

constexpr int iabs3(int a) { return a < 0 ? -a : a; }
// class of the offset (|dx|, |dy|, |dz|), sorted: 000, 001, 002, 011, 003, 012, 111
constexpr int wclass3(int a, int b, int c) {
  return (a + b + c == 0) ? 0
         : (a + b + c == 1) ? 1
         : (a + b + c == 2) ? ((a == 2 || b == 2 || c == 2) ? 2 : 3)
         : ((a == 3 || b == 3 || c == 3) ? 4 : ((a == 1 && b == 1 && c == 1) ? 6 : 5));
}

// row pitch of the padded plane: >= E + 6 and = E (mod 16) (conflict-free warp rows)
constexpr int col3_pxr(int E) { return E + 6 + ((E - (E + 6)) % 16 + 16) % 16; }

template <int E>
struct Col3 {
  static constexpr int PXR = col3_pxr(E);    // row pitch (x)
  static constexpr int PY = E + 6;           // padded rows (y)
  static constexpr int PP = PXR * PY;        // plane pitch (z: E planes, no ring)
};

// Contribution of the xy offset (DX, DY) to the thread's E outputs: the z-segment of that
// column within reach A = 3 - |DX| - |DY| (all bounds compile-time, so out[] stays in registers)
template <int E, int DX, int DY>
__device__ __forceinline__ void col3_offset(const Ras3ColArgs& p, const double* pvb,
                                            const double* cl, int x, int y, double (&out)[E]) {
  constexpr int PXR = Col3<E>::PXR, PP = Col3<E>::PP;
  constexpr int R = iabs3(DX) + iabs3(DY);
  constexpr int A = 3 - R;
  const double* col = pvb + DY * PXR + DX;
  // c at this neighbour column (R == 1): c v enters Delta(c v); zero outside the extended box
  const bool cin = x + DX >= 0 && x + DX < E && y + DY >= 0 && y + DY < E;
  const double* ccol = cl + (y + DY) * E + (x + DX);
  // planes zz < 0 and zz >= E are zero (the modified BC): skipped at compile time
#pragma unroll
  for (int zz = 0; zz < E; ++zz) {
    const double val = col[zz * PP];
#pragma unroll
    for (int z = (zz - A > 0 ? zz - A : 0); z <= (zz + A < E - 1 ? zz + A : E - 1); ++z) {
      const int dz = zz - z;
      const int cls = wclass3(iabs3(DX), iabs3(DY), iabs3(dz));   // (unrolled: a constant)
      out[z] = fma(cls == 0 ? dt_w0<3>(p.dtp, p.W[0]) : p.W[cls], val, out[z]);
    }
    if constexpr (R == 1) {
      if (zz >= 0 && zz < E) {
        const double cv = cin ? ccol[zz * E * E] * val : 0.0;
        out[zz] = fma(-p.ih2, cv, out[zz]);
      }
    }
    if constexpr (R == 0) {   // z-neighbours and centre of Delta(c v) in the own column
      if (zz >= 0 && zz < E) {
        const double cz = cl[(zz * E + y) * E + x] * val;
        if (zz - 1 >= 0) out[zz - 1] = fma(-p.ih2, cz, out[zz - 1]);
        if (zz + 1 < E) out[zz + 1] = fma(-p.ih2, cz, out[zz + 1]);
        out[zz] = fma(6.0 * p.ih2, cz, out[zz]);
      }
    }
  }
}

// w = A_k v_J for the thread's column (pvb -> padded (x+3, y+3, 3)): the 25 xy offsets of
// the radius-3 diamond
template <int E>
__device__ __forceinline__ void col3_stencil(const Ras3ColArgs& p, const double* pvb,
                                             const double* cl, int x, int y, double (&out)[E]) {
#pragma unroll
  for (int z = 0; z < E; ++z) out[z] = 0.0;
#define O3(DX, DY) col3_offset<E, DX, DY>(p, pvb, cl, x, y, out);
  O3(0, -3)
  O3(-1, -2) O3(0, -2) O3(1, -2)
  O3(-2, -1) O3(-1, -1) O3(0, -1) O3(1, -1) O3(2, -1)
  O3(-3, 0) O3(-2, 0) O3(-1, 0) O3(0, 0) O3(1, 0) O3(2, 0) O3(3, 0)
  O3(-2, 1) O3(-1, 1) O3(0, 1) O3(1, 1) O3(2, 1)
  O3(-1, 2) O3(0, 2) O3(1, 2)
  O3(0, 3)
#undef O3
}

template <int K, int E, int J>
__device__ __forceinline__ bool col3_step(const Ras3ColArgs& p, double (&w)[E], const double* Vb,
                                          int nodes_stride, bool act, double* red, int& rb,
                                          double* h1, double* h2, double* hx, double* H,
                                          double* cs, double* sn, double* gv, double* pvb,
                                          double* Vnext, double beta, int nwt) {
  constexpr int PP = Col3<E>::PP;
  constexpr int NE = E * E * E;
  // basis value i at the thread's node z: v_J is also in the shared plane (bitwise the same
  // value), which saves one of the J+1 L2 reads in each of the three passes below
  auto vb = [&](int i, int z) -> double {
    return i == J ? pvb[z * PP] : Vb[(size_t)i * NE + z * nodes_stride];
  };
  // pass 1: h1 = V^T w
  {
    double acc[J + 1];
#pragma unroll
    for (int i = 0; i <= J; ++i) {
      double t = 0.0;
      if (act) {
#pragma unroll
        for (int z = 0; z < E; ++z) t = fma(vb(i, z), w[z], t);
      }
      acc[i] = t;
    }
    sized_allreduce<J + 1, NW3MAX>(acc, red + rb * NW3MAX * 16, h1, nwt);
    rb ^= 1;
  }
  // w' = w - V h1 ; pass 2: h2 = V^T w' and |w'|^2
  {
    double hv[J + 1];
#pragma unroll
    for (int i = 0; i <= J; ++i) hv[i] = h1[i];
    double acc[J + 2];
#pragma unroll
    for (int i = 0; i < J + 2; ++i) acc[i] = 0.0;
    if (act) {
#pragma unroll
      for (int z = 0; z < E; ++z) {
        double vv[J + 1];
        double ww = w[z];
#pragma unroll
        for (int i = 0; i <= J; ++i) {
          vv[i] = vb(i, z);
          ww = fma(-hv[i], vv[i], ww);
        }
#pragma unroll
        for (int i = 0; i <= J; ++i) acc[i] = fma(vv[i], ww, acc[i]);
        acc[J + 1] = fma(ww, ww, acc[J + 1]);
        w[z] = ww;
      }
    }
    sized_allreduce<J + 2, NW3MAX>(acc, red + rb * NW3MAX * 16, h2, nwt);
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
  if (act) {
#pragma unroll
    for (int z = 0; z < E; ++z) {
      double ww = w[z];
#pragma unroll
      for (int i = 0; i <= J; ++i) ww = fma(-hv[i], vb(i, z), ww);
      w[z] = ww;
    }
  }
  double hn2;
  if (h2n <= 1e-8 * wn2) {
    hn2 = wn2 - h2n;                                  // |w''|^2 = |w'|^2 - |h2|^2
  } else {
    double acc[1] = {0.0};
#pragma unroll
    for (int z = 0; z < E; ++z) acc[0] = fma(w[z], w[z], acc[0]);
    sized_allreduce<1, NW3MAX>(acc, red + rb * NW3MAX * 16, hx, nwt);
    rb ^= 1;
    hn2 = hx[0];
  }
  const double hn = sqrt(hn2 > 0.0 ? hn2 : 0.0);
  if (threadIdx.x == 0) {   // Hessenberg column J: previous rotations, a new one (oracle order)
    double col[J + 2];
#pragma unroll
    for (int i = 0; i <= J; ++i) col[i] = h1[i] + h2[i];
    col[J + 1] = hn;
#pragma unroll
    for (int i = 0; i < J; ++i) {
      const double a = col[i], b = col[i + 1];
      col[i] = cs[i] * a + sn[i] * b;
      col[i + 1] = -sn[i] * a + cs[i] * b;
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
#pragma unroll
    for (int i = 0; i <= J; ++i) H[i + (K + 1) * J] = col[i];
  }
  if (hn <= 1e-14 * beta) return true;
  if constexpr (J + 1 < K) {
    const double ihn = 1.0 / hn;
    if (act) {
#pragma unroll
      for (int z = 0; z < E; ++z) {
        const double vn = w[z] * ihn;
        Vnext[z * nodes_stride] = vn;
        pvb[z * PP] = vn;
      }
    }
  }
  return false;
}

template <int K, int E, int J>
__device__ __forceinline__ bool col3_dispatch(int j, const Ras3ColArgs& p, double (&w)[E],
                                              const double* Vb, int ns, bool act, double* red,
                                              int& rb, double* h1, double* h2, double* hx,
                                              double* H, double* cs, double* sn, double* gv,
                                              double* pvb, double* Vw, double beta, int nwt) {
  if constexpr (J < K) {
    constexpr int NE = E * E * E;
    if (j == J)
      return col3_step<K, E, J>(p, w, Vb, ns, act, red, rb, h1, h2, hx, H, cs, sn, gv, pvb,
                                Vw + (size_t)(J + 1) * NE, beta, nwt);
    return col3_dispatch<K, E, J + 1>(j, p, w, Vb, ns, act, red, rb, h1, h2, hx, H, cs, sn, gv,
                                      pvb, Vw, beta, nwt);
  } else {
    return true;
  }
}

template <int K, int E>
__global__ void __launch_bounds__((E * E + 31) / 32 * 32, 1)
    ras3d_col_kernel(const __grid_constant__ Ras3ColArgs p) {
  if (p.gate && *p.gate) return;
  constexpr int PXR = Col3<E>::PXR, PP = Col3<E>::PP, NE = E * E * E;
  extern __shared__ __align__(128) double smem_dyn[];
  double* pv = smem_dyn;                      // E planes of PY x PXR, zero x/y ring
  double* cl = pv + E * PP;                   // E^3
  double* red = cl + NE;                      // 2 x NW3MAX x 16
  double* hwall = red + 2 * NW3MAX * 16;      // NW3MAX x 48
  __shared__ double H[(K + 1) * K];
  __shared__ double gv[K + 1], cs[K], sn[K], yv[K];

  const int tid = threadIdx.x, nwt = blockDim.x >> 5;
  double* h1 = hwall + (tid >> 5) * 48;
  double* h2 = h1 + 16;
  double* hx = h2 + 16;
  const bool act = tid < E * E;
  const int x = act ? tid % E : 0, y = act ? tid / E : 0;
  double* pvb = pv + (y + 3) * PXR + (x + 3);
  double* V0 = p.basis + (size_t)blockIdx.x * K * NE;   // this CTA's basis scratch
  const double* Vb = V0 + y * E + x;                      // own column, stride E^2
  double* Vw = V0 + y * E + x;
  const int nbx = p.nx / p.bx, nby = p.ny / p.by, nbz = p.nz / p.bz;
  const int nboxes = nbx * nby * nbz;
  const size_t NX = p.nx, NXY = (size_t)p.nx * p.ny;

  for (int q = tid; q < E * PP; q += blockDim.x) pv[q] = 0.0;

  for (int box = blockIdx.x; box < nboxes; box += gridDim.x) {
    const int ibx = box % nbx, iby = (box / nbx) % nby, ibz = box / (nbx * nby);
    const int gx0 = ibx * p.bx - p.o, gy0 = iby * p.by - p.o, gz0 = ibz * p.bz - p.o;
    double w[E];
    double acc0[1] = {0.0};
    __syncthreads();                      // previous box done with pv / cl / yv
    if (act) {
      const size_t gxy = (size_t)wrapi(gx0 + x, p.nx) + NX * wrapi(gy0 + y, p.ny);
      const bool oxy = x >= p.o && x < p.o + p.bx && y >= p.o && y < p.o + p.by;
#pragma unroll
      for (int z = 0; z < E; ++z) {
        const size_t g = gxy + NXY * wrapi(gz0 + z, p.nz);
        const bool owned = oxy && z >= p.o && z < p.o + p.bz;
        w[z] = (p.restrict_owned && !owned) ? 0.0 : p.v[g];
        cl[(z * E + y) * E + x] = p.c[g];
        acc0[0] = fma(w[z], w[z], acc0[0]);
      }
    } else {
#pragma unroll
      for (int z = 0; z < E; ++z) w[z] = 0.0;
    }
    int rb = 0;
    sized_allreduce<1, NW3MAX>(acc0, red + rb * NW3MAX * 16, hx, nwt);
    rb ^= 1;
    const double beta = sqrt(hx[0]);
    if (beta == 0.0) {
      if (tid == 0) ras_count(p.jcnt, 0);
      if (act) {
#pragma unroll
        for (int z = 0; z < E; ++z) {
          const int li = x - p.o, lj = y - p.o, lk = z - p.o;
          if (p.y_ext) p.y_ext[(size_t)box * NE + (z * E + y) * E + x] = 0.0;
          else if (li >= 0 && li < p.bx && lj >= 0 && lj < p.by && lk >= 0 && lk < p.bz)
            p.z[(size_t)(ibx * p.bx + li) + NX * (iby * p.by + lj) + NXY * (ibz * p.bz + lk)] = 0.0;
        }
      }
      continue;
    }
    {
      const double ib = 1.0 / beta;
      if (act) {
#pragma unroll
        for (int z = 0; z < E; ++z) {
          const double v0 = w[z] * ib;
          Vw[z * E * E] = v0;
          pvb[z * PP] = v0;
        }
      }
    }
    if (tid == 0) gv[0] = beta;
    int jm = 0;
#pragma unroll 1
    for (int j = 0; j < K; ++j) {
      __syncthreads();                    // pv holds v_j, cl holds c
      if (act) col3_stencil<E>(p, pvb, cl, x, y, w);
      else {
#pragma unroll
        for (int z = 0; z < E; ++z) w[z] = 0.0;
      }
      const bool stop = col3_dispatch<K, E, 0>(j, p, w, Vb, E * E, act, red, rb, h1, h2, hx, H,
                                               cs, sn, gv, pvb, Vw, beta, nwt);
      jm = j + 1;
      if (stop) break;
    }
    __syncthreads();
    if (tid == 0) {   // back substitution R yv = g (R reduced column by column)
      const int ld = K + 1;
      for (int i = jm - 1; i >= 0; --i) {
        double s = gv[i];
        for (int l = i + 1; l < jm; ++l) s -= H[i + ld * l] * yv[l];
        yv[i] = s / H[i + ld * i];
      }
      ras_count(p.jcnt, jm);
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int z = 0; z < E; ++z) {
        const int li = x - p.o, lj = y - p.o, lk = z - p.o;
        const bool own = li >= 0 && li < p.bx && lj >= 0 && lj < p.by && lk >= 0 && lk < p.bz;
        if (!p.y_ext && !own) continue;
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < K; ++i)
          if (i < jm) s = fma(yv[i], Vb[(size_t)i * NE + z * E * E], s);
        if (p.y_ext) p.y_ext[(size_t)box * NE + (z * E + y) * E + x] = s;
        else p.z[(size_t)(ibx * p.bx + li) + NX * (iby * p.by + lj) + NXY * (ibz * p.bz + lk)] = s;
      }
    }
  }
}

template <int K, int E>
size_t col3_smem() {
  return ((size_t)E * Col3<E>::PP + (size_t)E * E * E + 2 * NW3MAX * 16 + NW3MAX * 48) *
         sizeof(double);
}

typedef void (*ras3col_fn)(const Ras3ColArgs);

ras3col_fn pick3(int k, int e, size_t* smem) {
#define C3(K, E)                                             \
  if (k == K && e == E) {                                    \
    *smem = col3_smem<K, E>();                               \
    return ras3d_col_kernel<K, E>;                           \
  }
  C3(4, 12) C3(10, 12) C3(4, 20) C3(10, 20)
#undef C3
  return nullptr;
}

}  // namespace

// 1 if the on-chip 3D kernel handles this configuration (cubic extended box, instantiated K, E)
int ras3d_col_plan(pfc_ctx* ctx, size_t* scratch_doubles, int* grid) {
  const pfc_config& c = ctx->cfg;
  const int e = c.ras_box[0] + 2 * c.ras_overlap;
  if (c.ras_box[1] != c.ras_box[0] || c.ras_box[2] != c.ras_box[0]) return 0;
  size_t smem = 0;
  if (!pick3(c.ras_local_k, e, &smem)) return 0;
  const int nboxes = (c.n[0] / c.ras_box[0]) * (c.n[1] / c.ras_box[1]) * (c.n[2] / c.ras_box[2]);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  *grid = nboxes < sms ? nboxes : sms;
  *scratch_doubles = (size_t)(*grid) * c.ras_local_k * e * e * e;
  return 1;
}

cudaError_t launch_ras_3d_col(pfc_ctx* ctx, const double* v, const double* c, double dt,
                              double* z, double* scratch) {
  const pfc_config& cf = ctx->cfg;
  const int e = cf.ras_box[0] + 2 * cf.ras_overlap;
  size_t smem = 0;
  ras3col_fn fn = pick3(cf.ras_local_k, e, &smem);
  if (!fn) return cudaErrorInvalidValue;
  cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
  if (err != cudaSuccess) return err;
  size_t sd = 0;
  int grid = 0;
  ras3d_col_plan(ctx, &sd, &grid);
  Ras3ColArgs p{};
  p.v = v; p.c = c; p.z = z; p.basis = scratch;
  p.nx = cf.n[0]; p.ny = cf.n[1]; p.nz = cf.n[2];
  p.bx = cf.ras_box[0]; p.by = cf.ras_box[1]; p.bz = cf.ras_box[2]; p.o = cf.ras_overlap;
  p.restrict_owned = cf.ras_variant == PFC_RAS_RIGHT;
  p.y_ext = cf.ras_variant == PFC_RAS_LEFT ? nullptr : ctx->ras_y;
  p.gate = ctx->gate;
  p.jcnt = ctx->prof ? ctx->d_jcnt : nullptr;
  // class weights of v/dt - alpha Delta v - Delta^2 v - Delta^3 v / 2 with h^2 Delta = L:
  // L (000) -6, (001) 1;  L^2 (000) 42, (001) -12, (002) 1, (011) 2;
  // L^3 (000) -324, (001) 123, (002) -18, (011) -36, (003) 1, (012) 3, (111) 6
  const double ih2 = ctx->ih2, ih4 = ih2 * ih2, ih6 = ih4 * ih2;
  const double al = 0.5 * (1.0 - cf.gamma);
  p.W[0] = 1.0 / dt + 6.0 * al * ih2 - 42.0 * ih4 + 162.0 * ih6;
  p.dtp = ctx->dtdev;
  p.W[1] = -al * ih2 + 12.0 * ih4 - 61.5 * ih6;
  p.W[2] = -ih4 + 9.0 * ih6;
  p.W[3] = -2.0 * ih4 + 18.0 * ih6;
  p.W[4] = -0.5 * ih6;
  p.W[5] = -1.5 * ih6;
  p.W[6] = -3.0 * ih6;
  p.ih2 = ih2;
  const int threads = (e * e + 31) / 32 * 32;
  fn<<<grid, threads, smem, ctx->stream>>>(p);
  ctx->launches++;
  {
    const double nb = (double)(cf.n[0] / cf.ras_box[0]) * (cf.n[1] / cf.ras_box[1]) *
                      (cf.n[2] / cf.ras_box[2]);
    const double next = nb * e * e * e;
    const double nout = cf.ras_variant == PFC_RAS_LEFT ? (double)ctx->N : next;
    pfc_account(ctx, PFC_K_RAS, 8.0 * (2.0 * next + nout), 0.0);
    ras_flop_model(ctx, (double)e * e * e, 31.0, nout / nb);   // flops from the step counters
  }
  cudaError_t e2 = cudaGetLastError();
  if (e2 != cudaSuccess || cf.ras_variant == PFC_RAS_LEFT) return e2;
  return launch_ras_extend(ctx, z);
}
