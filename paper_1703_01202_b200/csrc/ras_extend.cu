// ras_extend.cu -- the extension (R_k^delta)^T of classical AS (Eq. invM) and
// right-RAS (Eq. eq:ash): z = sum_k (R_k^delta)^T y_k, an overlap-add of the
// ext-box solutions y_k written by the subdomain-solve kernels to ctx->ras_y.
//
// Written as a GATHER so it is deterministic without atomics: each node sums, in a fixed
// order (box offsets -1, 0, +1 per axis, z then y then x), the y_k of the at most 3^d boxes
// whose extended box covers it.  Overlap o < box edge b (pfc_create) means only the owner box
// and its neighbours can cover a node; with two boxes on an axis the -1 and +1 neighbour are
// the same box and are visited once.
#include "pfc_device.cuh"
#include "pfc_internal.h"

namespace {

constexpr int NT = 256;

struct ExtArgs {
  const double* y;    // [box][ext node], ext node x-fastest on Ex x Ey x Ez
  double* z;
  int n[3], b[3], nb[3], E[3], o;
  int nd;
  int mirror;        // mirror BCs (R23): boxes never wrap, ext-box nodes outside the domain
  const int* gate;   // device-resident FGMRES: skip the launch when *gate != 0 (f1)
};

// candidate boxes along one axis covering coordinate x: unique indices, local coordinates
__device__ __forceinline__ int axis_candidates(int x, int n, int b, int nb, int E, int o,
                                               int mirror, int (&box)[3], int (&loc)[3]) {
  const int own = x / b;
  int cnt = 0;
#pragma unroll
  for (int d = -1; d <= 1; ++d) {
    if (mirror && (own + d < 0 || own + d >= nb)) continue;   // clipped subdomains: no wrap
    const int c = wrapi(own + d, nb);
    bool dup = false;
    for (int i = 0; i < cnt; ++i) dup = dup || box[i] == c;
    if (dup) continue;
    const int l = mirror ? x - (c * b - o) : wrapi(x - (c * b - o), n);   // local coordinate
    if (l >= 0 && l < E) {
      box[cnt] = c;
      loc[cnt] = l;
      ++cnt;
    }
  }
  return cnt;
}

__global__ void __launch_bounds__(NT) k_ras_extend(const ExtArgs p) {
  if (p.gate && *p.gate) return;
  const size_t N = (size_t)p.n[0] * p.n[1] * p.n[2];
  const size_t next = (size_t)p.E[0] * p.E[1] * p.E[2];
  for (size_t q = blockIdx.x * (size_t)NT + threadIdx.x; q < N; q += (size_t)gridDim.x * NT) {
    const int x = (int)(q % p.n[0]);
    const int y = (int)((q / p.n[0]) % p.n[1]);
    const int zz = (int)(q / ((size_t)p.n[0] * p.n[1]));
    int bx[3], lx[3], by[3], ly[3], bz[3], lz[3];
    const int cx = axis_candidates(x, p.n[0], p.b[0], p.nb[0], p.E[0], p.o, p.mirror, bx, lx);
    const int cy = axis_candidates(y, p.n[1], p.b[1], p.nb[1], p.E[1], p.o, p.mirror, by, ly);
    int cz = 1;
    bz[0] = 0; lz[0] = 0;
    if (p.nd == 3)
      cz = axis_candidates(zz, p.n[2], p.b[2], p.nb[2], p.E[2], p.o, p.mirror, bz, lz);
    double s = 0.0;
    for (int k = 0; k < cz; ++k)
      for (int j = 0; j < cy; ++j)
        for (int i = 0; i < cx; ++i) {
          const size_t box = (size_t)bx[i] + (size_t)p.nb[0] * (by[j] + (size_t)p.nb[1] * bz[k]);
          const size_t l = (size_t)lx[i] + (size_t)p.E[0] * (ly[j] + (size_t)p.E[1] * lz[k]);
          s += p.y[box * next + l];
        }
    p.z[q] = s;
  }
}

}  // namespace

cudaError_t launch_ras_extend(pfc_ctx* ctx, double* z) {
  const pfc_config& c = ctx->cfg;
  ExtArgs p{};
  p.y = ctx->ras_y;
  p.z = z;
  p.nd = c.ndim;
  p.o = c.ras_overlap;
  p.mirror = c.bc == PFC_BC_MIRROR;
  p.gate = ctx->gate;
  for (int d = 0; d < 3; ++d) {
    const bool act = d < c.ndim;
    p.n[d] = c.n[d];
    p.b[d] = act ? c.ras_box[d] : 1;
    p.nb[d] = act ? c.n[d] / c.ras_box[d] : 1;
    p.E[d] = act ? c.ras_box[d] + 2 * c.ras_overlap : 1;
  }
  size_t blocks = (ctx->N + NT - 1) / NT;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_ras_extend<<<(int)blocks, NT, 0, ctx->stream>>>(p);
  ctx->launches++;
  double e = 1.0;
  for (int d = 0; d < c.ndim; ++d) e *= (double)p.E[d] / p.b[d];
  pfc_account(ctx, PFC_K_RAS, 8.0 * (e + 1.0) * ctx->N, e * ctx->N);
  return cudaGetLastError();
}

size_t ras_ext_doubles(const pfc_ctx* ctx) {
  const pfc_config& c = ctx->cfg;
  size_t nb = 1, ne = 1;
  for (int d = 0; d < c.ndim; ++d) {
    nb *= (size_t)(c.n[d] / c.ras_box[d]);
    ne *= (size_t)(c.ras_box[d] + 2 * c.ras_overlap);
  }
  return nb * ne;
}
