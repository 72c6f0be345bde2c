// stencil3d.cu -- fused 3D DVD residual (K1) and Jacobian-vector product (K2), sm_100a.
//
// Same operators as stencil2d.cu (Eq. NSOP, Eq. discretedG, Eq. Jacobi
// P:351-356), the 7-point Delta_d composed three times: a radius-3, 63-point stencil:
//   resid: u = (Phi+psi)/2,  L1 = Delta u,  A = (1-gamma)u + 2 L1 + Delta L1 + N(Phi,psi),
//          F = (Phi-psi)/dt - Delta A
//   jv:    L1 = Delta v,  B = ((1-gamma)/2 + c) v + L1 + Delta L1 / 2,  Jv = v/dt - Delta B
//
// 2.5D z-march.  A CTA (one per SM) owns a TX x TY = 32 x 32 column of outputs and a chunk of
// ZC z-planes.  Input planes z0-3 .. z0+ZC+2 stream through a RING-slot ring per field filled
// by TMA (cp.async.bulk.tensor.3d, one 40 x 38 x 1 box per field and plane, PREFETCH planes in
// flight, one mbarrier per slot).  Each thread owns a fixed 2 x 2 block (two x-adjacent
// columns, two rows) of the 40 x 38 plane window for all stages.  At streamed plane t it computes
//     L1(t-1) [halo 2]  ->  A(t-2) [halo 1]  ->  F(t-3) [halo 0]
// z-neighbours, block-internal neighbours and centres come from registers; only the block's
// outside neighbours are read from shared memory (two 16-byte and four 8-byte loads per stage:
// about 96 B of shared-memory traffic per point and stage pipeline).  Every stage of
// iteration t reads planes written in iteration t-1, so one barrier per plane suffices.  Points
// of a block outside a stage region are computed too; such values are never consumed by an
// in-region point (each region is the previous one shrunk by one).  Periodic x/y wrap: TMA
// zero-fills out-of-range cells and edge tiles reload exactly those cells with wrapped loads;
// z wraps incrementally.  Optional fused ||F||^2 partial per CTA.
#include "pfc_device.cuh"
#include "pfc_internal.h"

namespace {

constexpr int TX = 32, TY = 32;
constexpr int HX = 4, HY = 3;
constexpr int WX = TX + 2 * HX;   // 40
constexpr int WY = TY + 2 * HY;   // 38
constexpr int WN = WX * WY;       // 1520
constexpr int NPC = WX / 2;       // pair columns (20)
constexpr int NST = WY / 2;       // two-row strips (19)
constexpr int NBLK = NPC * NST;   // 380 blocks
constexpr int NT = 384;           // 12 warps: 3 per SM sub-partition -> up to 168 registers
constexpr int RING = 6;
constexpr int PREFETCH = 3;

enum { OP_RESID = 0, OP_JV = 1 };

struct S3Args {
  const double* a;   // Phi | v
  const double* b;   // psi | c
  double* out;
  double* partials;
  int nx, ny, nz;
  int zc;            // planes per chunk
  double idt, gamma, ih2;
  int use_tma;
  const int* gate;   // device-resident FGMRES: skip the launch when *gate != 0 (f1)
};

struct d2 { double x, y; };
struct blk { d2 r0, r1; };      // rows 0 and 1 of a 2 x 2 block (columns x, x+1)

__device__ __forceinline__ d2 ld2(const double* p) {
  const double2 v = *reinterpret_cast<const double2*>(p);
  return {v.x, v.y};
}
__device__ __forceinline__ void st2(double* p, d2 v) {
  *reinterpret_cast<double2*>(p) = make_double2(v.x, v.y);
}

// window indices of a block's outside neighbours: the single left/right element of both rows
// and the pair above row 0 / below row 1 (clamped inside the window at its edge)
struct nbr_idx { int l0, r0, l1, r1, t, d; };

// Sum of the OUTSIDE neighbours of each point of the block in plane f (5-point xy stencil).
__device__ __forceinline__ blk outside_sum(const double* f, const nbr_idx& n) {
  const double L0 = f[n.l0], R0 = f[n.r0], L1 = f[n.l1], R1 = f[n.r1];
  const d2 T = ld2(f + n.t), D = ld2(f + n.d);
  return {{L0 + T.x, R0 + T.y}, {L1 + D.x, R1 + D.y}};
}

// ih2 * (outside sum + in-block neighbours - 4 centre + z-part); zc = centre plane values
__device__ __forceinline__ blk lap3(const blk& out, const blk& zm, const blk& zc, const blk& zp,
                                    double ih2) {
  blk o;
  o.r0.x = ih2 * ((out.r0.x + zc.r0.y + zc.r1.x - 4.0 * zc.r0.x) + (zm.r0.x + zp.r0.x - 2.0 * zc.r0.x));
  o.r0.y = ih2 * ((out.r0.y + zc.r0.x + zc.r1.y - 4.0 * zc.r0.y) + (zm.r0.y + zp.r0.y - 2.0 * zc.r0.y));
  o.r1.x = ih2 * ((out.r1.x + zc.r1.y + zc.r0.x - 4.0 * zc.r1.x) + (zm.r1.x + zp.r1.x - 2.0 * zc.r1.x));
  o.r1.y = ih2 * ((out.r1.y + zc.r1.x + zc.r0.y - 4.0 * zc.r1.y) + (zm.r1.y + zp.r1.y - 2.0 * zc.r1.y));
  return o;
}

__device__ __forceinline__ double cubic(double a, double b) {
  return 0.25 * (a * a * a + a * a * b + a * b * b + b * b * b);
}

template <int OP>
__global__ void __launch_bounds__(NT, 1) stencil3d_kernel(const __grid_constant__ CUtensorMap ma,
                                                          const __grid_constant__ CUtensorMap mb,
                                                          S3Args p) {
  extern __shared__ __align__(128) double smem_dyn[];   // LDS/STS addressing, 128-B aligned
  double* ringA = smem_dyn;                // RING planes
  double* ringB = ringA + RING * WN;       // RING planes
  double* L1b = ringB + RING * WN;         // 2 planes
  double* AAb = L1b + 2 * WN;              // 2 planes
  __shared__ uint64_t bars[RING];
  __shared__ double red[64];

  if (p.gate && *p.gate) return;
  const int tid = threadIdx.x;
  const int ntx = (p.nx + TX - 1) / TX;
  const int x0 = (blockIdx.x % ntx) * TX, y0 = (blockIdx.x / ntx) * TY;
  const int z0 = blockIdx.y * p.zc;
  const int zc = min(p.zc, p.nz - z0);
  const int gx0 = x0 - HX, gy0 = y0 - HY;
  const int nx = p.nx, ny = p.ny, nz = p.nz;
  const size_t plane = (size_t)nx * ny;
  const int T = zc + 6;                    // planes streamed
  const bool edge = gx0 < 0 || gy0 < 0 || gx0 + WX > nx || gy0 + WY > ny;
  const double ih2 = p.ih2;

  // this thread's 2 x 2 block: columns qx, qx+1; rows qy, qy+1
  const bool valid = tid < NBLK;
  const int bi = valid ? tid : 0;
  const int qx = 2 * (bi % NPC), qy = 2 * (bi / NPC);
  const int qa = qy * WX + qx, qb = qa + WX;
  nbr_idx nb;
  nb.l0 = qx >= 1 ? qa - 1 : qa;
  nb.r0 = qx + 2 < WX ? qa + 2 : qa + 1;
  nb.l1 = nb.l0 + WX;
  nb.r1 = nb.r0 + WX;
  nb.t = qy >= 1 ? qa - WX : qa;
  nb.d = qy + 2 < WY ? qb + WX : qb;
  auto in_rows = [&](int row, int r) { return row >= HY - r && row < HY + TY + r; };
  auto in_cols = [&](int r) { return qx + 1 >= HX - r && qx < HX + TX + r; };
  const bool w2a = valid && in_cols(2) && in_rows(qy, 2), w2b = valid && in_cols(2) && in_rows(qy + 1, 2);
  const bool w1a = valid && in_cols(1) && in_rows(qy, 1), w1b = valid && in_cols(1) && in_rows(qy + 1, 1);
  const int gx = gx0 + qx, gya = gy0 + qy, gyb = gya + 1;
  auto col0 = [&](int c) { return c >= HX && c < HX + TX; };
  // output flags per point (in region 0 and inside a ragged grid)
  const bool o_a0 = valid && in_rows(qy, 0) && col0(qx) && gx < nx && gya < ny;
  const bool o_a1 = valid && in_rows(qy, 0) && col0(qx + 1) && gx + 1 < nx && gya < ny;
  const bool o_b0 = valid && in_rows(qy + 1, 0) && col0(qx) && gx < nx && gyb < ny;
  const bool o_b1 = valid && in_rows(qy + 1, 0) && col0(qx + 1) && gx + 1 < nx && gyb < ny;
  auto oob = [&](int x, int y) { return x < 0 || x >= nx || y < 0 || y >= ny; };
  const bool ob0 = oob(gx, gya), ob1 = oob(gx + 1, gya), ob2 = oob(gx, gyb), ob3 = oob(gx + 1, gyb);
  const bool reload = valid && (!p.use_tma || (edge && (ob0 || ob1 || ob2 || ob3)));
  const size_t g0 = (size_t)wrapi(gx, nx) + (size_t)nx * wrapi(gya, ny);
  const size_t g1 = (size_t)wrapi(gx + 1, nx) + (size_t)nx * wrapi(gya, ny);
  const size_t g2 = (size_t)wrapi(gx, nx) + (size_t)nx * wrapi(gyb, ny);
  const size_t g3 = (size_t)wrapi(gx + 1, nx) + (size_t)nx * wrapi(gyb, ny);
  // 16-B pair stores need an aligned first plane and an even plane stride (nx even)
  const bool vec_a = o_a0 && o_a1 && (nx % 2 == 0) && ((reinterpret_cast<uintptr_t>(p.out + g0) & 15u) == 0);
  const bool vec_b = o_b0 && o_b1 && (nx % 2 == 0) && ((reinterpret_cast<uintptr_t>(p.out + g2) & 15u) == 0);

  const int zfirst = wrapi(z0 - 3, nz);
  if (p.use_tma) {
    if (tid == 0) {
      for (int i = 0; i < RING; ++i) mbar_init(&bars[i], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
      int zi = zfirst;
      for (int t = 0; t < PREFETCH && t < T; ++t) {
        mbar_expect_tx(&bars[t], 2u * WN * sizeof(double));
        tma_load_3d(ringA + t * WN, &ma, &bars[t], gx0, gy0, zi);
        tma_load_3d(ringB + t * WN, &mb, &bars[t], gx0, gy0, zi);
        zi = (zi + 1 == nz) ? 0 : zi + 1;
      }
    }
  }
  int zpre = wrapi(z0 - 3 + PREFETCH, nz);   // plane of the next TMA issue
  int zcur = zfirst;                          // plane t
  int slot = 0, pslot = PREFETCH % RING;
  uint32_t phase = 0;

  const blk Z{{0, 0}, {0, 0}};
  // register queues, all of length 3 so that the 3x-unrolled loop rotates them by renaming.
  // At the start of iteration t:  a = v | Phi-psi at t-3, t-2, t-1;  c = c | N at t-3, t-2, t-1;
  // u at t-3, t-2, t-1 (resid);  l = L1 at t-4, t-3, t-2;  A at t-5, t-4, t-3.
  blk a0 = Z, a1 = Z, a2 = Z, c0 = Z, c1 = Z, c2 = Z, u0 = Z, u1 = Z, u2 = Z;
  blk l0 = Z, l1 = Z, l2 = Z, A0 = Z, A1 = Z, A2 = Z;
  double nrm = 0.0;
  const size_t zoff0 = plane * (size_t)z0;
  const int Tp = (T + 2) / 3 * 3;          // padded to the unroll factor; extra planes are inert

#pragma unroll 3
  for (int t = 0; t < Tp; ++t) {
    double* pa = ringA + slot * WN;
    double* pb = ringB + slot * WN;
    if (p.use_tma) {
      if (tid == 0 && t + PREFETCH < Tp) {
        mbar_expect_tx(&bars[pslot], 2u * WN * sizeof(double));
        tma_load_3d(ringA + pslot * WN, &ma, &bars[pslot], gx0, gy0, zpre);
        tma_load_3d(ringB + pslot * WN, &mb, &bars[pslot], gx0, gy0, zpre);
      }
      zpre = (zpre + 1 == nz) ? 0 : zpre + 1;
      mbar_wait(&bars[slot], phase);
    }
    // ---- own inputs of plane t
    blk va, vb;
    va.r0 = ld2(pa + qa); va.r1 = ld2(pa + qb);
    vb.r0 = ld2(pb + qa); vb.r1 = ld2(pb + qb);
    if (reload) {
      const size_t zo = plane * zcur;
      const bool all = !p.use_tma;
      if (all || ob0) { va.r0.x = p.a[g0 + zo]; vb.r0.x = p.b[g0 + zo]; }
      if (all || ob1) { va.r0.y = p.a[g1 + zo]; vb.r0.y = p.b[g1 + zo]; }
      if (all || ob2) { va.r1.x = p.a[g2 + zo]; vb.r1.x = p.b[g2 + zo]; }
      if (all || ob3) { va.r1.y = p.a[g3 + zo]; vb.r1.y = p.b[g3 + zo]; }
      st2(pa + qa, va.r0); st2(pa + qb, va.r1);
      st2(pb + qa, vb.r0); st2(pb + qb, vb.r1);
      if (p.use_tma) fence_proxy_async();   // generic write before a later TMA overwrite
    }
    zcur = (zcur + 1 == nz) ? 0 : zcur + 1;
    const int prv = slot == 0 ? RING - 1 : slot - 1;           // ring slot of plane t-1
    // ---- outside neighbours of the planes produced in iteration t-1 (loads before any store)
    blk x1;
    if (OP == OP_RESID) {   // u(t-1) = (Phi + psi)/2 from both rings
      const blk xa = outside_sum(ringA + prv * WN, nb), xb = outside_sum(ringB + prv * WN, nb);
      x1 = {{0.5 * (xa.r0.x + xb.r0.x), 0.5 * (xa.r0.y + xb.r0.y)},
            {0.5 * (xa.r1.x + xb.r1.x), 0.5 * (xa.r1.y + xb.r1.y)}};
    } else {
      x1 = outside_sum(ringA + prv * WN, nb);
    }
    const blk x2 = outside_sum(L1b + ((t - 2) & 1) * WN, nb);
    const blk x3 = outside_sum(AAb + ((t - 3) & 1) * WN, nb);
    // ---- compute (garbage of the warm-up iterations never reaches a stored output)
    blk anew, cnew, ufresh;          // plane-t values entering the queues
    if (OP == OP_RESID) {
      anew = {{va.r0.x - vb.r0.x, va.r0.y - vb.r0.y}, {va.r1.x - vb.r1.x, va.r1.y - vb.r1.y}};
      cnew = {{cubic(va.r0.x, vb.r0.x), cubic(va.r0.y, vb.r0.y)},
              {cubic(va.r1.x, vb.r1.x), cubic(va.r1.y, vb.r1.y)}};
      ufresh = {{0.5 * (va.r0.x + vb.r0.x), 0.5 * (va.r0.y + vb.r0.y)},
                {0.5 * (va.r1.x + vb.r1.x), 0.5 * (va.r1.y + vb.r1.y)}};
    } else {
      anew = va;                      // v
      cnew = vb;                      // c
      ufresh = va;
    }
    const blk& um = (OP == OP_RESID) ? u1 : a1;   // u | v at t-2
    const blk& uc = (OP == OP_RESID) ? u2 : a2;   // u | v at t-1
    // L1(t-1) on halo 2
    const blk lnew = lap3(x1, um, uc, ufresh, ih2);
    // A(t-2) | bracket(t-2) on halo 1
    blk Anew;
    {
      const blk lapL = lap3(x2, l1, l2, lnew, ih2);
      if (OP == OP_RESID) {
        const double gm = 1.0 - p.gamma;
        Anew.r0.x = gm * u1.r0.x + 2.0 * l2.r0.x + lapL.r0.x + c1.r0.x;
        Anew.r0.y = gm * u1.r0.y + 2.0 * l2.r0.y + lapL.r0.y + c1.r0.y;
        Anew.r1.x = gm * u1.r1.x + 2.0 * l2.r1.x + lapL.r1.x + c1.r1.x;
        Anew.r1.y = gm * u1.r1.y + 2.0 * l2.r1.y + lapL.r1.y + c1.r1.y;
      } else {
        const double al = 0.5 * (1.0 - p.gamma);
        Anew.r0.x = (al + c1.r0.x) * a1.r0.x + l2.r0.x + 0.5 * lapL.r0.x;
        Anew.r0.y = (al + c1.r0.y) * a1.r0.y + l2.r0.y + 0.5 * lapL.r0.y;
        Anew.r1.x = (al + c1.r1.x) * a1.r1.x + l2.r1.x + 0.5 * lapL.r1.x;
        Anew.r1.y = (al + c1.r1.y) * a1.r1.y + l2.r1.y + 0.5 * lapL.r1.y;
      }
    }
    // F(t-3) on halo 0: (Phi-psi)/dt | v/dt  minus  Delta A
    const blk lapA = lap3(x3, A1, A2, Anew, ih2);
    const d2 oa = {a0.r0.x * p.idt - lapA.r0.x, a0.r0.y * p.idt - lapA.r0.y};
    const d2 obv = {a0.r1.x * p.idt - lapA.r1.x, a0.r1.y * p.idt - lapA.r1.y};
    // ---- queue rotation (renames under the 3x unroll)
    a0 = a1; a1 = a2; a2 = anew;
    c0 = c1; c1 = c2; c2 = cnew;
    if (OP == OP_RESID) { u0 = u1; u1 = u2; u2 = ufresh; }
    l0 = l1; l1 = l2; l2 = lnew;
    A0 = A1; A1 = A2; A2 = Anew;
    // ---- stores
    double* Lw = L1b + ((t - 1) & 1) * WN;
    double* Aw = AAb + ((t - 2) & 1) * WN;
    if (w2a) st2(Lw + qa, lnew.r0);
    if (w2b) st2(Lw + qb, lnew.r1);
    if (w1a) st2(Aw + qa, Anew.r0);
    if (w1b) st2(Aw + qb, Anew.r1);
    if (t >= 6 && t - 6 < zc) {
      const size_t zo = zoff0 + plane * (size_t)(t - 6);
      if (vec_a) {
        st2(p.out + g0 + zo, oa);
        nrm += oa.x * oa.x + oa.y * oa.y;
      } else {
        if (o_a0) { p.out[g0 + zo] = oa.x; nrm += oa.x * oa.x; }
        if (o_a1) { p.out[g1 + zo] = oa.y; nrm += oa.y * oa.y; }
      }
      if (vec_b) {
        st2(p.out + g2 + zo, obv);
        nrm += obv.x * obv.x + obv.y * obv.y;
      } else {
        if (o_b0) { p.out[g2 + zo] = obv.x; nrm += obv.x * obv.x; }
        if (o_b1) { p.out[g3 + zo] = obv.y; nrm += obv.y * obv.y; }
      }
    }
    slot = slot + 1 == RING ? 0 : slot + 1;
    pslot = pslot + 1 == RING ? 0 : pslot + 1;
    phase ^= (slot == 0) ? 1u : 0u;
    __syncthreads();
  }
  if (p.partials) {
    double sblk = block_sum(nrm, red);
    if (tid == 0) p.partials[blockIdx.y * gridDim.x + blockIdx.x] = sblk;
  }
}

constexpr int SMEM_BYTES = (2 * RING + 4) * WN * (int)sizeof(double);

template <int OP>
cudaError_t launch3d(pfc_ctx* ctx, const double* a, const double* b, double dt, double* out,
                     double* partials, int* nparts) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(stencil3d_kernel<OP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int nx = ctx->cfg.n[0], ny = ctx->cfg.n[1], nz = ctx->cfg.n[2];
  const int ntiles = ((nx + TX - 1) / TX) * ((ny + TY - 1) / TY);
  // z chunk: about 4 waves of 148 CTAs, 8..64 planes per chunk
  int want = (ntiles * nz) / (148 * 4);
  int zc = want < 8 ? 8 : (want > 64 ? 64 : want);
  if (zc > nz) zc = nz;
  const int nzc = (nz + zc - 1) / zc;
  S3Args p{a, b, out, partials, nx, ny, nz, zc, 1.0 / dt, ctx->cfg.gamma, ctx->ih2, 0,
           OP == OP_JV ? ctx->gate : nullptr};
  CUtensorMap ma, mb;
  memset(&ma, 0, sizeof(ma));
  memset(&mb, 0, sizeof(mb));
  const int box[3] = {WX, WY, 1};
  if (nx % 2 == 0 && nx >= WX && ny >= WY && tma_usable(a) && tma_usable(b) &&
      tma_encode(&ma, a, 3, ctx->cfg.n, box) && tma_encode(&mb, b, 3, ctx->cfg.n, box))
    p.use_tma = 1;
  dim3 grid(ntiles, nzc);
  if (nparts) *nparts = grid.x * grid.y;
  stencil3d_kernel<OP><<<grid, NT, SMEM_BYTES, ctx->stream>>>(ma, mb, p);
  ctx->launches++;
  pfc_account(ctx, OP == OP_RESID ? PFC_K_RESIDUAL : PFC_K_JV, 24.0 * ctx->N,
              (OP == OP_RESID ? 42.0 : 31.0) * ctx->N);
  return cudaGetLastError();
}

}  // namespace

int stencil3d_tiles(int nx, int ny) { return ((nx + TX - 1) / TX) * ((ny + TY - 1) / TY); }

cudaError_t launch_residual_3d(pfc_ctx* ctx, const double* phi_new, const double* phi_old,
                               double dt, double* F, double* partials, int* nparts) {
  return launch3d<OP_RESID>(ctx, phi_new, phi_old, dt, F, partials, nparts);
}

cudaError_t launch_jv_3d(pfc_ctx* ctx, const double* v, const double* c, double dt,
                         double* out) {
  return launch3d<OP_JV>(ctx, v, c, dt, out, nullptr, nullptr);
}
