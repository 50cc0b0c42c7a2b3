// 2D fine-level kernels (batched): matrix-free Q1 operator apply, fused
// damped-Jacobi pre-smoothing + residual restriction, fused prolongation +
// correction + post-smoothing (+ A_0 apply of the result), coarse stencil.
//
// Operator (Eq. sys_matrix; 2D stencils PAPER.md:124-129):
//   A(k,eps) = K - M(k,eps) - i B(k),  element-constant lambda_e = k_e^2 + i eps_e
//   (reading C1), boundary edges weighted by the adjacent element's k_e (C3).
// Per element e with the node at one corner and its element neighbours
// xh (along x), xv (along y), xd (diagonal):
//   K^e row  = 2/3 xp - 1/6 (xh + xv) - 1/3 xd
//   M^e row  = h^2/36 (4 xp + 2 (xh + xv) + xd)
//   B^f row  = h/6 (2 xp + x_other)                 (boundary edge f)
// Interior nodes use the assembled 9-point form: K = (1/3)[-1 -1 -1; -1 8 -1; -1 -1 -1]
// plus sum_q lambda_q M^{e_q} (constant k: the printed mass stencil).
// Jacobi: u <- u + omega D^{-1} (f - A_eps u), D = diag(A_eps) incl. -i k B
// (reading C6).  Transfers: I^T with weights
// 1, 1/2, 1/4 (reading C5) and bilinear I.
//
// B200 design: one CTA computes a TX x TY tile of fine nodes of one sample
// (blockIdx.z); every input of the multi-step sequence is staged once in
// shared memory with a halo of R = nu + 1 nodes, and every intermediate Jacobi
// iterate lives in shared memory (halo recompute / temporal blocking), so a
// whole V-cycle reads each fine input once and writes each output once.
#include "hh_internal.cuh"

namespace {

#ifndef FINE_CONST_MINB
#define FINE_CONST_MINB 4   // CTAs per SM the constant-k smoothers are compiled for
#endif
#ifndef FINE_DI_GLOBAL
#define FINE_DI_GLOBAL 0   // 1: heterogeneous D^{-1} read through L1 instead of staged in smem (measured: no gain)
#endif
#ifndef FINE_TX
#define FINE_TX 32
#endif
#ifndef FINE_TY
#define FINE_TY 16
#endif
constexpr int TX = FINE_TX;   // tile width  (fine nodes along x, even)
constexpr int TY = FINE_TY;   // tile height (even)
static_assert((TX / 2) * (TY / 2) <= 256, "the restriction takes one coarse node per thread");
constexpr int NT = 256;  // threads per CTA

struct Tile {
  int X0, Y0, R, SX, SY;
  __device__ __forceinline__ int gx(int sx) const { return X0 - R + sx; }
  __device__ __forceinline__ int gy(int sy) const { return Y0 - R + sy; }
};

// element coefficient (k, eps): the smem copy covers (SX+1) x (SY+1) elements
// starting at (X0-R-1, Y0-R-1) so the diagonal of every region node is available.
template <bool HET>
__device__ __forceinline__ double2 elem_coef(const double2* sE, const Tile& t, int ex, int ey,
                                             double2 kc) {
  if (HET) return sE[(ex - (t.X0 - t.R - 1)) + (ey - (t.Y0 - t.R - 1)) * (t.SX + 1)];
  return kc;
}

// generic (boundary-safe) row of A x at smem slot si: quadrant loop + boundary edges
template <bool HET, bool EPS>
__device__ __noinline__ cplx node_op_generic(const cplx* __restrict__ X, int si, const Tile& t,
                                             int gx, int gy, int n, double h, const double2* sE,
                                             double2 kc) {
  const int SX = t.SX;
  const double h2 = h * h * (1.0 / 36.0);
  const cplx xp = X[si];
  cplx ax = cmake(0, 0);
  for (int q = 0; q < 4; ++q) {
    const int dx = (q & 1) ? 1 : -1, dy = (q & 2) ? 1 : -1;
    const int ex = gx + (dx < 0 ? -1 : 0), ey = gy + (dy < 0 ? -1 : 0);
    if (ex < 0 || ex >= n || ey < 0 || ey >= n) continue;
    const cplx xh = X[si + dx], xv = X[si + dy * SX], xd = X[si + dx + dy * SX];
    const cplx hv = cadd(xh, xv);
    const cplx kp = cmake((2.0 / 3.0) * xp.x - (1.0 / 6.0) * hv.x - (1.0 / 3.0) * xd.x,
                          (2.0 / 3.0) * xp.y - (1.0 / 6.0) * hv.y - (1.0 / 3.0) * xd.y);
    const cplx mp = cmake(h2 * (4.0 * xp.x + 2.0 * hv.x + xd.x), h2 * (4.0 * xp.y + 2.0 * hv.y + xd.y));
    const double2 c = elem_coef<HET>(sE, t, ex, ey, kc);
    const cplx lam = cmake(c.x * c.x, EPS ? c.y : 0.0);
    ax = cadd(ax, kp);
    cfms(ax, lam, mp);
  }
  const double h6 = h * (1.0 / 6.0);
  auto edge = [&](int ex, int ey, cplx xo) {
    const double k = elem_coef<HET>(sE, t, ex, ey, kc).x;
    const cplx s = cmake(2.0 * xp.x + xo.x, 2.0 * xp.y + xo.y);
    ax.x += k * h6 * s.y;      // -i k h/6 s
    ax.y -= k * h6 * s.x;
  };
  if (gx == 0 || gx == n) {
    const int ex = (gx == 0) ? 0 : n - 1;
    if (gy > 0) edge(ex, gy - 1, X[si - SX]);
    if (gy < n) edge(ex, gy, X[si + SX]);
  }
  if (gy == 0 || gy == n) {
    const int ey = (gy == 0) ? 0 : n - 1;
    if (gx > 0) edge(gx - 1, ey, X[si - 1]);
    if (gx < n) edge(gx, ey, X[si + 1]);
  }
  return ax;
}

// Per-sample constant-coefficient interior stencil  A = c0 xp + c1 (E+W+N+S) + c2 (corners)
struct Const9 { cplx c0, c1, c2; };
__device__ __forceinline__ Const9 make_const9(double2 kc, double h, bool eps) {
  const double h2 = h * h / 36.0;
  const cplx lam = cmake(kc.x * kc.x, eps ? kc.y : 0.0);
  Const9 c;
  c.c0 = cmake(8.0 / 3.0 - 16.0 * h2 * lam.x, -16.0 * h2 * lam.y);
  c.c1 = cmake(-1.0 / 3.0 - 4.0 * h2 * lam.x, -4.0 * h2 * lam.y);
  c.c2 = cmake(-1.0 / 3.0 - h2 * lam.x, -h2 * lam.y);
  return c;
}

// row of A x at smem slot si (fast interior paths, generic at the boundary)
template <bool HET, bool EPS>
__device__ __forceinline__ cplx node_op(const cplx* __restrict__ X, int si, const Tile& t, int gx,
                                        int gy, int n, double h, const double2* sE, double2 kc,
                                        const Const9& c9) {
  if (gx <= 0 || gx >= n || gy <= 0 || gy >= n)
    return node_op_generic<HET, EPS>(X, si, t, gx, gy, n, h, sE, kc);
  const int SX = t.SX;
  const cplx xp = X[si];
  const cplx W = X[si - 1], E = X[si + 1], S = X[si - SX], N = X[si + SX];
  const cplx SW = X[si - SX - 1], SE = X[si - SX + 1], NW = X[si + SX - 1], NE = X[si + SX + 1];
  if (!HET) {
    const cplx e4 = cmake(W.x + E.x + S.x + N.x, W.y + E.y + S.y + N.y);
    const cplx c4 = cmake(SW.x + SE.x + NW.x + NE.x, SW.y + SE.y + NW.y + NE.y);
    cplx ax = cmul(c9.c0, xp);
    cfma(ax, c9.c1, e4);
    cfma(ax, c9.c2, c4);
    return ax;
  }
  // K part: (1/3)(8 xp - sum of the 8 neighbours)
  const double sx8 = W.x + E.x + S.x + N.x + SW.x + SE.x + NW.x + NE.x;
  const double sy8 = W.y + E.y + S.y + N.y + SW.y + SE.y + NW.y + NE.y;
  cplx ax = cmake((8.0 * xp.x - sx8) * (1.0 / 3.0), (8.0 * xp.y - sy8) * (1.0 / 3.0));
  const double h2 = h * h * (1.0 / 36.0);
  const int e0 = (gx - 1 - (t.X0 - t.R - 1)) + (gy - 1 - (t.Y0 - t.R - 1)) * (t.SX + 1);
  auto quad = [&](int eidx, cplx xh, cplx xv, cplx xd) {
    const double2 c = sE[eidx];
    const cplx lam = cmake(c.x * c.x * h2, EPS ? c.y * h2 : 0.0);
    const cplx mp = cmake(4.0 * xp.x + 2.0 * (xh.x + xv.x) + xd.x, 4.0 * xp.y + 2.0 * (xh.y + xv.y) + xd.y);
    cfms(ax, lam, mp);
  };
  quad(e0, W, S, SW);
  quad(e0 + 1, E, S, SE);
  quad(e0 + t.SX + 1, W, N, NW);
  quad(e0 + t.SX + 2, E, N, NE);
  return ax;
}

// D_p = diag(A_eps): sum over adjacent elements of 2/3 - lambda_e h^2/9, -i k_e h/3 per boundary edge
template <bool HET>
__device__ __forceinline__ cplx node_diag(const Tile& t, int gx, int gy, int n, double h,
                                          const double2* sE, double2 kc) {
  const double h2 = h * h * (4.0 / 36.0);
  cplx dg = cmake(0, 0);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int ex = gx - 1 + (q & 1), ey = gy - 1 + ((q >> 1) & 1);
    if (ex < 0 || ex >= n || ey < 0 || ey >= n) continue;
    const double2 c = elem_coef<HET>(sE, t, ex, ey, kc);
    dg.x += 2.0 / 3.0 - c.x * c.x * h2;
    dg.y -= c.y * h2;
  }
  if (gx == 0 || gx == n || gy == 0 || gy == n) {
    const double h3 = h / 3.0;
    if (gx == 0 || gx == n) {
      const int ex = (gx == 0) ? 0 : n - 1;
      if (gy > 0) dg.y -= elem_coef<HET>(sE, t, ex, gy - 1, kc).x * h3;
      if (gy < n) dg.y -= elem_coef<HET>(sE, t, ex, gy, kc).x * h3;
    }
    if (gy == 0 || gy == n) {
      const int ey = (gy == 0) ? 0 : n - 1;
      if (gx > 0) dg.y -= elem_coef<HET>(sE, t, gx - 1, ey, kc).x * h3;
      if (gx < n) dg.y -= elem_coef<HET>(sE, t, gx, ey, kc).x * h3;
    }
  }
  return dg;
}

// Iterate the region of halo `hal` around the tile without per-element integer
// division; the body sees sx, sy, gx, gy, si and `in` (node inside the domain).
#define FOR_REGION(hal, ...)                                                   \
  {                                                                            \
    const int _w = TX + 2 * (hal), _h = TY + 2 * (hal);                        \
    const int _q = NT / _w, _r = NT - _q * _w;                                 \
    int _x = threadIdx.x % _w, _y = threadIdx.x / _w;                          \
    for (; _y < _h;) {                                                         \
      const int sx = t.R - (hal) + _x, sy = t.R - (hal) + _y;                  \
      const int gx = t.gx(sx), gy = t.gy(sy);                                  \
      const bool in = (gx >= 0 && gx <= n && gy >= rlo && gy <= rhi);          \
      const int si = sy * t.SX + sx;                                           \
      { __VA_ARGS__ }                                                          \
      _x += _r; _y += _q;                                                      \
      if (_x >= _w) { _x -= _w; ++_y; }                                        \
    }                                                                          \
  }

#ifndef FINE_PAIR
#define FINE_PAIR 1   // constant k: a thread takes two vertically adjacent nodes (12 shared-memory loads, not 18)
#endif
// The region of halo `hal` in vertical node pairs (rows sy, sy + 1; the region
// height TY + 2 hal is even); the body sees sx, sy, gx, gy, si of the lower node
// and in0 / in1 (lower / upper node inside the domain).
#define FOR_REGION2(hal, ...)                                                  \
  {                                                                            \
    const int _w = TX + 2 * (hal), _h = (TY + 2 * (hal)) / 2;                  \
    const int _q = NT / _w, _r = NT - _q * _w;                                 \
    int _x = threadIdx.x % _w, _y = threadIdx.x / _w;                          \
    for (; _y < _h;) {                                                         \
      const int sx = t.R - (hal) + _x, sy = t.R - (hal) + 2 * _y;              \
      const int gx = t.gx(sx), gy = t.gy(sy);                                  \
      const bool inx = gx >= 0 && gx <= n;                                     \
      const bool in0 = inx && gy >= rlo && gy <= rhi;                          \
      const bool in1 = inx && gy + 1 >= rlo && gy + 1 <= rhi;                  \
      const int si = sy * t.SX + sx;                                           \
      { __VA_ARGS__ }                                                          \
      _x += _r; _y += _q;                                                      \
      if (_x >= _w) { _x -= _w; ++_y; }                                        \
    }                                                                          \
  }

// Constant k: rows of A x at the vertical pair (si, si + SX).  Both interior:
// the 12 values of rows sy - 1 .. sy + 2 are read once and the sums are formed
// in node_op's order (bit-identical results); otherwise node_op per node.
template <bool EPS>
__device__ __forceinline__ void node_op_pair(const cplx* __restrict__ X, int si, const Tile& t, int gx, int gy,
                                             int n, double h, const double2* sE, double2 kc, const Const9& c9,
                                             bool in0, bool in1, cplx& a0, cplx& a1) {
  if (in0 && in1 && gx > 0 && gx < n && gy > 0 && gy + 1 < n) {
    const int SX = t.SX;
    const cplx* r0 = X + si - SX;
    const cplx W0 = r0[-1], C0 = r0[0], E0 = r0[1];
    const cplx W1 = X[si - 1], C1 = X[si], E1 = X[si + 1];
    const cplx* r2 = X + si + SX;
    const cplx W2 = r2[-1], C2 = r2[0], E2 = r2[1];
    const cplx* r3 = r2 + SX;
    const cplx W3 = r3[-1], C3 = r3[0], E3 = r3[1];
    const cplx h1 = cmake(W1.x + E1.x, W1.y + E1.y);
    {
      const cplx e4 = cmake(h1.x + C0.x + C2.x, h1.y + C0.y + C2.y);
      const cplx c4 = cmake(W0.x + E0.x + W2.x + E2.x, W0.y + E0.y + W2.y + E2.y);
      a0 = cmul(c9.c0, C1);
      cfma(a0, c9.c1, e4);
      cfma(a0, c9.c2, c4);
    }
    {
      const cplx e4 = cmake(W2.x + E2.x + C1.x + C3.x, W2.y + E2.y + C1.y + C3.y);
      const cplx c4 = cmake(h1.x + W3.x + E3.x, h1.y + W3.y + E3.y);
      a1 = cmul(c9.c0, C2);
      cfma(a1, c9.c1, e4);
      cfma(a1, c9.c2, c4);
    }
    return;
  }
  if (in0) a0 = node_op<false, EPS>(X, si, t, gx, gy, n, h, sE, kc, c9);
  if (in1) a1 = node_op<false, EPS>(X, si + t.SX, t, gx, gy + 1, n, h, sE, kc, c9);
}

#ifndef FINE_ASYNC
#define FINE_ASYNC 1   // 1: stage the smoothers' inputs with cp.async (all in flight at once, no registers)
#endif
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// g = virtual global base of the entry's vector; rows outside [rlo, rhi] read as 0.
// Flat index over the region, 4 loads issued per thread before any is used.
__device__ __forceinline__ void load_region(cplx* sX, const cplx* __restrict__ g, const Tile& t,
                                            int n, double scale, int rlo, int rhi) {
  const int N1 = n + 1;
  const int total = t.SX * t.SY;
  for (int base = threadIdx.x; base < total; base += 4 * NT) {
    cplx v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int idx = base + k * NT;
      const int sy = idx / t.SX, sx = idx - sy * t.SX;
      const int gy = t.gy(sy), gx = t.gx(sx);
      v[k] = (idx < total && gy >= rlo && gy <= rhi && gx >= 0 && gx <= n)
                 ? __ldg(&g[(int64_t)gy * N1 + gx]) : cmake(0, 0);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int idx = base + k * NT;
      if (idx < total) sX[idx] = cscale(v[k], scale);
    }
  }
}

__device__ __forceinline__ void load_coef(double2* sE, const double2* __restrict__ coef,
                                          const Tile& t, int n) {
  const int EX = t.SX + 1, EY = t.SY + 1;
  const int total = EX * EY;
  for (int base = threadIdx.x; base < total; base += 4 * NT) {
    double2 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int idx = base + k * NT;
      const int ey0 = idx / EX, ex0 = idx - ey0 * EX;
      const int ey = t.Y0 - t.R - 1 + ey0, ex = t.X0 - t.R - 1 + ex0;
      v[k] = (idx < total && ex >= 0 && ex < n && ey >= 0 && ey < n) ? __ldg(&coef[(int64_t)ey * n + ex])
                                                                     : make_double2(0, 0);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int idx = base + k * NT;
      if (idx < total) sE[idx] = v[k];
    }
  }
}

// cp.async variants: unscaled copies, zero-filled outside the grid / slab rows;
// the caller waits (cp_async_wait_all) before its barrier
__device__ __forceinline__ void load_region_async(cplx* sX, const cplx* __restrict__ g, const Tile& t, int n, int rlo,
                                                  int rhi) {
  const int N1 = n + 1;
  const int total = t.SX * t.SY;
  for (int idx = threadIdx.x; idx < total; idx += NT) {
    const int sy = idx / t.SX, sx = idx - sy * t.SX;
    const int gy = t.gy(sy), gx = t.gx(sx);
    const bool ok = gy >= rlo && gy <= rhi && gx >= 0 && gx <= n;
    cp_async16(&sX[idx], ok ? g + (int64_t)gy * N1 + gx : g + (int64_t)rlo * N1, ok);
  }
}
__device__ __forceinline__ void load_coef_async(double2* sE, const double2* __restrict__ coef, const Tile& t, int n) {
  const int EX = t.SX + 1, EY = t.SY + 1;
  const int total = EX * EY;
  for (int idx = threadIdx.x; idx < total; idx += NT) {
    const int ey0 = idx / EX, ex0 = idx - ey0 * EX;
    const int ey = t.Y0 - t.R - 1 + ey0, ex = t.X0 - t.R - 1 + ex0;
    const bool ok = ex >= 0 && ex < n && ey >= 0 && ey < n;
    cp_async16(&sE[idx], ok ? coef + (int64_t)ey * n + ex : coef, ok);
  }
}

struct FineK {   // per-launch constants
  const cplx* dinv; int64_t stride;        // precomputed D^{-1} (het), entry stride
  int n; double h; double omega; int nu;
  const double2* coef; int64_t coef_bs;   // het
  const double2* kc;                       // constant k: [B]
  const int* st;
  const int2* slab; int G;                 // slab layout (Level)
};

// tile placement inside entry b's owned rows; false: tile beyond the slab
#define SLAB_TILE(P, b, n)                                                       \
  const int2 sl = slab_of(P.slab, b, n);                                         \
  const int rlo = max(0, sl.x - P.G), rhi = min(n, sl.y - 1 + P.G);              \
  const int64_t vofs = (int64_t)(sl.x - P.G) * (n + 1);                          \
  if (sl.x + (int)blockIdx.y * TY >= sl.y) return;

// --------------------------------------------------------------------- apply
template <bool HET, bool EPS>
__global__ void __launch_bounds__(NT) k_apply2d(FineK P, VArg x, VArg y, VArg sub) {
  const int b = blockIdx.z;
  if (P.st && P.st[b]) return;
  extern __shared__ double4 smem_raw[];
  const int n = P.n;
  SLAB_TILE(P, b, n)
  Tile t;
  t.X0 = blockIdx.x * TX; t.Y0 = sl.x + blockIdx.y * TY; t.R = 1; t.SX = TX + 2; t.SY = TY + 2;
  cplx* sX = reinterpret_cast<cplx*>(smem_raw);
  double2* sE = reinterpret_cast<double2*>(sX + t.SX * t.SY);
  const double2 kc = HET ? make_double2(0, 0) : P.kc[b];
  const Const9 c9 = make_const9(kc, P.h, EPS);
  load_region(sX, x.at(b) - vofs, t, n, 1.0, rlo, rhi);
  if (HET) load_coef(sE, P.coef + b * P.coef_bs, t, n);
  __syncthreads();
  cplx* yb = y.at(b) - vofs;
  const cplx* sb = sub.p ? sub.at(b) - vofs : nullptr;
  FOR_REGION(0, if (in && gy < sl.y) {
    cplx ax = node_op<HET, EPS>(sX, si, t, gx, gy, n, P.h, sE, kc, c9);
    const int64_t gi = (int64_t)gy * (n + 1) + gx;
    if (sb) ax = csub(sb[gi], ax);
    yb[gi] = ax;
  })
}

// D^{-1} at a region node: heterogeneous -> the precomputed copy staged in smem;
// constant k -> the interior centre coefficient, the element loop at the boundary
template <bool HET>
__device__ __forceinline__ cplx dinv_at(const cplx* sDi, const cplx* dg, int si, const Tile& t, int gx,
                                        int gy, int n, double h, const double2* sE, double2 kc, cplx di_int) {
  if (HET) return FINE_DI_GLOBAL ? __ldg(&dg[(int64_t)gy * (n + 1) + gx]) : sDi[si];
  if (gx > 0 && gx < n && gy > 0 && gy < n) return di_int;
  return cinv(node_diag<false>(t, gx, gy, n, h, sE, kc));
}

// Per-sample scalars of a fine launch, loaded together before any is used
// (status, slab bounds, the Krylov slot behind f, its scale, constant k) so the
// prologue pays one memory latency instead of a chain of them.
#define FINE_PROLOGUE(P, b, n, f, fs)                                            \
  const int stb = P.st ? __ldg(P.st + b) : 0;                                    \
  const int2 sl = slab_of(P.slab, b, n);                                         \
  const cplx* fg = f.at(b);                                                      \
  const double fsc = fs.at(b);                                                   \
  const double2 kc = HET ? make_double2(0, 0) : __ldg(P.kc + b);                 \
  if (stb) return;                                                               \
  const int rlo = max(0, sl.x - P.G), rhi = min(n, sl.y - 1 + P.G);              \
  const int64_t vofs = (int64_t)(sl.x - P.G) * (n + 1);                          \
  if (sl.x + (int)blockIdx.y * TY >= sl.y) return;

// ------------------------------------------------- pre-smoothing + restriction
// u = S^nu(0; f), rc = I^T (f - A_eps u).  Halo R = nu + 1.
// NUC > 0: nu fixed at compile time (region sizes, smem strides and the step
// loop fold to constants); NUC = 0: nu from P.
template <bool HET, int NUC>
__global__ void __launch_bounds__(NT, HET && !FINE_DI_GLOBAL ? 3 : FINE_CONST_MINB) k_pre2d(FineK P, VArg f, SArg fs, VArg uo, VArg rco) {
  const int b = blockIdx.z;
  extern __shared__ double4 smem_raw[];
  const int n = P.n, nu = NUC > 0 ? NUC : P.nu;
  const double omega = P.omega, h = P.h;
  FINE_PROLOGUE(P, b, n, f, fs)
  Tile t;
  t.X0 = blockIdx.x * TX; t.Y0 = sl.x + blockIdx.y * TY; t.R = nu + 1;
  t.SX = TX + 2 * t.R; t.SY = TY + 2 * t.R;
  const int S = t.SX * t.SY;
  cplx* sF = reinterpret_cast<cplx*>(smem_raw);
  cplx* sA = sF + S;
  cplx* sB = sA + S;
  cplx* sDi = sB + S;                                   // HET, D^{-1} staged
  double2* sE = reinterpret_cast<double2*>(sDi + (FINE_DI_GLOBAL ? 0 : S));   // HET only
  const cplx* dg = HET ? P.dinv + (int64_t)b * P.stride - vofs : nullptr;
  const Const9 c9 = make_const9(kc, h, true);
  // constant k: interior D = centre coefficient; its reciprocal (an FP64 division) is
  // formed while the region loads are in flight, not after the barrier
  const cplx di_int = HET ? cmake(0, 0) : cinv(c9.c0);
  // f staged unscaled with cp.async (the Krylov scale fsc is applied where it is read)
  const double fsa = FINE_ASYNC ? fsc : 1.0;
  if (FINE_ASYNC) {
    load_region_async(sF, fg - vofs, t, n, rlo, rhi);
    if (HET) {
      if (!FINE_DI_GLOBAL) load_region_async(sDi, dg, t, n, rlo, rhi);
      load_coef_async(sE, P.coef + b * P.coef_bs, t, n);
    }
    cp_async_wait_all();
  } else {
    load_region(sF, fg - vofs, t, n, fsc, rlo, rhi);
    if (HET) {
      if (!FINE_DI_GLOBAL) load_region(sDi, dg, t, n, 1.0, rlo, rhi);
      load_coef(sE, P.coef + b * P.coef_bs, t, n);
    }
  }
  __syncthreads();
  // the first step from u = 0 (pointwise) on the full region
  FOR_REGION(t.R, {
    cplx v = cmake(0, 0);
    if (in) v = cscale(cmul(dinv_at<HET>(sDi, dg, si, t, gx, gy, n, h, sE, kc, di_int), sF[si]), omega * fsa);
    sA[si] = v;
    sB[si] = cmake(0, 0);
  })
  __syncthreads();
  cplx* cur = sA;
  cplx* nxt = sB;
  for (int step = 2; step <= nu; ++step) {
    const int hal = t.R - step + 1;
    auto jac = [&](int si, int gx, int gy, cplx ax) {
      const cplx di = dinv_at<HET>(sDi, dg, si, t, gx, gy, n, h, sE, kc, di_int);
      cplx v = cur[si];
      cfma(v, cscale(di, omega), csub(cscale(sF[si], fsa), ax));
      nxt[si] = v;
    };
    if constexpr (!HET && FINE_PAIR) {
      FOR_REGION2(hal, if (in0 || in1) {
        cplx a0, a1;
        node_op_pair<true>(cur, si, t, gx, gy, n, h, sE, kc, c9, in0, in1, a0, a1);
        if (in0) jac(si, gx, gy, a0);
        if (in1) jac(si + t.SX, gx, gy + 1, a1);
      })
    } else {
      FOR_REGION(hal, if (in) jac(si, gx, gy, node_op<HET, true>(cur, si, t, gx, gy, n, h, sE, kc, c9));)
    }
    __syncthreads();
    cplx* tmp = cur; cur = nxt; nxt = tmp;
  }
  // residual on halo 1 -> nxt ; u on the tile (owned rows) -> global
  cplx* ub = uo.at(b) - vofs;
  auto res = [&](int si, int sx, int sy, int gx, int gy, cplx ax) {
    nxt[si] = csub(cscale(sF[si], fsa), ax);
    if (sx >= t.R && sx < t.R + TX && sy >= t.R && sy < t.R + TY && gy < sl.y)
      ub[(int64_t)gy * (n + 1) + gx] = cur[si];
  };
  if constexpr (!HET && FINE_PAIR) {
    FOR_REGION2(1, if (in0 || in1) {
      cplx a0, a1;
      node_op_pair<true>(cur, si, t, gx, gy, n, h, sE, kc, c9, in0, in1, a0, a1);
      if (in0) res(si, sx, sy, gx, gy, a0);
      if (in1) res(si + t.SX, sx, sy + 1, gx, gy + 1, a1);
    })
  } else {
    FOR_REGION(1, if (in) res(si, sx, sy, gx, gy, node_op<HET, true>(cur, si, t, gx, gy, n, h, sE, kc, c9));)
  }
  __syncthreads();
  // restriction I^T at coarse nodes (2I, 2J) inside the tile
  const int nc = n / 2;
  cplx* rcb = rco.at(b);
  {
    const int i = threadIdx.x;   // (TX/2) x (TY/2) = 128 coarse nodes per tile
    if (i < (TX / 2) * (TY / 2)) {
      const int cx = t.X0 / 2 + (i % (TX / 2)), cy = t.Y0 / 2 + i / (TX / 2);
      if (cx <= nc && cy <= nc && 2 * cy < sl.y) {
        const int sx = t.R + 2 * cx - t.X0, sy = t.R + 2 * cy - t.Y0;
        cplx acc = cmake(0, 0);
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
          for (int dx = -1; dx <= 1; ++dx) {
            const int gx = 2 * cx + dx, gy = 2 * cy + dy;
            if (gx < 0 || gx > n || gy < 0 || gy > n) continue;
            const double w = (dx ? 0.5 : 1.0) * (dy ? 0.5 : 1.0);
            const cplx r = nxt[(sy + dy) * t.SX + sx + dx];
            acc.x += w * r.x;
            acc.y += w * r.y;
          }
        rcb[(int64_t)cy * (nc + 1) + cx] = acc;
      }
    }
  }
}

// coarse block staged by the post-smoother: coarse nodes (cx0 + i, cy0 + j)
constexpr int CW_EXTRA = 2;
__host__ __device__ constexpr int post_cw(int R) { return TX / 2 + R + CW_EXTRA; }
__host__ __device__ constexpr int post_ch(int R) { return TY / 2 + R + CW_EXTRA; }

// ------------------------------------- prolongation + correction + post-smoothing
// z = S^nu(u + I ec; f); if w: w = A_0 z.  Halo R = nu + (w ? 1 : 0).
template <bool HET, bool WITH_W, int NUC>
__global__ void __launch_bounds__(NT, HET ? 3 : FINE_CONST_MINB) k_post2d(FineK P, VArg f, SArg fs, VArg uin, VArg ecin,
                                                            VArg zo, VArg wo) {
  const int b = blockIdx.z;
  extern __shared__ double4 smem_raw[];
  const int n = P.n, nu = NUC > 0 ? NUC : P.nu;
  const double omega = P.omega, h = P.h;
  FINE_PROLOGUE(P, b, n, f, fs)
  Tile t;
  t.X0 = blockIdx.x * TX; t.Y0 = sl.x + blockIdx.y * TY; t.R = nu + (WITH_W ? 1 : 0);
  t.SX = TX + 2 * t.R; t.SY = TY + 2 * t.R;
  const int S = t.SX * t.SY;
  const int CW = post_cw(t.R), CH = post_ch(t.R);
  cplx* sF = reinterpret_cast<cplx*>(smem_raw);
  cplx* sA = sF + S;
  cplx* sB = sA + S;
  cplx* sC = sB + S;                                    // coarse block, CW x CH
  cplx* sDi = sC + CW * CH;                             // HET, D^{-1} staged
  double2* sE = reinterpret_cast<double2*>(sDi + (FINE_DI_GLOBAL ? 0 : S));   // HET only
  const cplx* dg = HET ? P.dinv + (int64_t)b * P.stride - vofs : nullptr;
  const Const9 c9e = make_const9(kc, h, true);
  const cplx di_int = HET ? cmake(0, 0) : cinv(c9e.c0);   // formed under the region loads
  const double fsa = FINE_ASYNC ? fsc : 1.0;
  if (FINE_ASYNC) {
    load_region_async(sF, fg - vofs, t, n, rlo, rhi);
    load_region_async(sA, uin.at(b) - vofs, t, n, rlo, rhi);
    if (HET) {
      if (!FINE_DI_GLOBAL) load_region_async(sDi, dg, t, n, rlo, rhi);
      load_coef_async(sE, P.coef + b * P.coef_bs, t, n);
    }
  } else {
    load_region(sF, fg - vofs, t, n, fsc, rlo, rhi);
    load_region(sA, uin.at(b) - vofs, t, n, 1.0, rlo, rhi);
  }
  // coarse nodes under the region: cx in [cx0, cx0 + CW), cy in [cy0, cy0 + CH)
  const int nc = n / 2, NC1 = nc + 1;
  const int cx0 = (t.X0 - t.R) >> 1, cy0 = (t.Y0 - t.R) >> 1;
  {
    const cplx* ecv = ecin.at(b);
    const int total = CW * CH;
    for (int base = threadIdx.x; base < total; base += 2 * NT) {
      cplx v[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int idx = base + k * NT;
        const int j = idx / CW, i = idx - j * CW;
        const int cx = cx0 + i, cy = cy0 + j;
        v[k] = (idx < total && cx >= 0 && cx <= nc && cy >= 0 && cy <= nc) ? __ldg(&ecv[cy * NC1 + cx])
                                                                           : cmake(0, 0);
      }
#pragma unroll
      for (int k = 0; k < 2; ++k)
        if (base + k * NT < total) sC[base + k * NT] = v[k];
    }
  }
  if (HET && !FINE_ASYNC) {
    if (!FINE_DI_GLOBAL) load_region(sDi, dg, t, n, 1.0, rlo, rhi);
    load_coef(sE, P.coef + b * P.coef_bs, t, n);
  }
  if (FINE_ASYNC) cp_async_wait_all();
  __syncthreads();
  // u + I ec on the full region (bilinear interpolation from the staged block)
  FOR_REGION(t.R, {
    if (in) {
      cplx v = sA[si];
      const int ci = (gx >> 1) - cx0, cj = (gy >> 1) - cy0;
      const cplx* c = sC + cj * CW + ci;
      const cplx a = c[0];
      if (gx & 1) {
        const cplx bq = c[1];
        if (gy & 1) {
          const cplx cc = c[CW], d = c[CW + 1];
          v.x += 0.25 * (a.x + bq.x + cc.x + d.x);
          v.y += 0.25 * (a.y + bq.y + cc.y + d.y);
        } else {
          v.x += 0.5 * (a.x + bq.x);
          v.y += 0.5 * (a.y + bq.y);
        }
      } else if (gy & 1) {
        const cplx cc = c[CW];
        v.x += 0.5 * (a.x + cc.x);
        v.y += 0.5 * (a.y + cc.y);
      } else {
        v.x += a.x;
        v.y += a.y;
      }
      sA[si] = v;
    }
    sB[si] = cmake(0, 0);
  })
  __syncthreads();
  cplx* cur = sA;
  cplx* nxt = sB;
  for (int step = 1; step <= nu; ++step) {
    const int hal = t.R - step;
    auto jac = [&](int si, int gx, int gy, cplx ax) {
      const cplx di = dinv_at<HET>(sDi, dg, si, t, gx, gy, n, h, sE, kc, di_int);
      cplx v = cur[si];
      cfma(v, cscale(di, omega), csub(cscale(sF[si], fsa), ax));
      nxt[si] = v;
    };
    if constexpr (!HET && FINE_PAIR) {
      FOR_REGION2(hal, if (in0 || in1) {
        cplx a0, a1;
        node_op_pair<true>(cur, si, t, gx, gy, n, h, sE, kc, c9e, in0, in1, a0, a1);
        if (in0) jac(si, gx, gy, a0);
        if (in1) jac(si + t.SX, gx, gy + 1, a1);
      })
    } else {
      FOR_REGION(hal, if (in) jac(si, gx, gy, node_op<HET, true>(cur, si, t, gx, gy, n, h, sE, kc, c9e));)
    }
    __syncthreads();
    cplx* tmp = cur; cur = nxt; nxt = tmp;
  }
  cplx* zb = zo.at(b) - vofs;
  cplx* wb = WITH_W ? wo.at(b) - vofs : nullptr;
  const Const9 c90 = make_const9(kc, h, false);
  if constexpr (!HET && FINE_PAIR) {
    FOR_REGION2(0, {
      const bool o0 = in0 && gy < sl.y, o1 = in1 && gy + 1 < sl.y;
      if (o0 || o1) {
        cplx a0, a1;
        if (WITH_W) node_op_pair<false>(cur, si, t, gx, gy, n, h, sE, kc, c90, o0, o1, a0, a1);
        const int64_t gi = (int64_t)gy * (n + 1) + gx;
        if (o0) {
          zb[gi] = cur[si];
          if (WITH_W) wb[gi] = a0;
        }
        if (o1) {
          zb[gi + n + 1] = cur[si + t.SX];
          if (WITH_W) wb[gi + n + 1] = a1;
        }
      }
    })
  } else {
    FOR_REGION(0, if (in && gy < sl.y) {
      const int64_t gi = (int64_t)gy * (n + 1) + gx;
      zb[gi] = cur[si];
      if (WITH_W) wb[gi] = node_op<HET, false>(cur, si, t, gx, gy, n, h, sE, kc, c90);
    })
  }
}

// ------------------------------------------------------------ precomputed D^{-1}
// D_p = sum over adjacent elements of 2/3 - lambda_e h^2/9, -i k_e h/3 per boundary
// edge (reading C6), at every stored node of entry b (owned + ghost rows)
__global__ void k_dinv2d(int n, double h, const double2* __restrict__ coef, int64_t coef_bs,
                         const int2* __restrict__ slab, int G, int64_t stride, int rows, cplx* __restrict__ dinv) {
  const int b = blockIdx.z;
  const int N1 = n + 1;
  const int2 sl = slab_of(slab, b, n);
  const int gx = blockIdx.x * blockDim.x + threadIdx.x;
  const int gy = sl.x - G + (int)blockIdx.y;
  if (gx > n || gy < 0 || gy > n || (int)blockIdx.y >= rows) return;
  const double2* cf = coef + b * coef_bs;
  const double h2 = h * h * (4.0 / 36.0), h3 = h / 3.0;
  auto K = [&](int ex, int ey) { return __ldg(&cf[(int64_t)ey * n + ex]); };
  cplx dg = cmake(0, 0);
  for (int q = 0; q < 4; ++q) {
    const int ex = gx - 1 + (q & 1), ey = gy - 1 + ((q >> 1) & 1);
    if (ex < 0 || ex >= n || ey < 0 || ey >= n) continue;
    const double2 c = K(ex, ey);
    dg.x += 2.0 / 3.0 - c.x * c.x * h2;
    dg.y -= c.y * h2;
  }
  if (gx == 0 || gx == n) {
    const int ex = gx == 0 ? 0 : n - 1;
    if (gy > 0) dg.y -= K(ex, gy - 1).x * h3;
    if (gy < n) dg.y -= K(ex, gy).x * h3;
  }
  if (gy == 0 || gy == n) {
    const int ey = gy == 0 ? 0 : n - 1;
    if (gx > 0) dg.y -= K(gx - 1, ey).x * h3;
    if (gx < n) dg.y -= K(gx, ey).x * h3;
  }
  dinv[(int64_t)b * stride + (int64_t)blockIdx.y * N1 + gx] = cinv(dg);
}

// ------------------------------------------------------------ coarse stencil
// st[b][node * 9 + (dx+1) + 3 (dy+1)] = entry of A_eps^{(1)} (rediscretisation on
// the 2h mesh; reading C4)
template <bool HET>
__global__ void k_stencil2d(int n, double h, const double2* __restrict__ coef, int64_t coef_bs,
                            const double2* __restrict__ kcv, cplx* __restrict__ stv) {
  const int N1 = n + 1;
  const int b = blockIdx.y;
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= (int64_t)N1 * N1) return;
  const double2* cf = HET ? coef + b * coef_bs : nullptr;
  const double2 kc = HET ? make_double2(0, 0) : kcv[b];
  cplx* st = stv + (int64_t)b * N1 * N1 * 9;
  const int gx = node % N1, gy = node / N1;
  cplx e[9];
#pragma unroll
  for (int o = 0; o < 9; ++o) e[o] = cmake(0, 0);
  const double h2 = h * h / 36.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int dx = (q & 1) ? 1 : -1, dy = (q & 2) ? 1 : -1;
    const int ex = gx + (dx < 0 ? -1 : 0), ey = gy + (dy < 0 ? -1 : 0);
    if (ex < 0 || ex >= n || ey < 0 || ey >= n) continue;
    const double2 c = HET ? cf[(int64_t)ey * n + ex] : kc;
    const cplx lam = cmake(c.x * c.x, c.y);
    auto add = [&](int o, double kv, double mv) {
      e[o].x += kv - lam.x * mv * h2;
      e[o].y += -lam.y * mv * h2;
    };
    add(4, 2.0 / 3.0, 4.0);                      // self
    add(4 + dx, -1.0 / 6.0, 2.0);                // x neighbour
    add(4 + 3 * dy, -1.0 / 6.0, 2.0);            // y neighbour
    add(4 + dx + 3 * dy, -1.0 / 3.0, 1.0);       // diagonal
  }
  auto bedge = [&](int ex, int ey, int o) {
    const double k = HET ? cf[(int64_t)ey * n + ex].x : kc.x;
    e[4].y -= k * h / 3.0;
    e[o].y -= k * h / 6.0;
  };
  if (gx == 0 || gx == n) {
    const int ex = gx == 0 ? 0 : n - 1;
    if (gy > 0) bedge(ex, gy - 1, 4 - 3);
    if (gy < n) bedge(ex, gy, 4 + 3);
  }
  if (gy == 0 || gy == n) {
    const int ey = gy == 0 ? 0 : n - 1;
    if (gx > 0) bedge(gx - 1, ey, 3);
    if (gx < n) bedge(gx, ey, 5);
  }
#pragma unroll
  for (int o = 0; o < 9; ++o) st[node * 9 + o] = e[o];
}

size_t smem_bytes(int R, int nfields, bool het) {
  const int SX = TX + 2 * R, SY = TY + 2 * R;
  size_t b = (size_t)SX * SY * sizeof(cplx) * nfields;
  if (het) b += (size_t)(SX + 1) * (SY + 1) * sizeof(double2);
  return b;
}
// pre: f, two iterates (+ D^{-1}, element coefficients if heterogeneous)
size_t pre_smem(int R, bool het) { return smem_bytes(R, het && !FINE_DI_GLOBAL ? 4 : 3, het); }
// post: as pre plus the staged coarse block
size_t post_smem(int R, bool het) {
  return pre_smem(R, het) + (size_t)post_cw(R) * post_ch(R) * sizeof(cplx);
}

hh_status set_smem(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) {
    HH_CUDA_TRY(smem_attr((const void*)fn, bytes));
  }
  return HH_OK;
}

FineK make_k(const Level& L, int nu, double omega, const int* st) {
  FineK P;
  P.n = L.n; P.h = L.h; P.omega = omega; P.nu = nu;
  P.coef = L.coef; P.coef_bs = L.coef_bs; P.kc = L.kc; P.st = st;
  P.dinv = L.dinv; P.stride = L.stride;
  P.slab = L.slab; P.G = L.G;
  return P;
}

}  // namespace

// ----------------------------------------------------------------- host API
hh_status fine_apply2d(const Level& L, int B, const int* st, int op, VArg x, VArg y, VArg sub,
                       cudaStream_t s) {
  const int n = L.n;
  dim3 grid((n + 1 + TX - 1) / TX, (L.maxloc + TY - 1) / TY, B);
  const size_t sm = smem_bytes(1, 1, L.het);
  const FineK P = make_k(L, 0, 0, st);
#define LAUNCH_APPLY(H, E)                                        \
  {                                                               \
    HH_TRY(set_smem((const void*)k_apply2d<H, E>, sm));           \
    k_apply2d<H, E><<<grid, NT, sm, s>>>(P, x, y, sub);           \
  }
  if (L.het) {
    if (op == HH_OP_A0) LAUNCH_APPLY(true, false) else LAUNCH_APPLY(true, true)
  } else {
    if (op == HH_OP_A0) LAUNCH_APPLY(false, false) else LAUNCH_APPLY(false, true)
  }
#undef LAUNCH_APPLY
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status fine_pre2d(const Level& L, int B, const int* st, int nu, double omega, VArg f, SArg fs,
                     VArg u, VArg rc, cudaStream_t s) {
  const int n = L.n;
  dim3 grid((n + 1 + TX - 1) / TX, (L.maxloc + TY - 1) / TY, B);
  if (L.het && !L.dinv) { hh_set_error("fine_pre2d: heterogeneous level without D^-1"); return HH_E_STATE; }
  const size_t sm = pre_smem(nu + 1, L.het);
  const FineK P = make_k(L, nu, omega, st);
#define LAUNCH_PRE(H, NU)                                         \
  {                                                               \
    HH_TRY(set_smem((const void*)k_pre2d<H, NU>, sm));            \
    k_pre2d<H, NU><<<grid, NT, sm, s>>>(P, f, fs, u, rc);         \
  }
  if (L.het) {
    if (nu == 2) LAUNCH_PRE(true, 2) else LAUNCH_PRE(true, 0)
  } else {
    if (nu == 2) LAUNCH_PRE(false, 2) else LAUNCH_PRE(false, 0)
  }
#undef LAUNCH_PRE
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status fine_post2d(const Level& L, int B, const int* st, int nu, double omega, VArg f, SArg fs,
                      VArg u, VArg ec, VArg z, VArg w, cudaStream_t s) {
  const int n = L.n;
  dim3 grid((n + 1 + TX - 1) / TX, (L.maxloc + TY - 1) / TY, B);
  const bool ww = w.p != nullptr;
  if (L.het && !L.dinv) { hh_set_error("fine_post2d: heterogeneous level without D^-1"); return HH_E_STATE; }
  const size_t sm = post_smem(nu + (ww ? 1 : 0), L.het);
  const FineK P = make_k(L, nu, omega, st);
#define LAUNCH_POST1(H, W, NU)                                             \
  {                                                                        \
    HH_TRY(set_smem((const void*)k_post2d<H, W, NU>, sm));                 \
    k_post2d<H, W, NU><<<grid, NT, sm, s>>>(P, f, fs, u, ec, z, w);        \
  }
#define LAUNCH_POST(H, W) \
  if (nu == 2) LAUNCH_POST1(H, W, 2) else LAUNCH_POST1(H, W, 0)
  if (L.het) {
    if (ww) { LAUNCH_POST(true, true) } else { LAUNCH_POST(true, false) }
  } else {
    if (ww) { LAUNCH_POST(false, true) } else { LAUNCH_POST(false, false) }
  }
#undef LAUNCH_POST1
#undef LAUNCH_POST
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status coarse_stencil2d(const Level& C, int B, cplx* st, cudaStream_t s) {
  const int64_t N = C.nodes;
  const int bs = 128;
  dim3 g((unsigned)((N + bs - 1) / bs), B);
  if (C.het)
    k_stencil2d<true><<<g, bs, 0, s>>>(C.n, C.h, C.coef, C.coef_bs, nullptr, st);
  else
    k_stencil2d<false><<<g, bs, 0, s>>>(C.n, C.h, nullptr, 0, C.kc, st);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status fine_dinv2d(const Level& L, int B, cudaStream_t s) {
  const int rows = L.maxloc + 2 * L.G;
  dim3 g((L.n + 1 + 127) / 128, rows, B);
  k_dinv2d<<<g, 128, 0, s>>>(L.n, L.h, L.coef, L.coef_bs, L.slab, L.G, L.stride, rows, L.dinv);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}
