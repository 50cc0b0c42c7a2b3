// 3D fine-level kernels (batched): matrix-free trilinear Q1 operator on the
// 27-point neighbourhood, damped Jacobi, residual, I^T restriction and
// trilinear prolongation.
//
// Element matrices (tensor products of the 1D P1 forms):
//   K^e row of a corner node: h/36 (12 xp + 0 * (3 one-axis nbrs)
//                                   - 3 * (3 two-axis nbrs) - 3 * (body diagonal))
//   M^e row: h^3/216 (8 xp + 4 sum(one-axis) + 2 sum(two-axis) + body diagonal)
//   boundary face (2D mass, weight k_e): h^2/36 (4 xp + 2 sum(in-face one-axis) + in-face diagonal)
// Assembled interior stencils: K centre 8h/3, face 0, edge -h/6, corner -h/12;
// M = (h/6)^3 [1 4 1] x [1 4 1] x [1 4 1].  D = diag(A_eps) (reading C6).
// Restriction weights prod_d (1 - |delta_d|/2) (reading C5), prolongation its transpose.
//
// Round-1 3D design: one thread per node, neighbours through L1/L2 (__ldg), one
// kernel per Jacobi step (the 3D two-grid is dominated by the coarse solve,
// SURVEY 8(d)); temporal blocking as in 2D is future work.
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include "hh_internal.cuh"

namespace {

constexpr int BX = 32, BY = 8;

struct F3 {
  const cplx* dinv; int64_t stride;      // precomputed D^{-1} (het), entry stride
  int n; double h; double omega;
  const double2* coef; int64_t coef_bs;
  const double2* kc;
  const int* st;
  int N1;
  const int2* slab; int G; int maxloc;   // slab layout (Level)
  int ext;                               // planes computed beyond the owned ones (per side)
};

// node of this thread: planes [max(0, z0 - ext), min(n + 1, z1 + ext)) of entry b;
// vofs = offset of the virtual global base of entry b's fine vectors
__device__ __forceinline__ bool node_of(const F3& P, int& b, int& gx, int& gy, int& gz, int64_t& vofs) {
  gx = blockIdx.x * BX + threadIdx.x;
  gy = blockIdx.y * BY + threadIdx.y;
  const int span = P.maxloc + 2 * P.ext;
  b = blockIdx.z / span;
  const int2 sl = slab_of(P.slab, b, P.n);
  const int zlo = max(0, sl.x - P.ext), zhi = min(P.N1, sl.y + P.ext);
  gz = zlo + (int)(blockIdx.z % span);
  vofs = (int64_t)(sl.x - P.G) * P.N1 * P.N1;
  return gx < P.N1 && gy < P.N1 && gz < zhi;
}

template <bool HET>
__device__ __forceinline__ double2 coef3(const F3& P, const double2* cf, double2 kc, int ex, int ey,
                                         int ez) {
  if (HET) return __ldg(&cf[((int64_t)ez * P.n + ey) * P.n + ex]);
  return kc;
}

// row of A x at node (gx, gy, gz) reading x from global memory
// x values through an accessor: plain loads, or (first post-smoothing step of the
// z-marching path's boundary nodes) u + I e_c formed on the fly
struct LdgAcc {
  const cplx* x;
  __device__ __forceinline__ cplx operator()(int64_t i, int, int, int) const { return __ldg(&x[i]); }
};
struct ProlongAcc {   // u + I e_c at fine node (gx, gy, gz) (trilinear I, weights 1, 1/2, 1/4, 1/8)
  const cplx* u;
  const cplx* ec;
  int NC1;
  __device__ __forceinline__ cplx operator()(int64_t i, int gx, int gy, int gz) const {
    cplx v = __ldg(&u[i]);
    const int cx0 = gx >> 1, cy0 = gy >> 1, cz0 = gz >> 1;
    const double w = ((gx & 1) ? 0.5 : 1.0) * ((gy & 1) ? 0.5 : 1.0) * ((gz & 1) ? 0.5 : 1.0);
    for (int k = 0; k <= (gz & 1); ++k)
      for (int j = 0; j <= (gy & 1); ++j)
        for (int q = 0; q <= (gx & 1); ++q) {
          const cplx c = __ldg(&ec[((int64_t)(cz0 + k) * NC1 + cy0 + j) * NC1 + cx0 + q]);
          v.x += w * c.x;
          v.y += w * c.y;
        }
    return v;
  }
};

template <bool HET, bool EPS, typename ACC = LdgAcc>
__device__ cplx row3(const F3& P, ACC acc, const double2* cf, double2 kc, int gx, int gy, int gz) {
  const int n = P.n, N1 = P.N1;
  const double h = P.h;
  const int64_t gi = ((int64_t)gz * N1 + gy) * N1 + gx;
  auto X = [&](int dx, int dy, int dz) {
    return acc(gi + ((int64_t)dz * N1 + dy) * N1 + dx, gx + dx, gy + dy, gz + dz);
  };
  const cplx xp = X(0, 0, 0);
  const double hk = h / 36.0, hm = h * h * h / 216.0;
  cplx ax = cmake(0, 0);
  const bool interior = gx > 0 && gx < n && gy > 0 && gy < n && gz > 0 && gz < n;
  if (interior && !HET) {
    // assembled 27-point stencil: classes centre / face / edge / corner
    cplx sf = cmake(0, 0), se = cmake(0, 0), sc = cmake(0, 0);
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
      for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
          const int cls = (dx != 0) + (dy != 0) + (dz != 0);
          if (cls == 0) continue;
          const cplx v = X(dx, dy, dz);
          cplx& a = cls == 1 ? sf : (cls == 2 ? se : sc);
          a.x += v.x; a.y += v.y;
        }
    const cplx lam = cmake(kc.x * kc.x, EPS ? kc.y : 0.0);
    const cplx c0 = cmake(8.0 * h / 3.0 - 64.0 * hm * lam.x, -64.0 * hm * lam.y);
    const cplx cf_ = cmake(-16.0 * hm * lam.x, -16.0 * hm * lam.y);
    const cplx ce = cmake(-h / 6.0 - 4.0 * hm * lam.x, -4.0 * hm * lam.y);
    const cplx cc = cmake(-h / 12.0 - hm * lam.x, -hm * lam.y);
    ax = cmul(c0, xp);
    cfma(ax, cf_, sf);
    cfma(ax, ce, se);
    cfma(ax, cc, sc);
    return ax;
  }
  // element (octant) loop
  for (int o = 0; o < 8; ++o) {
    const int dx = (o & 1) ? 1 : -1, dy = (o & 2) ? 1 : -1, dz = (o & 4) ? 1 : -1;
    const int ex = gx + (dx < 0 ? -1 : 0), ey = gy + (dy < 0 ? -1 : 0), ez = gz + (dz < 0 ? -1 : 0);
    if (ex < 0 || ex >= n || ey < 0 || ey >= n || ez < 0 || ez >= n) continue;
    const cplx a1x = X(dx, 0, 0), a1y = X(0, dy, 0), a1z = X(0, 0, dz);
    const cplx a2xy = X(dx, dy, 0), a2xz = X(dx, 0, dz), a2yz = X(0, dy, dz);
    const cplx a3 = X(dx, dy, dz);
    const cplx s1 = cmake(a1x.x + a1y.x + a1z.x, a1x.y + a1y.y + a1z.y);
    const cplx s2 = cmake(a2xy.x + a2xz.x + a2yz.x, a2xy.y + a2xz.y + a2yz.y);
    const cplx kp = cmake(hk * (12.0 * xp.x - 3.0 * s2.x - 3.0 * a3.x),
                          hk * (12.0 * xp.y - 3.0 * s2.y - 3.0 * a3.y));
    const cplx mp = cmake(hm * (8.0 * xp.x + 4.0 * s1.x + 2.0 * s2.x + a3.x),
                          hm * (8.0 * xp.y + 4.0 * s1.y + 2.0 * s2.y + a3.y));
    const double2 c = coef3<HET>(P, cf, kc, ex, ey, ez);
    const cplx lam = cmake(c.x * c.x, EPS ? c.y : 0.0);
    ax = cadd(ax, kp);
    cfms(ax, lam, mp);
  }
  // boundary faces
  if (!interior) {
    const double hb = h * h / 36.0;
    // face normal to axis a at coordinate side; the in-face axes u, v
    for (int a = 0; a < 3; ++a) {
      const int ga = a == 0 ? gx : (a == 1 ? gy : gz);
      if (ga != 0 && ga != n) continue;
      const int ea = ga == 0 ? 0 : n - 1;
      const int u = (a + 1) % 3, v = (a + 2) % 3;
      const int gu = u == 0 ? gx : (u == 1 ? gy : gz);
      const int gv = v == 0 ? gx : (v == 1 ? gy : gz);
      for (int q = 0; q < 4; ++q) {
        const int du = (q & 1) ? 1 : -1, dv = (q & 2) ? 1 : -1;
        const int eu = gu + (du < 0 ? -1 : 0), ev = gv + (dv < 0 ? -1 : 0);
        if (eu < 0 || eu >= n || ev < 0 || ev >= n) continue;
        int e3[3], d_u[3] = {0, 0, 0}, d_v[3] = {0, 0, 0};
        e3[a] = ea; e3[u] = eu; e3[v] = ev;
        d_u[u] = du; d_v[v] = dv;
        const double k = coef3<HET>(P, cf, kc, e3[0], e3[1], e3[2]).x;
        const cplx xu = X(d_u[0], d_u[1], d_u[2]), xv = X(d_v[0], d_v[1], d_v[2]);
        const cplx xd = X(d_u[0] + d_v[0], d_u[1] + d_v[1], d_u[2] + d_v[2]);
        const cplx s = cmake(hb * (4.0 * xp.x + 2.0 * (xu.x + xv.x) + xd.x),
                             hb * (4.0 * xp.y + 2.0 * (xu.y + xv.y) + xd.y));
        ax.x += k * s.y;   // -i k s
        ax.y -= k * s.x;
      }
    }
  }
  return ax;
}

template <bool HET>
__device__ cplx diag3(const F3& P, const double2* cf, double2 kc, int gx, int gy, int gz) {
  const int n = P.n;
  const double h = P.h;
  const double hm8 = 8.0 * h * h * h / 216.0;
  cplx dg = cmake(0, 0);
  for (int o = 0; o < 8; ++o) {
    const int ex = gx - 1 + (o & 1), ey = gy - 1 + ((o >> 1) & 1), ez = gz - 1 + ((o >> 2) & 1);
    if (ex < 0 || ex >= n || ey < 0 || ey >= n || ez < 0 || ez >= n) continue;
    const double2 c = coef3<HET>(P, cf, kc, ex, ey, ez);
    dg.x += h / 3.0 - c.x * c.x * hm8;
    dg.y -= c.y * hm8;
  }
  const double hb4 = 4.0 * h * h / 36.0;
  for (int a = 0; a < 3; ++a) {
    const int ga = a == 0 ? gx : (a == 1 ? gy : gz);
    if (ga != 0 && ga != n) continue;
    const int ea = ga == 0 ? 0 : n - 1;
    const int u = (a + 1) % 3, v = (a + 2) % 3;
    const int gu = u == 0 ? gx : (u == 1 ? gy : gz);
    const int gv = v == 0 ? gx : (v == 1 ? gy : gz);
    for (int q = 0; q < 4; ++q) {
      const int eu = gu - 1 + (q & 1), ev = gv - 1 + ((q >> 1) & 1);
      if (eu < 0 || eu >= n || ev < 0 || ev >= n) continue;
      int e3[3];
      e3[a] = ea; e3[u] = eu; e3[v] = ev;
      dg.y -= coef3<HET>(P, cf, kc, e3[0], e3[1], e3[2]).x * hb4;
    }
  }
  return dg;
}

// y = A x  or  y = sub - A x
template <bool HET, bool EPS>
__global__ void __launch_bounds__(BX * BY) k_apply3d(F3 P, VArg x, VArg y, VArg sub) {
  int b, gx, gy, gz;
  int64_t vo;
  if (!node_of(P, b, gx, gy, gz, vo)) return;
  if (P.st && P.st[b]) return;
  const double2* cf = HET ? P.coef + b * P.coef_bs : nullptr;
  const double2 kc = HET ? make_double2(0, 0) : P.kc[b];
  cplx ax = row3<HET, EPS>(P, LdgAcc{x.at(b) - vo}, cf, kc, gx, gy, gz);
  const int64_t gi = ((int64_t)gz * P.N1 + gy) * P.N1 + gx;
  if (sub.p) ax = csub((sub.at(b) - vo)[gi], ax);
  (y.at(b) - vo)[gi] = ax;
}

// u_out = u + omega D^{-1} (f*fs - A_eps u)   (u == NULL: first step from zero)
template <bool HET>
__global__ void __launch_bounds__(BX * BY) k_jacobi3d(F3 P, VArg f, SArg fs, VArg u, VArg uo) {
  int b, gx, gy, gz;
  int64_t vo;
  if (!node_of(P, b, gx, gy, gz, vo)) return;
  if (P.st && P.st[b]) return;
  const double2* cf = HET ? P.coef + b * P.coef_bs : nullptr;
  const double2 kc = HET ? make_double2(0, 0) : P.kc[b];
  const int64_t gi = ((int64_t)gz * P.N1 + gy) * P.N1 + gx;
  const cplx fv = cscale(__ldg(&(f.at(b) - vo)[gi]), fs.at(b));
  const cplx di = (HET && P.dinv) ? __ldg(&(P.dinv + (int64_t)b * P.stride - vo)[gi])
                                  : cinv(diag3<HET>(P, cf, kc, gx, gy, gz));
  cplx v;
  if (u.p) {
    const cplx* ub = u.at(b) - vo;
    const cplx ax = row3<HET, true>(P, LdgAcc{ub}, cf, kc, gx, gy, gz);
    v = ub[gi];
    cfma(v, cscale(di, P.omega), csub(fv, ax));
  } else {
    v = cscale(cmul(di, fv), P.omega);
  }
  (uo.at(b) - vo)[gi] = v;
}

// r = f*fs - A_eps u  (fine residual)
template <bool HET>
__global__ void __launch_bounds__(BX * BY) k_resid3d(F3 P, VArg f, SArg fs, VArg u, VArg r) {
  int b, gx, gy, gz;
  int64_t vo;
  if (!node_of(P, b, gx, gy, gz, vo)) return;
  if (P.st && P.st[b]) return;
  const double2* cf = HET ? P.coef + b * P.coef_bs : nullptr;
  const double2 kc = HET ? make_double2(0, 0) : P.kc[b];
  const int64_t gi = ((int64_t)gz * P.N1 + gy) * P.N1 + gx;
  const cplx ax = row3<HET, true>(P, LdgAcc{u.at(b) - vo}, cf, kc, gx, gy, gz);
  (r.at(b) - vo)[gi] = csub(cscale(__ldg(&(f.at(b) - vo)[gi]), fs.at(b)), ax);
}

// rc = I^T r  (one thread per OWNED coarse node: coarse plane cz with 2 cz in [z0, z1))
__global__ void __launch_bounds__(BX * BY) k_restrict3d(F3 P, int cspan, VArg r, VArg rc) {
  const int n = P.n, nc = n / 2, NC1 = nc + 1, N1 = n + 1;
  const int cx = blockIdx.x * BX + threadIdx.x, cy = blockIdx.y * BY + threadIdx.y;
  const int b = blockIdx.z / cspan;
  const int2 sl = slab_of(P.slab, b, n);
  const int cz = sl.x / 2 + (int)(blockIdx.z % cspan);
  if (cx > nc || cy > nc || 2 * cz >= sl.y) return;
  if (P.st && P.st[b]) return;
  const cplx* rb = r.at(b) - (int64_t)(sl.x - P.G) * N1 * N1;
  cplx acc = cmake(0, 0);
  for (int dz = -1; dz <= 1; ++dz) {
    const int gz = 2 * cz + dz;
    if (gz < 0 || gz > n) continue;
    for (int dy = -1; dy <= 1; ++dy) {
      const int gy = 2 * cy + dy;
      if (gy < 0 || gy > n) continue;
      for (int dx = -1; dx <= 1; ++dx) {
        const int gx = 2 * cx + dx;
        if (gx < 0 || gx > n) continue;
        const double w = (dx ? 0.5 : 1.0) * (dy ? 0.5 : 1.0) * (dz ? 0.5 : 1.0);
        const cplx v = __ldg(&rb[((int64_t)gz * N1 + gy) * N1 + gx]);
        acc.x += w * v.x;
        acc.y += w * v.y;
      }
    }
  }
  rc.at(b)[((int64_t)cz * NC1 + cy) * NC1 + cx] = acc;
}

// uo = u + I ec
__global__ void __launch_bounds__(BX * BY) k_prolong3d(F3 P, VArg u, VArg ec, VArg uo) {
  const int n = P.n, N1 = n + 1, NC1 = n / 2 + 1;
  int b, gx, gy, gz;
  int64_t vo;
  if (!node_of(P, b, gx, gy, gz, vo)) return;
  if (P.st && P.st[b]) return;
  const cplx* e = ec.at(b);
  const int64_t gi = ((int64_t)gz * N1 + gy) * N1 + gx;
  cplx v = (u.at(b) - vo)[gi];
  const int cx0 = gx >> 1, cy0 = gy >> 1, cz0 = gz >> 1;
  for (int k = 0; k <= (gz & 1); ++k)
    for (int j = 0; j <= (gy & 1); ++j)
      for (int i = 0; i <= (gx & 1); ++i) {
        const double w = ((gx & 1) ? 0.5 : 1.0) * ((gy & 1) ? 0.5 : 1.0) * ((gz & 1) ? 0.5 : 1.0);
        const cplx c = __ldg(&e[((int64_t)(cz0 + k) * NC1 + cy0 + j) * NC1 + cx0 + i]);
        v.x += w * c.x;
        v.y += w * c.y;
      }
  (uo.at(b) - vo)[gi] = v;
}

// D^{-1} at every stored node of every entry (het setup)
template <bool HET>
__global__ void __launch_bounds__(BX * BY) k_dinv3d(F3 P, cplx* __restrict__ dinv) {
  int b, gx, gy, gz;
  int64_t vo;
  if (!node_of(P, b, gx, gy, gz, vo)) return;
  const double2* cf = HET ? P.coef + b * P.coef_bs : nullptr;
  const double2 kc = HET ? make_double2(0, 0) : P.kc[b];
  const int64_t gi = ((int64_t)gz * P.N1 + gy) * P.N1 + gx;
  (dinv + (int64_t)b * P.stride - vo)[gi] = cinv(diag3<HET>(P, cf, kc, gx, gy, gz));
}

// coarse stencil: st[b][node*27 + (dx+1) + 3(dy+1) + 9(dz+1)]
template <bool HET>
__global__ void k_stencil3d(F3 P, cplx* __restrict__ stv) {
  int b, gx, gy, gz;
  int64_t vo;
  if (!node_of(P, b, gx, gy, gz, vo)) return;
  const int n = P.n, N1 = P.N1;
  const double h = P.h;
  const double2* cf = HET ? P.coef + b * P.coef_bs : nullptr;
  const double2 kc = HET ? make_double2(0, 0) : P.kc[b];
  const int64_t node = ((int64_t)gz * N1 + gy) * N1 + gx;
  cplx* st = stv + ((int64_t)b * N1 * N1 * N1 + node) * 27;
  cplx e[27];
  for (int o = 0; o < 27; ++o) e[o] = cmake(0, 0);
  const double hk = h / 36.0, hm = h * h * h / 216.0;
  for (int o = 0; o < 8; ++o) {
    const int dx = (o & 1) ? 1 : -1, dy = (o & 2) ? 1 : -1, dz = (o & 4) ? 1 : -1;
    const int ex = gx + (dx < 0 ? -1 : 0), ey = gy + (dy < 0 ? -1 : 0), ez = gz + (dz < 0 ? -1 : 0);
    if (ex < 0 || ex >= n || ey < 0 || ey >= n || ez < 0 || ez >= n) continue;
    const double2 c = coef3<HET>(P, cf, kc, ex, ey, ez);
    const cplx lam = cmake(c.x * c.x, c.y);
    // the 8 nodes of this element relative to the node: offsets in {0, d}^3
    for (int m = 0; m < 8; ++m) {
      const int ox = (m & 1) ? dx : 0, oy = (m & 2) ? dy : 0, oz = (m & 4) ? dz : 0;
      const int cls = (ox != 0) + (oy != 0) + (oz != 0);
      const double kv = hk * (cls == 0 ? 12.0 : (cls == 1 ? 0.0 : -3.0));
      const double mv = hm * (cls == 0 ? 8.0 : (cls == 1 ? 4.0 : (cls == 2 ? 2.0 : 1.0)));
      const int idx = (ox + 1) + 3 * (oy + 1) + 9 * (oz + 1);
      e[idx].x += kv - lam.x * mv;
      e[idx].y -= lam.y * mv;
    }
  }
  const double hb = h * h / 36.0;
  const int g3[3] = {gx, gy, gz};
  for (int a = 0; a < 3; ++a) {
    if (g3[a] != 0 && g3[a] != n) continue;
    const int ea = g3[a] == 0 ? 0 : n - 1;
    const int u = (a + 1) % 3, v = (a + 2) % 3;
    for (int q = 0; q < 4; ++q) {
      const int du = (q & 1) ? 1 : -1, dv = (q & 2) ? 1 : -1;
      const int eu = g3[u] + (du < 0 ? -1 : 0), ev = g3[v] + (dv < 0 ? -1 : 0);
      if (eu < 0 || eu >= n || ev < 0 || ev >= n) continue;
      int e3[3];
      e3[a] = ea; e3[u] = eu; e3[v] = ev;
      const double k = coef3<HET>(P, cf, kc, e3[0], e3[1], e3[2]).x;
      for (int m = 0; m < 4; ++m) {
        int off[3] = {0, 0, 0};
        if (m & 1) off[u] = du;
        if (m & 2) off[v] = dv;
        const int cls = (m & 1) + ((m >> 1) & 1);
        const double bv = hb * (cls == 0 ? 4.0 : (cls == 1 ? 2.0 : 1.0));
        const int idx = (off[0] + 1) + 3 * (off[1] + 1) + 9 * (off[2] + 1);
        e[idx].y -= k * bv;
      }
    }
  }
  for (int o = 0; o < 27; ++o) st[o] = e[o];
}

// ------------------------------------------------------------ z-marching kernels
// 2.5D tiles: a CTA owns a 32 x 8 column tile of nodes of one entry and marches
// through a range of z planes.  The input field x (with a 1-node halo in x, y) is
// staged plane by plane in a 4-plane shared-memory ring, the element
// coefficients (k_e, eps_e) in a 3-plane ring; the next plane's global loads are
// issued into registers before the current plane is computed (one barrier per
// plane), so load latency overlaps the arithmetic.
//
// Interior nodes use the assembled forms, evaluated with in-plane pair sums:
// per plane z' the centre c, the 4 edge-adjacent e, the 4 diagonal d values and
// the quadrant sums P(sx,sy) = 4c + 2x(sx) + 2y(sy) + xy(sx,sy);
//   K u   = 8h/3 c_z - h/6 (d_z + e_{z-1} + e_{z+1}) - h/12 (d_{z-1} + d_{z+1})
//   M_l u = h^3/216 sum_q [2 (lb_q + la_q) P_z(q) + lb_q P_{z-1}(q) + la_q P_{z+1}(q)]
// (lb / la: lambda of the quadrant-q element below / above the node plane; a
// constant lambda gives the assembled mass 64 / 16 / 4 / 1), D = 8h/3 -
// h^3/27 sum_e lambda_e computed on the fly.  Boundary nodes take the element
// loop (+ boundary faces) on the staged values.  (SURVEY.md 8(d) kernel notes.)
constexpr int MTX = 32, MTY = 8, MT = MTX * MTY;
constexpr int NPX = MTX + 2, NPY = MTY + 2, NPL = NPX * NPY;   // node plane with halo
constexpr int EPX = MTX + 1, EPY = MTY + 1, EPL = EPX * EPY;   // element plane
constexpr int NRING = 4, ERING = 3;

// 16-byte asynchronous global -> shared copy (zero-fill when !valid)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
enum { M_APPLY = 0, M_JAC = 1, M_JACP = 2, M_RES = 3 };

struct MarchSmem {
  cplx u[NRING][NPL];
  double2 c[ERING][EPL];
};

// Interior nodes only (x, y, z in 1..n-1): the tiles start at x0 = 1 + 32 i,
// y0 = 1 + 8 j and march the interior planes of the entry's range; the domain
// boundary faces (2-3% of the nodes: the absorbing-boundary terms and the
// partial element sets) are computed by k_bnd3d below.
template <bool HET, int MODE, int MINB>
__global__ void __launch_bounds__(MT, MINB) k_march3d(F3 P, VArg x, VArg f, SArg fs, VArg ec, VArg sub, VArg out,
                                                     int eps, int zlen, int nzc) {
  extern __shared__ double4 smem_raw[];
  MarchSmem& S = *reinterpret_cast<MarchSmem*>(smem_raw);
  const int n = P.n, N1 = P.N1;
  const int tid = threadIdx.x, tx = tid % MTX, ty = tid / MTX;
  const int x0 = 1 + blockIdx.x * MTX, y0 = 1 + blockIdx.y * MTY;
  const int b = blockIdx.z / nzc, chunk = blockIdx.z % nzc;
  if (P.st && P.st[b]) return;
  const int2 sl = slab_of(P.slab, b, n);
  const int zlo = max(1, sl.x - P.ext), zhi = min(n, sl.y + P.ext);   // interior planes
  const int zs = zlo + chunk * zlen, ze = min(zhi, zs + zlen);
  if (zs >= ze) return;
  const int64_t vo = (int64_t)(sl.x - P.G) * N1 * N1;
  const cplx* xb = x.at(b) - vo;
  const double2* cf = HET ? P.coef + b * P.coef_bs : nullptr;
  const double2 kc = HET ? make_double2(0, 0) : P.kc[b];
  const int NC1 = n / 2 + 1;
  const cplx* eb = MODE == M_JACP ? ec.at(b) : nullptr;
  // ---- staging: node plane gz (x or x + I e_c) and element plane ez.  Every
  // thread stages the same <= 2 node / element slots of each plane: their plane
  // offsets are computed once, so a plane costs one 64-bit add per load.
  const int64_t NN = (int64_t)N1 * N1, EE = (int64_t)n * n;
  int64_t noff[2], eoff[2];
  int ngx[2], ngy[2];
  bool nok[2], eok[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int q = tid + k * MT;
    const int qx = q % NPX, qy = q / NPX;
    ngx[k] = x0 - 1 + qx;
    ngy[k] = y0 - 1 + qy;
    nok[k] = q < NPL && ngx[k] <= n && ngy[k] <= n;   // >= 0 by construction
    noff[k] = (int64_t)ngy[k] * N1 + ngx[k];
    const int ex = x0 - 1 + q % EPX, ey = y0 - 1 + q / EPX;
    eok[k] = HET && q < EPL && ex < n && ey < n;
    eoff[k] = (int64_t)ey * n + ex;
  }
  cplx rn[2];
  double2 rc[2];
  auto fetch = [&](int gz, int ez) {
    const cplx* xp = xb + gz * NN;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      rn[k] = cmake(0, 0);
      if (nok[k]) {
        cplx v = __ldg(xp + noff[k]);
        if (MODE == M_JACP) {   // trilinear prolongation of the coarse correction (Alg. 1 line 4)
          const int gx = ngx[k], gy = ngy[k];
          const int cx0 = gx >> 1, cy0 = gy >> 1, cz0 = gz >> 1;
          const double w = ((gx & 1) ? 0.5 : 1.0) * ((gy & 1) ? 0.5 : 1.0) * ((gz & 1) ? 0.5 : 1.0);
          for (int kk = 0; kk <= (gz & 1); ++kk)
            for (int j = 0; j <= (gy & 1); ++j)
              for (int i = 0; i <= (gx & 1); ++i) {
                const cplx c = __ldg(&eb[((int64_t)(cz0 + kk) * NC1 + cy0 + j) * NC1 + cx0 + i]);
                v.x += w * c.x;
                v.y += w * c.y;
              }
        }
        rn[k] = v;
      }
      if (HET) rc[k] = eok[k] ? __ldg(cf + ez * EE + eoff[k]) : make_double2(0, 0);
    }
  };
  auto commit = [&](cplx* un, double2* ce) {   // -> node plane slot un, element plane slot ce
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int q = tid + k * MT;
      if (q < NPL) un[q] = rn[k];
      if (HET && q < EPL) ce[q] = rc[k];
    }
  };
  // Asynchronous staging (every mode but JACP, whose staged values need the
  // prolongation added): cp.async copies global -> shared directly (no
  // registers), out-of-range slots are zero-filled (src-size 0).
  constexpr bool ASYNC = MODE != M_JACP;
  auto issue = [&](int gz, int ez, cplx* un, double2* ce, bool elem) {
    const cplx* xp = xb + gz * NN;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int q = tid + k * MT;
      if (q < NPL) cp_async16(&un[q], nok[k] ? xp + noff[k] : xb, nok[k]);
      if (HET && elem && q < EPL) cp_async16(&ce[q], eok[k] ? cf + ez * EE + eoff[k] : cf, eok[k]);
    }
    cp_async_commit();
  };
  // ring slots (rotated, no modulo in the loop): node planes t-1, t, t+1, t+2;
  // element planes t-1, t, t+1
  cplx* Un[NRING] = {S.u[0], S.u[1], S.u[2], S.u[3]};
  double2* Ce[ERING] = {S.c[0], S.c[1], S.c[2]};
  // prologue: node planes zs - 1, zs and element plane zs - 1 in shared memory,
  // node plane zs + 1 / element plane zs in flight (registers or cp.async)
  if (ASYNC) {
    issue(zs - 1, zs - 1, Un[0], Ce[0], true);
    issue(zs, zs, Un[1], Ce[0], false);
    issue(zs + 1, zs, Un[2], Ce[1], true);
  } else {
    fetch(zs - 1, zs - 1);
    commit(Un[0], Ce[0]);
    fetch(zs, zs);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int q = tid + k * MT;
      if (q < NPL) Un[1][q] = rn[k];
    }
    fetch(zs + 1, zs);
  }
  const int gx = x0 + tx, gy = y0 + ty;
  const bool act = gx < n && gy < n;
  const double h = P.h, hm = h * h * h / 216.0;
  const double kc0 = 8.0 * h / 3.0, ke = -h / 6.0, kk = -h / 12.0;
  const int ci = (ty + 1) * NPX + tx + 1;    // this node in a node plane
  const int e0 = ty * EPX + tx;              // element (gx - 1, gy - 1) in an element plane
  const cplx lamc = HET ? cmake(0, 0) : cmake(kc.x * kc.x, eps ? kc.y : 0.0);
  // Per node plane z: centre c, K_in = 8h/3 c - h/6 d (its role as the node's own
  // plane), K_off = -h/6 e - h/12 d (as the plane above / below); HET: quadrant
  // sums P(q); constant k: the mass folded in (A_in / A_off).
  struct PlaneQ { cplx c, kin, koff, Pq[4]; };
  auto planeq = [&](const cplx* U, PlaneQ& Q) {
    const cplx c = U[ci], xm = U[ci - 1], xp = U[ci + 1], ym = U[ci - NPX], yp = U[ci + NPX];
    const cplx mm = U[ci - NPX - 1], pm = U[ci - NPX + 1], mp = U[ci + NPX - 1], pp = U[ci + NPX + 1];
    const cplx e = cmake(xm.x + xp.x + ym.x + yp.x, xm.y + xp.y + ym.y + yp.y);
    const cplx d = cmake(mm.x + pm.x + mp.x + pp.x, mm.y + pm.y + mp.y + pp.y);
    Q.c = c;
    Q.kin = cmake(kc0 * c.x + ke * d.x, kc0 * c.y + ke * d.y);
    Q.koff = cmake(ke * e.x + kk * d.x, ke * e.y + kk * d.y);
    if (HET) {   // quadrants q = (sx > 0) + 2 (sy > 0)
      Q.Pq[0] = cmake(4 * c.x + 2 * (xm.x + ym.x) + mm.x, 4 * c.y + 2 * (xm.y + ym.y) + mm.y);
      Q.Pq[1] = cmake(4 * c.x + 2 * (xp.x + ym.x) + pm.x, 4 * c.y + 2 * (xp.y + ym.y) + pm.y);
      Q.Pq[2] = cmake(4 * c.x + 2 * (xm.x + yp.x) + mp.x, 4 * c.y + 2 * (xm.y + yp.y) + mp.y);
      Q.Pq[3] = cmake(4 * c.x + 2 * (xp.x + yp.x) + pp.x, 4 * c.y + 2 * (xp.y + yp.y) + pp.y);
    } else {
      const cplx in = cmake(64 * c.x + 16 * e.x + 4 * d.x, 64 * c.y + 16 * e.y + 4 * d.y);
      const cplx of = cmake(16 * c.x + 4 * e.x + d.x, 16 * c.y + 4 * e.y + d.y);
      cfms(Q.kin, cscale(lamc, hm), in);
      cfms(Q.koff, cscale(lamc, hm), of);
    }
  };
  // element plane ez (between node planes ez, ez + 1), HET: mass of the lower node
  // (weights 2 P_lo + P_hi), of the upper node (2 P_hi + P_lo), and sum of lambda
  auto eplane = [&](const double2* C, const cplx* Plo, const cplx* Phi, cplx& mlo, cplx& mhi, cplx& ls) {
    mlo = mhi = ls = cmake(0, 0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 cq = C[e0 + (q & 1) + (q >> 1) * EPX];
      const cplx l = cmake(cq.x * cq.x, eps ? cq.y : 0.0);
      ls = cadd(ls, l);
      cfma(mlo, l, cmake(2 * Plo[q].x + Phi[q].x, 2 * Plo[q].y + Phi[q].y));
      cfma(mhi, l, cmake(2 * Phi[q].x + Plo[q].x, 2 * Phi[q].y + Plo[q].y));
    }
  };
  // f (or sub) of this node at plane t, loaded one plane ahead
  const cplx* fb = MODE != M_APPLY ? f.at(b) - vo : (sub.p ? sub.at(b) - vo : nullptr);
  const int64_t nodeoff = (int64_t)gy * N1 + gx;
  const cplx* fp = (act && fb) ? fb + zs * NN + nodeoff : nullptr;   // advanced by one plane per step
  const double fsc = MODE != M_APPLY ? fs.at(b) : 1.0;
  cplx fnext = fp ? __ldg(fp) : cmake(0, 0);
  // carried along z: node t's partial operator row acc and its lambda sum below;
  // plane t's P, K_off (const: A_off) and centre
  cplx acc = cmake(0, 0), lsb = cmake(0, 0), koff_t = cmake(0, 0), c_t = cmake(0, 0);
  cplx Pt[4] = {cmake(0, 0), cmake(0, 0), cmake(0, 0), cmake(0, 0)};
  cplx* op = out.at(b) - vo + zs * NN + nodeoff;
  for (int t = zs; t < ze; ++t, op += NN) {
    // slots this step: node planes t-1 = Un[0], t = Un[1], t+1 = Un[2] (being
    // committed), t+2 = Un[3] (next); element planes t-1 = Ce[0], t = Ce[1]
    if (ASYNC) {
      cp_async_wait_all();         // node plane t + 1, element plane t landed
      __syncthreads();
      if (t + 2 <= ze) issue(t + 2, t + 1, Un[3], Ce[2], true);
    } else {
      commit(Un[2], Ce[1]);        // node plane t + 1, element plane t
      __syncthreads();
      if (t + 2 <= ze) fetch(t + 2, t + 1);
    }
    const cplx fcur = fnext;
    if (fp && t + 1 < ze) {
      fp += NN;
      fnext = __ldg(fp);
    }
    if (act) {
      if (t == zs) {   // start of the march: planes zs - 1, zs and element plane zs - 1
        PlaneQ Qm, Q0;
        planeq(Un[0], Qm);
        planeq(Un[1], Q0);
        acc = cadd(Q0.kin, Qm.koff);
        if (HET) {
          cplx mlo, mhi, ls;
          eplane(Ce[0], Qm.Pq, Q0.Pq, mlo, mhi, ls);
          cfms(acc, cmake(hm, 0), mhi);
          lsb = ls;
#pragma unroll
          for (int q = 0; q < 4; ++q) Pt[q] = Q0.Pq[q];
        }
        koff_t = Q0.koff;
        c_t = Q0.c;
      }
      PlaneQ Q1;
      planeq(Un[2], Q1);
      cplx ax = cadd(acc, Q1.koff), dg;
      const cplx xc = c_t;
      if (HET) {
        cplx mlo, mhi, ls;
        eplane(Ce[1], Pt, Q1.Pq, mlo, mhi, ls);
        cfms(ax, cmake(hm, 0), mlo);
        dg = cmake(kc0 - 8.0 * hm * (lsb.x + ls.x), -8.0 * hm * (lsb.y + ls.y));
        acc = cadd(Q1.kin, koff_t);        // node t + 1
        cfms(acc, cmake(hm, 0), mhi);
        lsb = ls;
#pragma unroll
        for (int q = 0; q < 4; ++q) Pt[q] = Q1.Pq[q];
      } else {
        dg = cmake(kc0 - 64.0 * hm * lamc.x, -64.0 * hm * lamc.y);
        acc = cadd(Q1.kin, koff_t);
      }
      koff_t = Q1.koff;
      c_t = Q1.c;
      if (MODE == M_APPLY) {
        *op = fb ? csub(fcur, ax) : ax;
      } else {
        const cplx r = csub(cscale(fcur, fsc), ax);
        if (MODE == M_RES) {
          *op = r;
        } else {
          cplx v = xc;
          cfma(v, cscale(cinv(dg), P.omega), r);
          *op = v;
        }
      }
    }
    // rotate the rings
    cplx* u0 = Un[0];
    Un[0] = Un[1]; Un[1] = Un[2]; Un[2] = Un[3]; Un[3] = u0;
    double2* c0 = Ce[0];
    Ce[0] = Ce[1]; Ce[1] = Ce[2]; Ce[2] = c0;
  }
}

// Domain-boundary nodes of the marching kernels' operations: planes z = 0, n
// entirely, the perimeter of every other plane of the entry's range; one thread
// per node, the element loop + boundary faces of row3 / diag3 from global memory.
template <bool HET, int MODE, bool EPS>
__global__ void __launch_bounds__(256) k_bnd3d(F3 P, VArg x, VArg f, SArg fs, VArg ec, VArg sub, VArg out) {
  const int n = P.n, N1 = P.N1;
  const int b = blockIdx.z;
  if (P.st && P.st[b]) return;
  const int2 sl = slab_of(P.slab, b, n);
  const int zlo = max(0, sl.x - P.ext), zhi = min(N1, sl.y + P.ext);
  // flattened: the perimeters (4n nodes) of all planes of the range, then the
  // interiors ((n-1)^2 nodes) of the planes z = 0 and z = n if in the range
  const int span = zhi - zlo, per = 4 * n, in2 = (n - 1) * (n - 1);
  const bool f0 = zlo == 0, f1 = zhi == N1;
  const int64_t total = (int64_t)span * per + (int64_t)((f0 ? 1 : 0) + (f1 ? 1 : 0)) * in2;
  const int64_t vo = (int64_t)(sl.x - P.G) * N1 * N1;
  const double2* cf = HET ? P.coef + b * P.coef_bs : nullptr;
  const double2 kc = HET ? make_double2(0, 0) : P.kc[b];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int gx, gy, z;
    if (i < (int64_t)span * per) {   // perimeter: (r, 0), (n, r), (n - r, n), (0, n - r), r in 0..n-1
      z = zlo + (int)(i / per);
      const int j = (int)(i % per), side = j / n, r = j % n;
      gx = side == 0 ? r : (side == 1 ? n : (side == 2 ? n - r : 0));
      gy = side == 0 ? 0 : (side == 1 ? r : (side == 2 ? n : n - r));
    } else {
      const int64_t j = i - (int64_t)span * per;
      z = (j < in2 && f0) ? 0 : n;
      const int r = (int)(j % in2);
      gx = 1 + r % (n - 1);
      gy = 1 + r / (n - 1);
    }
    const int64_t gi = ((int64_t)z * N1 + gy) * N1 + gx;
    cplx ax, xc;
    if (MODE == M_JACP) {
      const ProlongAcc acc{x.at(b) - vo, ec.at(b), n / 2 + 1};
      ax = row3<HET, EPS>(P, acc, cf, kc, gx, gy, z);
      xc = acc(gi, gx, gy, z);
    } else {
      const LdgAcc acc{x.at(b) - vo};
      ax = row3<HET, EPS>(P, acc, cf, kc, gx, gy, z);
      xc = acc(gi, gx, gy, z);
    }
    cplx* ob = out.at(b) - vo;
    if (MODE == M_APPLY) {
      ob[gi] = sub.p ? csub(__ldg(&(sub.at(b) - vo)[gi]), ax) : ax;
    } else {
      const cplx r = csub(cscale(__ldg(&(f.at(b) - vo)[gi]), fs.at(b)), ax);
      if (MODE == M_RES) {
        ob[gi] = r;
      } else {
        cplx v = xc;
        cfma(v, cscale(cinv(diag3<HET>(P, cf, kc, gx, gy, z)), P.omega), r);
        ob[gi] = v;
      }
    }
  }
}

// Pointwise steps as streaming kernels (grid-stride over the entry's planes, two
// nodes in flight per thread): MODE 0 = the first Jacobi step from u = 0,
// uo = omega D^{-1} f fs (D^{-1}: the precomputed copy (heterogeneous), the
// interior constant / diag3 at the boundary (constant k)); MODE 1 = prolongation
// and correction uo = u + I e_c.
template <bool HET, int MODE>
__global__ void __launch_bounds__(256) k_pw3d(F3 P, VArg f, SArg fs, VArg u, VArg ec, VArg uo) {
  const int n = P.n, N1 = P.N1;
  const int b = blockIdx.y;
  if (P.st && P.st[b]) return;
  const int2 sl = slab_of(P.slab, b, n);
  const int zlo = max(0, sl.x - P.ext), zhi = min(N1, sl.y + P.ext);
  const int64_t NN = (int64_t)N1 * N1, i0 = zlo * NN, i1 = zhi * NN;
  const int64_t vo = (int64_t)(sl.x - P.G) * NN;
  cplx* ob = uo.at(b) - vo;
  const double2* cf = HET ? P.coef + b * P.coef_bs : nullptr;
  const double2 kc = HET ? make_double2(0, 0) : P.kc[b];
  const int NC1 = n / 2 + 1;
  const cplx* fb = MODE == 0 ? f.at(b) - vo : nullptr;
  const double fsc = MODE == 0 ? fs.at(b) : 1.0;
  const cplx* ub = MODE == 1 ? u.at(b) - vo : nullptr;
  const cplx* eb = MODE == 1 ? ec.at(b) : nullptr;
  const cplx* dib = (MODE == 0 && HET) ? P.dinv + (int64_t)b * P.stride - vo : nullptr;
  const double hm = P.h * P.h * P.h / 216.0;
  const cplx di_int = HET ? cmake(0, 0)   // constant k: interior D = 8h/3 - 64 h^3/216 lambda
                          : cinv(cmake(8.0 * P.h / 3.0 - 64.0 * hm * kc.x * kc.x, -64.0 * hm * kc.y));
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < i1; i += 2 * step) {
    const int64_t j = i + step;
    const bool two = j < i1;
    if (MODE == 0) {
      const cplx f0 = __ldg(&fb[i]), f1 = two ? __ldg(&fb[j]) : cmake(0, 0);
      cplx d0, d1;
      if (HET) {
        d0 = __ldg(&dib[i]);
        d1 = two ? __ldg(&dib[j]) : cmake(0, 0);
      } else {
        auto dg = [&](int64_t k) {
          const int gx = (int)(k % N1), gy = (int)((k / N1) % N1), gz = (int)(k / NN);
          const bool inter = gx > 0 && gx < n && gy > 0 && gy < n && gz > 0 && gz < n;
          return inter ? di_int : cinv(diag3<false>(P, nullptr, kc, gx, gy, gz));
        };
        d0 = dg(i);
        d1 = two ? dg(j) : cmake(0, 0);
      }
      ob[i] = cscale(cmul(d0, cscale(f0, fsc)), P.omega);
      if (two) ob[j] = cscale(cmul(d1, cscale(f1, fsc)), P.omega);
    } else {
      const cplx u0 = __ldg(&ub[i]), u1 = two ? __ldg(&ub[j]) : cmake(0, 0);
      auto pro = [&](int64_t k, cplx v) {
        const int gx = (int)(k % N1), gy = (int)((k / N1) % N1), gz = (int)(k / NN);
        const int cx0 = gx >> 1, cy0 = gy >> 1, cz0 = gz >> 1;
        const double w = ((gx & 1) ? 0.5 : 1.0) * ((gy & 1) ? 0.5 : 1.0) * ((gz & 1) ? 0.5 : 1.0);
        for (int kk = 0; kk <= (gz & 1); ++kk)
          for (int jj = 0; jj <= (gy & 1); ++jj)
            for (int ii = 0; ii <= (gx & 1); ++ii) {
              const cplx c = __ldg(&eb[((int64_t)(cz0 + kk) * NC1 + cy0 + jj) * NC1 + cx0 + ii]);
              v.x += w * c.x;
              v.y += w * c.y;
            }
        return v;
      };
      ob[i] = pro(i, u0);
      if (two) ob[j] = pro(j, u1);
    }
  }
}

template <bool HET, int MODE>
static hh_status pw3(const F3& P, int B, VArg f, SArg fs, VArg u, VArg ec, VArg uo, cudaStream_t s) {
  const int64_t nodes = (int64_t)std::min(P.N1, P.maxloc + 2 * P.ext) * P.N1 * P.N1;
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(148 * 8 / std::max(1, B) + 1, (nodes + 511) / 512));
  k_pw3d<HET, MODE><<<dim3(gx, B), 256, 0, s>>>(P, f, fs, u, ec, uo);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

F3 make3(const Level& L, double omega, const int* st, int ext) {
  F3 P;
  P.n = L.n; P.h = L.h; P.omega = omega; P.coef = L.coef; P.coef_bs = L.coef_bs; P.kc = L.kc;
  P.st = st; P.N1 = L.n + 1;
  P.slab = L.slab; P.G = L.G; P.maxloc = L.maxloc; P.ext = ext;
  P.dinv = L.dinv; P.stride = L.stride;
  return P;
}
dim3 grid3(const F3& P, int B) {
  return dim3((P.N1 + BX - 1) / BX, (P.N1 + BY - 1) / BY, (P.maxloc + 2 * P.ext) * B);
}

}  // namespace

// z-marching launch: CTAs per entry = x tiles x y tiles x z chunks, with enough
// z chunks to put ~4 CTAs on every SM
static bool g_march = getenv("HH_3D_NAIVE") == nullptr;   // HH_3D_NAIVE=1: the one-node-per-thread kernels
// side stream of the boundary-face kernel (runs beside the marching kernel:
// disjoint nodes), one per device; the fork / join sequence is serialised so
// concurrent callers never interleave their event records
struct Side { cudaStream_t s = nullptr; cudaEvent_t a = nullptr, b = nullptr; };
static std::mutex g_side_mu;
static hh_status side_of(Side** out) {
  static std::map<int, Side> sides;
  int dev = 0;
  HH_CUDA_TRY(cudaGetDevice(&dev));
  Side& sd = sides[dev];
  if (!sd.s) {
    HH_CUDA_TRY(cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking));
    HH_CUDA_TRY(cudaEventCreateWithFlags(&sd.a, cudaEventDisableTiming));
    HH_CUDA_TRY(cudaEventCreateWithFlags(&sd.b, cudaEventDisableTiming));
  }
  *out = &sd;
  return HH_OK;
}
static const bool g_side = getenv("HH_3D_NOSIDE") == nullptr;

template <int MODE>
static hh_status march3(const Level& L, const F3& P, int B, VArg x, VArg f, SArg fs, VArg ec, VArg sub, VArg out,
                        bool eps, cudaStream_t s) {
  std::unique_lock<std::mutex> lk(g_side_mu, std::defer_lock);
  Side* sd = nullptr;
  cudaStream_t sb = s;   // stream of the boundary-face kernel
  if (g_side) {
    lk.lock();
    HH_TRY(side_of(&sd));
    HH_CUDA_TRY(cudaEventRecord(sd->a, s));
    HH_CUDA_TRY(cudaStreamWaitEvent(sd->s, sd->a, 0));
    sb = sd->s;
  }
  const int ni = P.n - 1;   // interior nodes per side
  const int tx = (ni + MTX - 1) / MTX, ty = (ni + MTY - 1) / MTY;
  const int span = std::min(P.N1, P.maxloc + 2 * P.ext);
  // register budget: 3 CTAs per SM (80 registers) or 2 (128); HH_3D_MINB selects,
  // default = the measured faster one
  static const int minb_env = getenv("HH_3D_MINB") ? atoi(getenv("HH_3D_MINB")) : 0;
  const int minb = minb_env ? minb_env : (L.het ? 2 : 3);   // spill-free budgets
  // z-chunks per column of tiles: the count whose launch takes the fewest plane
  // steps, rounds of resident CTAs (sms * minb slots) x (planes per chunk + the
  // 3 planes a chunk stages before its first output), instead of ">= 4 CTAs per
  // SM" (cfg3: 5 chunks = 640 CTAs = 1.44 rounds of 444 slots -> 3 chunks = 384
  // CTAs in one round).  HH_3D_NZC forces a count, HH_3D_NZC_OLD=1 the old rule.
  static const int nzc_env = getenv("HH_3D_NZC") ? atoi(getenv("HH_3D_NZC")) : 0;
  static const bool nzc_old = getenv("HH_3D_NZC_OLD") && atoi(getenv("HH_3D_NZC_OLD")) != 0;
  static const int sms = [] {
    int d = 0, n = 0;
    if (cudaGetDevice(&d) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || n <= 0) n = 148;
    return n;
  }();
  int nzc;
  if (nzc_env > 0) {
    nzc = std::min(span, nzc_env);
  } else if (nzc_old) {
    const int want = std::max(1, (4 * 148 + tx * ty * B - 1) / (tx * ty * B));
    nzc = std::max(1, std::min(span, want));
  } else {
    const int64_t tiles = (int64_t)tx * ty * B, slots = (int64_t)sms * minb;
    int64_t best = INT64_MAX;
    nzc = 1;
    for (int c = 1; c <= std::min(span, 32); ++c) {
      const int64_t rounds = (tiles * c + slots - 1) / slots;
      const int64_t cost = rounds * ((span + c - 1) / c + 3);
      if (cost < best) { best = cost; nzc = c; }
    }
  }
  const int zlen = (span + nzc - 1) / nzc;
  const size_t sm = sizeof(MarchSmem);
  const dim3 g(tx, ty, nzc * B);
  const int e = eps ? 1 : 0;
  if (L.het && minb == 2) {
    HH_CUDA_TRY(smem_attr((const void*)k_march3d<true, MODE, 2>, sm));
    k_march3d<true, MODE, 2><<<g, MT, sm, s>>>(P, x, f, fs, ec, sub, out, e, zlen, nzc);
  } else if (L.het) {
    HH_CUDA_TRY(smem_attr((const void*)k_march3d<true, MODE, 3>, sm));
    k_march3d<true, MODE, 3><<<g, MT, sm, s>>>(P, x, f, fs, ec, sub, out, e, zlen, nzc);
  } else if (minb == 2) {
    HH_CUDA_TRY(smem_attr((const void*)k_march3d<false, MODE, 2>, sm));
    k_march3d<false, MODE, 2><<<g, MT, sm, s>>>(P, x, f, fs, ec, sub, out, e, zlen, nzc);
  } else {
    HH_CUDA_TRY(smem_attr((const void*)k_march3d<false, MODE, 3>, sm));
    k_march3d<false, MODE, 3><<<g, MT, sm, s>>>(P, x, f, fs, ec, sub, out, e, zlen, nzc);
  }
  HH_CUDA_TRY(cudaGetLastError());
  // the boundary faces (side stream, disjoint nodes), joined back into s
  const int64_t nb = (int64_t)span * 4 * P.n + 2LL * (P.n - 1) * (P.n - 1);   // boundary nodes per entry (max)
  const dim3 gb((unsigned)std::max<int64_t>(1, std::min<int64_t>(2048, (nb + 255) / 256)), 1, B);
  if (L.het) {
    if (eps) k_bnd3d<true, MODE, true><<<gb, 256, 0, sb>>>(P, x, f, fs, ec, sub, out);
    else k_bnd3d<true, MODE, false><<<gb, 256, 0, sb>>>(P, x, f, fs, ec, sub, out);
  } else {
    if (eps) k_bnd3d<false, MODE, true><<<gb, 256, 0, sb>>>(P, x, f, fs, ec, sub, out);
    else k_bnd3d<false, MODE, false><<<gb, 256, 0, sb>>>(P, x, f, fs, ec, sub, out);
  }
  HH_CUDA_TRY(cudaGetLastError());
  if (sd) {
    HH_CUDA_TRY(cudaEventRecord(sd->b, sd->s));
    HH_CUDA_TRY(cudaStreamWaitEvent(s, sd->b, 0));
  }
  return HH_OK;
}

hh_status fine_apply3d(const Level& L, int B, const int* st, int op, VArg x, VArg y, VArg sub,
                       cudaStream_t s) {
  const F3 P = make3(L, 0, st, 0);
  if (g_march) return march3<M_APPLY>(L, P, B, x, VArg(), SArg(), VArg(), sub, y, op != HH_OP_A0, s);
  const dim3 g = grid3(P, B), bl(BX, BY);
  if (L.het) {
    if (op == HH_OP_A0) k_apply3d<true, false><<<g, bl, 0, s>>>(P, x, y, sub);
    else k_apply3d<true, true><<<g, bl, 0, s>>>(P, x, y, sub);
  } else {
    if (op == HH_OP_A0) k_apply3d<false, false><<<g, bl, 0, s>>>(P, x, y, sub);
    else k_apply3d<false, true><<<g, bl, 0, s>>>(P, x, y, sub);
  }
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

static hh_status jac3(const Level& L, const F3& P, int B, VArg f, SArg fs, VArg u, VArg uo,
                      cudaStream_t s) {
  if (g_march && u.p) return march3<M_JAC>(L, P, B, u, f, fs, VArg(), VArg(), uo, true, s);
  if (g_march)   // the first step from u = 0: pointwise
    return L.het ? pw3<true, 0>(P, B, f, fs, VArg(), VArg(), uo, s) : pw3<false, 0>(P, B, f, fs, VArg(), VArg(), uo, s);
  const dim3 g = grid3(P, B), bl(BX, BY);
  if (L.het) k_jacobi3d<true><<<g, bl, 0, s>>>(P, f, fs, u, uo);
  else k_jacobi3d<false><<<g, bl, 0, s>>>(P, f, fs, u, uo);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

// Pre-smoothing + residual + I^T.  With G ghost planes of f valid, step k of
// the smoother is computed on ext = G - k + 1 planes beyond the owned ones and
// the residual on ext = G - nu >= 1, which is what the restriction of the
// owned coarse planes reads: no exchange inside the V-cycle's pre-smoothing.
hh_status fine_pre3d(const Level& L, int B, const int* st, int nu, double omega, VArg f, SArg fs,
                     VArg u, VArg rc, cudaStream_t s) {
  const int64_t N = L.stride;
  VArg t0 = varg(L.tmp, 2 * N), t1 = varg(L.tmp + N, 2 * N);
  // nu steps ending in u: ping-pong so that the last write lands in u
  VArg bufs[2] = {t0, u};
  int cur = (nu % 2 == 1) ? 1 : 0;   // first destination
  VArg none;
  HH_TRY(jac3(L, make3(L, omega, st, L.G), B, f, fs, none, bufs[cur], s));
  for (int k = 2; k <= nu; ++k) {
    HH_TRY(jac3(L, make3(L, omega, st, L.G - k + 1), B, f, fs, bufs[cur], bufs[cur ^ 1], s));
    cur ^= 1;
  }
  const F3 Pr = make3(L, omega, st, std::max(L.G - nu, 0));
  const dim3 g = grid3(Pr, B), bl(BX, BY);
  if (g_march) HH_TRY(march3<M_RES>(L, Pr, B, u, f, fs, VArg(), VArg(), t1, true, s));
  else if (L.het) k_resid3d<true><<<g, bl, 0, s>>>(Pr, f, fs, u, t1);
  else k_resid3d<false><<<g, bl, 0, s>>>(Pr, f, fs, u, t1);
  const int NC1 = L.n / 2 + 1;
  const int cspan = L.maxloc / 2 + 1;
  const dim3 gc((NC1 + BX - 1) / BX, (NC1 + BY - 1) / BY, cspan * B);
  k_restrict3d<<<gc, bl, 0, s>>>(make3(L, omega, st, 0), cspan, t1, rc);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

// Prolongation + correction + post-smoothing (+ A_0 z): with u valid on G = nu + 1
// ghost planes the prolongation runs on ext = nu + 1, step k on nu + 1 - k, A_0 on 0.
hh_status fine_post3d(const Level& L, int B, const int* st, int nu, double omega, VArg f, SArg fs,
                      VArg u, VArg ec, VArg z, VArg w, cudaStream_t s) {
  const int64_t N = L.stride;
  VArg t0 = varg(L.tmp, 2 * N);
  const int e0 = std::min(L.G, nu + 1);
  const F3 Pp = make3(L, omega, st, e0);
  const dim3 bl(BX, BY);
  // the nu post-steps must end in z: pick the prolongation target accordingly
  VArg bufs[2] = {t0, z};
  // the prolongation fused into the first post-smoothing step (staged through
  // registers with the prolongation added) or a separate pointwise kernel followed
  // by the cp.async-staged steps; HH_3D_JACP=1 selects the fused one (A/B)
  static const bool fuse_p = getenv("HH_3D_JACP") && atoi(getenv("HH_3D_JACP")) != 0;
  if (g_march && fuse_p) {
    // prolongation fused into the first post-smoothing step (x + I e_c formed on load)
    int cur = (nu % 2 == 1) ? 1 : 0;   // first destination: the nu steps end in z
    HH_TRY(march3<M_JACP>(L, make3(L, omega, st, std::max(e0 - 1, 0)), B, u, f, fs, ec, VArg(), bufs[cur],
                          true, s));
    for (int k = 2; k <= nu; ++k) {
      HH_TRY(jac3(L, make3(L, omega, st, std::max(e0 - k, 0)), B, f, fs, bufs[cur], bufs[cur ^ 1], s));
      cur ^= 1;
    }
    if (w.p) HH_TRY(fine_apply3d(L, B, st, HH_OP_A0, z, w, VArg(), s));
    HH_CUDA_TRY(cudaGetLastError());
    return HH_OK;
  }
  int cur = (nu % 2 == 0) ? 1 : 0;
  if (g_march) HH_TRY((pw3<false, 1>(Pp, B, VArg(), SArg(), u, ec, bufs[cur], s)));
  else k_prolong3d<<<grid3(Pp, B), bl, 0, s>>>(Pp, u, ec, bufs[cur]);
  for (int k = 1; k <= nu; ++k) {
    HH_TRY(jac3(L, make3(L, omega, st, std::max(e0 - k, 0)), B, f, fs, bufs[cur], bufs[cur ^ 1], s));
    cur ^= 1;
  }
  if (w.p) HH_TRY(fine_apply3d(L, B, st, HH_OP_A0, z, w, VArg(), s));
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status fine_dinv3d(const Level& L, int B, cudaStream_t s) {
  F3 P = make3(L, 0, nullptr, L.G);
  P.dinv = nullptr;
  const dim3 g = grid3(P, B), bl(BX, BY);
  if (L.het) k_dinv3d<true><<<g, bl, 0, s>>>(P, L.dinv);
  else k_dinv3d<false><<<g, bl, 0, s>>>(P, L.dinv);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status coarse_stencil3d(const Level& C, int B, cplx* st, cudaStream_t s) {
  const F3 P = make3(C, 0, nullptr, 0);
  const dim3 g = grid3(P, B), bl(BX, BY);
  if (C.het) k_stencil3d<true><<<g, bl, 0, s>>>(P, st);
  else k_stencil3d<false><<<g, bl, 0, s>>>(P, st);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}
