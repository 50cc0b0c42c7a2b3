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
template <bool HET, bool EPS>
__device__ cplx row3(const F3& P, const cplx* __restrict__ x, const double2* cf, double2 kc,
                     int gx, int gy, int gz) {
  const int n = P.n, N1 = P.N1;
  const double h = P.h;
  const int64_t gi = ((int64_t)gz * N1 + gy) * N1 + gx;
  auto X = [&](int dx, int dy, int dz) {
    return __ldg(&x[gi + ((int64_t)dz * N1 + dy) * N1 + dx]);
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
  cplx ax = row3<HET, EPS>(P, x.at(b) - vo, cf, kc, gx, gy, gz);
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
    const cplx ax = row3<HET, true>(P, ub, cf, kc, gx, gy, gz);
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
  const cplx ax = row3<HET, true>(P, u.at(b) - vo, cf, kc, gx, gy, gz);
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

hh_status fine_apply3d(const Level& L, int B, const int* st, int op, VArg x, VArg y, VArg sub,
                       cudaStream_t s) {
  const F3 P = make3(L, 0, st, 0);
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
  if (L.het) k_resid3d<true><<<g, bl, 0, s>>>(Pr, f, fs, u, t1);
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
  int cur = (nu % 2 == 0) ? 1 : 0;
  k_prolong3d<<<grid3(Pp, B), bl, 0, s>>>(Pp, u, ec, bufs[cur]);
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
