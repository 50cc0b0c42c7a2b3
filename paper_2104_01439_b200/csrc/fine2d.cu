// 2D fine-level kernels: matrix-free Q1 operator apply, fused damped-Jacobi
// pre-smoothing + residual restriction, fused prolongation + correction +
// post-smoothing (+ A_0 apply of the result), coarse stencil assembly.
//
// Operator (Eq. sys_matrix; 2D stencils PAPER.md:124-129):
//   A(k,eps) = K - M(k,eps) - i B(k),  element-constant lambda_e = k_e^2 + i eps_e
//   (reading C1), boundary faces weighted by the adjacent element's k_e (C3).
// Per element e with the node at one corner and its element neighbours
// xh (along x), xv (along y), xd (diagonal):
//   K^e row  = 2/3 xp - 1/6 (xh + xv) - 1/3 xd
//   M^e row  = h^2/36 (4 xp + 2 (xh + xv) + xd)
//   B^f row  = h/6 (2 xp + x_other)                 (boundary edge f)
// Jacobi: u <- u + omega D^{-1} (f - A_eps u), D = diag(A_eps) incl. -i k B
// (reading C6).  Transfers: I^T with weights
// 1, 1/2, 1/4 (reading C5) and bilinear I.
//
// Design (B200): one CTA computes a TX x TY tile of fine nodes; the inputs
// of the whole multi-step sequence are staged once in shared memory with a
// halo of R = nu + 1 nodes and every intermediate Jacobi iterate lives in
// shared memory (halo recompute / temporal blocking), so a V-cycle touches
// HBM twice per fine vector instead of once per smoothing step.
#include "hh_internal.cuh"

namespace {

constexpr int TX = 32;   // tile width  (fine nodes along x, even)
constexpr int TY = 16;   // tile height (even)
constexpr int NT = 256;  // threads per CTA

struct Tile {
  int X0, Y0, R, SX, SY;
  __device__ __forceinline__ int gx(int sx) const { return X0 - R + sx; }
  __device__ __forceinline__ int gy(int sy) const { return Y0 - R + sy; }
};

// element coefficient (k, eps) of element (ex, ey); the smem copy covers the
// (SX+1) x (SY+1) elements starting at (X0-R-1, Y0-R-1) so that the diagonal
// of every node of the region is available.
template <bool HET>
__device__ __forceinline__ double2 elem_coef(const double2* sE, const Tile& t, int ex, int ey,
                                             double kc, double ec) {
  if (HET) return sE[(ex - (t.X0 - t.R - 1)) + (ey - (t.Y0 - t.R - 1)) * (t.SX + 1)];
  return make_double2(kc, ec);
}

// (A x)_p and optionally D_p at the node held in smem slot si (coords gx, gy).
// EPS: use lambda = k^2 + i eps (A_eps) if true, k^2 (A_0) otherwise.
template <bool HET, bool EPS, bool WANT_D>
__device__ __forceinline__ void node_op(const cplx* __restrict__ X, int si, const Tile& t, int gx,
                                        int gy, int n, double h, const double2* sE, double kc,
                                        double ec, cplx& ax, cplx& dg) {
  const int SX = t.SX;
  const double h2 = h * h * (1.0 / 36.0);
  const cplx xp = X[si];
  ax = cmake(0, 0);
  dg = cmake(0, 0);
  cplx ksum = cmake(0, 0), msum = cmake(0, 0);
  int nq = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int dx = (q & 1) ? 1 : -1, dy = (q & 2) ? 1 : -1;
    const int ex = gx + (dx < 0 ? -1 : 0), ey = gy + (dy < 0 ? -1 : 0);
    if (ex < 0 || ex >= n || ey < 0 || ey >= n) continue;
    const cplx xh = X[si + dx], xv = X[si + dy * SX], xd = X[si + dx + dy * SX];
    const cplx hv = cadd(xh, xv);
    cplx kp = cmake((2.0 / 3.0) * xp.x - (1.0 / 6.0) * hv.x - (1.0 / 3.0) * xd.x,
                    (2.0 / 3.0) * xp.y - (1.0 / 6.0) * hv.y - (1.0 / 3.0) * xd.y);
    cplx mp = cmake(h2 * (4.0 * xp.x + 2.0 * hv.x + xd.x), h2 * (4.0 * xp.y + 2.0 * hv.y + xd.y));
    if (HET) {
      const double2 c = elem_coef<true>(sE, t, ex, ey, kc, ec);
      const cplx lam = cmake(c.x * c.x, EPS ? c.y : 0.0);
      ax = cadd(ax, kp);
      cfms(ax, lam, mp);
      if (WANT_D) { dg.x += 2.0 / 3.0 - lam.x * 4.0 * h2; dg.y -= lam.y * 4.0 * h2; }
    } else {
      ksum = cadd(ksum, kp);
      msum = cadd(msum, mp);
      ++nq;
    }
  }
  if (!HET) {
    const cplx lam = cmake(kc * kc, EPS ? ec : 0.0);
    ax = ksum;
    cfms(ax, lam, msum);
    if (WANT_D) { dg.x = nq * (2.0 / 3.0 - lam.x * 4.0 * h2); dg.y = -nq * lam.y * 4.0 * h2; }
  }
  // boundary edges: -i k_e h/6 (2 xp + x_other)
  if (gx == 0 || gx == n || gy == 0 || gy == n) {
    const double h6 = h * (1.0 / 6.0);
    auto edge = [&](int ex, int ey, cplx xo) {
      const double k = elem_coef<HET>(sE, t, ex, ey, kc, ec).x;
      const cplx s = cmake(2.0 * xp.x + xo.x, 2.0 * xp.y + xo.y);
      ax.x += k * h6 * s.y;
      ax.y -= k * h6 * s.x;
      if (WANT_D) dg.y -= k * 2.0 * h6;
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
  }
}

// D_p = diag(A_eps) at node (gx, gy): sum over adjacent elements of
// K^e_pp - lambda_e M^e_pp = 2/3 - lambda_e h^2/9, minus i k_e h/3 per boundary edge.
template <bool HET>
__device__ __forceinline__ cplx node_diag(const Tile& t, int gx, int gy, int n, double h,
                                          const double2* sE, double kc, double ec) {
  const double h2 = h * h * (4.0 / 36.0);
  cplx dg = cmake(0, 0);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int ex = gx - 1 + (q & 1), ey = gy - 1 + ((q >> 1) & 1);
    if (ex < 0 || ex >= n || ey < 0 || ey >= n) continue;
    const double2 c = elem_coef<HET>(sE, t, ex, ey, kc, ec);
    dg.x += 2.0 / 3.0 - c.x * c.x * h2;
    dg.y -= c.y * h2;
  }
  if (gx == 0 || gx == n || gy == 0 || gy == n) {
    const double h3 = h / 3.0;
    if (gx == 0 || gx == n) {
      const int ex = (gx == 0) ? 0 : n - 1;
      if (gy > 0) dg.y -= elem_coef<HET>(sE, t, ex, gy - 1, kc, ec).x * h3;
      if (gy < n) dg.y -= elem_coef<HET>(sE, t, ex, gy, kc, ec).x * h3;
    }
    if (gy == 0 || gy == n) {
      const int ey = (gy == 0) ? 0 : n - 1;
      if (gx > 0) dg.y -= elem_coef<HET>(sE, t, gx - 1, ey, kc, ec).x * h3;
      if (gx < n) dg.y -= elem_coef<HET>(sE, t, gx, ey, kc, ec).x * h3;
    }
  }
  return dg;
}

template <bool HET>
__device__ __forceinline__ void load_region(cplx* sX, const cplx* __restrict__ g, const Tile& t,
                                            int n, double scale) {
  const int N1 = n + 1;
  for (int i = threadIdx.x; i < t.SX * t.SY; i += NT) {
    const int sx = i % t.SX, sy = i / t.SX;
    const int gx = t.gx(sx), gy = t.gy(sy);
    cplx v = cmake(0, 0);
    if (gx >= 0 && gx <= n && gy >= 0 && gy <= n) {
      v = g[(int64_t)gy * N1 + gx];
      v.x *= scale;
      v.y *= scale;
    }
    sX[i] = v;
  }
}

__device__ __forceinline__ void load_coef(double2* sE, const double2* __restrict__ coef,
                                          const Tile& t, int n) {
  const int EX = t.SX + 1, EY = t.SY + 1;
  for (int i = threadIdx.x; i < EX * EY; i += NT) {
    const int ex = t.X0 - t.R - 1 + i % EX, ey = t.Y0 - t.R - 1 + i / EX;
    double2 v = make_double2(0, 0);
    if (ex >= 0 && ex < n && ey >= 0 && ey < n) v = coef[(int64_t)ey * n + ex];
    sE[i] = v;
  }
}

// region of halo `hal` around the tile, clipped to the domain: iterate
#define FOR_REGION(hal, ...)                                                          \
  {                                                                                   \
    const int _w = TX + 2 * (hal), _hgt = TY + 2 * (hal);                             \
    for (int _i = threadIdx.x; _i < _w * _hgt; _i += NT) {                            \
      const int sx = t.R - (hal) + _i % _w, sy = t.R - (hal) + _i / _w;               \
      const int gx = t.gx(sx), gy = t.gy(sy);                                         \
      if (gx < 0 || gx > n || gy < 0 || gy > n) continue;                             \
      const int si = sy * t.SX + sx;                                                  \
      __VA_ARGS__                                                                     \
    }                                                                                 \
  }

// --------------------------------------------------------------------- apply
template <bool HET, bool EPS>
__global__ void __launch_bounds__(NT) k_apply2d(int n, double h, double kc, double ec,
                                                const double2* __restrict__ coef,
                                                const cplx* __restrict__ x, cplx* __restrict__ y,
                                                const cplx* __restrict__ sub) {
  extern __shared__ double4 smem_raw[];
  Tile t;
  t.X0 = blockIdx.x * TX; t.Y0 = blockIdx.y * TY; t.R = 1; t.SX = TX + 2; t.SY = TY + 2;
  cplx* sX = reinterpret_cast<cplx*>(smem_raw);
  double2* sE = reinterpret_cast<double2*>(sX + t.SX * t.SY);
  load_region<HET>(sX, x, t, n, 1.0);
  if (HET) load_coef(sE, coef, t, n);
  __syncthreads();
  FOR_REGION(0, {
    cplx ax, dg;
    node_op<HET, EPS, false>(sX, si, t, gx, gy, n, h, sE, kc, ec, ax, dg);
    const int64_t gi = (int64_t)gy * (n + 1) + gx;
    if (sub) ax = csub(sub[gi], ax);
    y[gi] = ax;
  })
}

// ------------------------------------------------- pre-smoothing + restriction
// u = S^nu(0; f), rc = I^T (f - A_eps u).  Halo R = nu + 1.
template <bool HET>
__global__ void __launch_bounds__(NT) k_pre2d(int n, double h, double omega, int nu, double kc,
                                              double ec, const double2* __restrict__ coef,
                                              const cplx* __restrict__ f,
                                              const double* __restrict__ fscale,
                                              cplx* __restrict__ u_out, cplx* __restrict__ rc) {
  extern __shared__ double4 smem_raw[];
  Tile t;
  t.X0 = blockIdx.x * TX; t.Y0 = blockIdx.y * TY; t.R = nu + 1;
  t.SX = TX + 2 * t.R; t.SY = TY + 2 * t.R;
  const int S = t.SX * t.SY;
  cplx* sF = reinterpret_cast<cplx*>(smem_raw);
  cplx* sA = sF + S;
  cplx* sB = sA + S;
  cplx* sDi = sB + S;
  double2* sE = reinterpret_cast<double2*>(sDi + S);
  const double sc = fscale ? *fscale : 1.0;
  load_region<HET>(sF, f, t, n, sc);
  if (HET) load_coef(sE, coef, t, n);
  for (int i = threadIdx.x; i < S; i += NT) { sA[i] = cmake(0, 0); sB[i] = cmake(0, 0); }
  __syncthreads();
  // D^{-1} and the first step from u = 0 (pointwise) on the full region
  FOR_REGION(t.R, {
    const cplx di = cinv(node_diag<HET>(t, gx, gy, n, h, sE, kc, ec));
    sDi[si] = di;
    sA[si] = cscale(cmul(di, sF[si]), omega);
  })
  __syncthreads();
  cplx* cur = sA;
  cplx* nxt = sB;
  for (int step = 2; step <= nu; ++step) {
    const int hal = t.R - step + 1;
    FOR_REGION(hal, {
      cplx ax, dg;
      node_op<HET, true, false>(cur, si, t, gx, gy, n, h, sE, kc, ec, ax, dg);
      cplx r = csub(sF[si], ax);
      cplx v = cur[si];
      cfma(v, cscale(sDi[si], omega), r);
      nxt[si] = v;
    })
    __syncthreads();
    cplx* tmp = cur; cur = nxt; nxt = tmp;
  }
  // residual on halo 1 -> nxt ; u on tile -> global
  FOR_REGION(1, {
    cplx ax, dg;
    node_op<HET, true, false>(cur, si, t, gx, gy, n, h, sE, kc, ec, ax, dg);
    nxt[si] = csub(sF[si], ax);
    if (sx >= t.R && sx < t.R + TX && sy >= t.R && sy < t.R + TY)
      u_out[(int64_t)gy * (n + 1) + gx] = cur[si];
  })
  // residual of out-of-domain halo slots must read as 0
  __syncthreads();
  // restriction I^T at coarse nodes (2I, 2J) inside the tile
  const int nc = n / 2;
  for (int i = threadIdx.x; i < (TX / 2) * (TY / 2); i += NT) {
    const int cx = t.X0 / 2 + i % (TX / 2), cy = t.Y0 / 2 + i / (TX / 2);
    if (cx > nc || cy > nc) continue;
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
    rc[(int64_t)cy * (nc + 1) + cx] = acc;
  }
}

// ------------------------------------- prolongation + correction + post-smoothing
// z = S^nu(u + I ec; f); if w: w = A_0 z.  Halo R = nu + (w ? 1 : 0).
template <bool HET>
__global__ void __launch_bounds__(NT) k_post2d(int n, double h, double omega, int nu, double kc,
                                               double ec, const double2* __restrict__ coef,
                                               const cplx* __restrict__ f,
                                               const double* __restrict__ fscale,
                                               const cplx* __restrict__ u,
                                               const cplx* __restrict__ ecv,
                                               cplx* __restrict__ z, cplx* __restrict__ w) {
  extern __shared__ double4 smem_raw[];
  Tile t;
  t.X0 = blockIdx.x * TX; t.Y0 = blockIdx.y * TY; t.R = nu + (w ? 1 : 0);
  t.SX = TX + 2 * t.R; t.SY = TY + 2 * t.R;
  const int S = t.SX * t.SY;
  cplx* sF = reinterpret_cast<cplx*>(smem_raw);
  cplx* sA = sF + S;
  cplx* sB = sA + S;
  cplx* sDi = sB + S;
  double2* sE = reinterpret_cast<double2*>(sDi + S);
  const double sc = fscale ? *fscale : 1.0;
  load_region<HET>(sF, f, t, n, sc);
  if (HET) load_coef(sE, coef, t, n);
  const int nc = n / 2, NC1 = nc + 1;
  // u + I ec on the full region
  for (int i = threadIdx.x; i < S; i += NT) {
    const int sx = i % t.SX, sy = i / t.SX;
    const int gx = t.gx(sx), gy = t.gy(sy);
    cplx v = cmake(0, 0);
    if (gx >= 0 && gx <= n && gy >= 0 && gy <= n) {
      v = u[(int64_t)gy * (n + 1) + gx];
      const int cx0 = gx >> 1, cy0 = gy >> 1;
      const int cx1 = (gx & 1) ? cx0 + 1 : cx0, cy1 = (gy & 1) ? cy0 + 1 : cy0;
      const double wx = (gx & 1) ? 0.5 : 1.0, wy = (gy & 1) ? 0.5 : 1.0;
      if (gx & 1) {
        if (gy & 1) {
          const cplx a = ecv[cy0 * NC1 + cx0], b = ecv[cy0 * NC1 + cx1];
          const cplx c = ecv[cy1 * NC1 + cx0], d = ecv[cy1 * NC1 + cx1];
          v.x += 0.25 * (a.x + b.x + c.x + d.x);
          v.y += 0.25 * (a.y + b.y + c.y + d.y);
        } else {
          const cplx a = ecv[cy0 * NC1 + cx0], b = ecv[cy0 * NC1 + cx1];
          v.x += wx * (a.x + b.x);
          v.y += wx * (a.y + b.y);
        }
      } else {
        if (gy & 1) {
          const cplx a = ecv[cy0 * NC1 + cx0], c = ecv[cy1 * NC1 + cx0];
          v.x += wy * (a.x + c.x);
          v.y += wy * (a.y + c.y);
        } else {
          const cplx a = ecv[cy0 * NC1 + cx0];
          v.x += a.x;
          v.y += a.y;
        }
      }
    }
    sA[i] = v;
    sB[i] = cmake(0, 0);
  }
  __syncthreads();
  FOR_REGION(t.R, { sDi[si] = cinv(node_diag<HET>(t, gx, gy, n, h, sE, kc, ec)); })
  __syncthreads();
  cplx* cur = sA;
  cplx* nxt = sB;
  for (int step = 1; step <= nu; ++step) {
    const int hal = t.R - step;
    FOR_REGION(hal, {
      cplx ax, dg;
      node_op<HET, true, false>(cur, si, t, gx, gy, n, h, sE, kc, ec, ax, dg);
      cplx r = csub(sF[si], ax);
      cplx v = cur[si];
      cfma(v, cscale(sDi[si], omega), r);
      nxt[si] = v;
    })
    __syncthreads();
    cplx* tmp = cur; cur = nxt; nxt = tmp;
  }
  FOR_REGION(0, {
    const int64_t gi = (int64_t)gy * (n + 1) + gx;
    z[gi] = cur[si];
    if (w) {
      cplx ax, dg;
      node_op<HET, false, false>(cur, si, t, gx, gy, n, h, sE, kc, ec, ax, dg);
      w[gi] = ax;
    }
  })
}

// ------------------------------------------------------------ coarse stencil
// st[node * 9 + (dx+1) + 3 (dy+1)] = entry of A_eps^{(1)} (rediscretisation on
// the 2h mesh; reading C4)
template <bool HET>
__global__ void k_stencil2d(int n, double h, double kc, double ec, const double2* __restrict__ coef,
                            cplx* __restrict__ st) {
  const int N1 = n + 1;
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= (int64_t)N1 * N1) return;
  const int gx = node % N1, gy = node / N1;
  cplx e[9];
#pragma unroll
  for (int o = 0; o < 9; ++o) e[o] = cmake(0, 0);
  const double h2 = h * h / 36.0;
  for (int q = 0; q < 4; ++q) {
    const int dx = (q & 1) ? 1 : -1, dy = (q & 2) ? 1 : -1;
    const int ex = gx + (dx < 0 ? -1 : 0), ey = gy + (dy < 0 ? -1 : 0);
    if (ex < 0 || ex >= n || ey < 0 || ey >= n) continue;
    double2 c = HET ? coef[(int64_t)ey * n + ex] : make_double2(kc, ec);
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
    const double k = HET ? coef[(int64_t)ey * n + ex].x : kc;
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
  for (int o = 0; o < 9; ++o) st[node * 9 + o] = e[o];
}

size_t smem_bytes(int R, int nfields, bool het) {
  const int SX = TX + 2 * R, SY = TY + 2 * R;
  size_t b = (size_t)SX * SY * sizeof(cplx) * nfields;
  if (het) b += (size_t)(SX + 1) * (SY + 1) * sizeof(double2);
  return b;
}

}  // namespace

// ----------------------------------------------------------------- host API
static hh_status set_smem(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) {
    HH_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  }
  return HH_OK;
}

hh_status fine_apply2d(const Level& L, int op, const cplx* x, cplx* y, const cplx* sub,
                       cudaStream_t s) {
  const int n = L.n;
  dim3 grid((n + 1 + TX - 1) / TX, (n + 1 + TY - 1) / TY);
  const size_t sm = smem_bytes(1, 1, L.het);
  const double ec = L.eps_const;
  if (L.het) {
    if (op == HH_OP_A0) {
      HH_TRY(set_smem((const void*)k_apply2d<true, false>, sm));
      k_apply2d<true, false><<<grid, NT, sm, s>>>(n, L.h, 0, 0, L.coef, x, y, sub);
    } else {
      HH_TRY(set_smem((const void*)k_apply2d<true, true>, sm));
      k_apply2d<true, true><<<grid, NT, sm, s>>>(n, L.h, 0, 0, L.coef, x, y, sub);
    }
  } else {
    if (op == HH_OP_A0) {
      HH_TRY(set_smem((const void*)k_apply2d<false, false>, sm));
      k_apply2d<false, false><<<grid, NT, sm, s>>>(n, L.h, L.k_const, ec, nullptr, x, y, sub);
    } else {
      HH_TRY(set_smem((const void*)k_apply2d<false, true>, sm));
      k_apply2d<false, true><<<grid, NT, sm, s>>>(n, L.h, L.k_const, ec, nullptr, x, y, sub);
    }
  }
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status fine_pre2d(const Level& L, int nu, double omega, const cplx* f, const double* fscale,
                     cplx* u, cplx* rc, cudaStream_t s) {
  const int n = L.n;
  dim3 grid((n + 1 + TX - 1) / TX, (n + 1 + TY - 1) / TY);
  const size_t sm = smem_bytes(nu + 1, 4, L.het);
  if (L.het) {
    HH_TRY(set_smem((const void*)k_pre2d<true>, sm));
    k_pre2d<true><<<grid, NT, sm, s>>>(n, L.h, omega, nu, 0, 0, L.coef, f, fscale, u, rc);
  } else {
    HH_TRY(set_smem((const void*)k_pre2d<false>, sm));
    k_pre2d<false><<<grid, NT, sm, s>>>(n, L.h, omega, nu, L.k_const, L.eps_const, nullptr, f,
                                        fscale, u, rc);
  }
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status fine_post2d(const Level& L, int nu, double omega, const cplx* f, const double* fscale,
                      const cplx* u, const cplx* ec, cplx* z, cplx* w, cudaStream_t s) {
  const int n = L.n;
  dim3 grid((n + 1 + TX - 1) / TX, (n + 1 + TY - 1) / TY);
  const size_t sm = smem_bytes(nu + (w ? 1 : 0), 4, L.het);
  if (L.het) {
    HH_TRY(set_smem((const void*)k_post2d<true>, sm));
    k_post2d<true><<<grid, NT, sm, s>>>(n, L.h, omega, nu, 0, 0, L.coef, f, fscale, u, ec, z, w);
  } else {
    HH_TRY(set_smem((const void*)k_post2d<false>, sm));
    k_post2d<false><<<grid, NT, sm, s>>>(n, L.h, omega, nu, L.k_const, L.eps_const, nullptr, f,
                                         fscale, u, ec, z, w);
  }
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status coarse_stencil2d(const Level& C, cplx* st, cudaStream_t s) {
  const int64_t N = C.nodes;
  const int bs = 128;
  const unsigned g = (unsigned)((N + bs - 1) / bs);
  if (C.het)
    k_stencil2d<true><<<g, bs, 0, s>>>(C.n, C.h, 0, 0, C.coef, st);
  else
    k_stencil2d<false><<<g, bs, 0, s>>>(C.n, C.h, C.k_const, C.eps_const, nullptr, st);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}
