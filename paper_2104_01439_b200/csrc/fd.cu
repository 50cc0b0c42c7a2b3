// Coarse solve by fast diagonalisation (constant k): e_c = (A_eps^(1))^{-1} r_c
// exactly, for the separable coarse operator of a constant-coefficient problem.
//
// What it computes.  Alg. 1 line 3 solves the coarse system
// A_eps^(1) e_c = r_c exactly ("direct LU", BASELINE configs[0]); the paper
// factors it (MUMPS).  For constant k and eps the Q1 coarse
// operator on the uniform grid of (0,1)^d is a Kronecker sum (PAPER.md:100-113
// with exact Q1 integration, readings C1-C4): with the 1D linear-element
// stiffness K1, mass M1 and boundary selector E = e_0 e_0^T + e_nc e_nc^T,
//     A = sum_axes M1 x .. x S0 x .. x M1  -  (k^2 + i eps) M1 x .. x M1,
//     S0 = K1 - i k E   (the boundary term -ik int_bdry u v),
// so with the generalised eigenpairs S0 V = M1 V Lambda, V^T M1 V = I,
//     A^{-1} = (V x .. x V) diag(1 / (lam_i + lam_j (+ lam_l) - k^2 - i eps)) (V^T x .. x V^T).
// This is the same exact solve (a direct method, Lynch-Rice-Thomas 1964), not an
// approximation: parity against the oracle's sparse LU is <= 1e-13 (DESIGN.md
// section 7e).  Cost: dense complex GEMMs -- O(m^3) (2D) / O(m^4) (3D) flops on
// the FP64 tensor cores (mma.sync m8n8k4 f64) against O(m^2 log m) / O(m^4)
// bytes of latency-bound triangular sweeps for the nested-dissection factor.
//
// The eigenpairs, without a general eigensolver:
//  * K1 and M1 are both diagonalised by the DCT-I vectors c_j(i) = cos(j pi i/nc)
//    (Neumann FE pencil): K1 c_j = mu_j M1 c_j, mu_j = (6/h^2)(1 - cos t_j)/(2 + cos t_j),
//    c_j^T M1 c_j = (4 + 2 cos t_j)/12 (x2 for j = 0, nc), t_j = j pi / nc;
//  * in the M1-orthonormal basis q_j, E = a a^T + b b^T with a_j = q_j(0),
//    b_j = q_j(nc) = (-1)^j a_j, so the even and odd modes decouple and each
//    parity block is Delta - 2ik z z^T: diagonal plus complex rank one;
//  * its eigenvalues are the roots of the secular equation
//    1 - 2ik sum_j z_j^2 / (mu_j - lam) = 0, found per root by Newton's method
//    continued from t = 0 (lam = mu_j) to t = 1 along Delta - t 2ik z z^T;
//    the eigenvector of root lam is (Delta - lam)^{-1} z, normalised v^T v = 1.
//  The roots are validated (finite, distinct, secular residual); a failure
//  (flag 1) makes HH_COARSE_AUTO fall back to the nested-dissection factor.
// Even/odd modes are symmetric/antisymmetric about the grid centre, so every
// coarse vector is FOLDED per axis (s_i = f_i + f_{nc-i}, a_i = f_i - f_{nc-i},
// P = nc/2 + 1 entries each) and the solve splits into 2^d independent blocks
// of size P^d -- half the flops per transform.
#include "hh_internal.cuh"

#include <math.h>
#include <cmath>
#include <cstdlib>

namespace {

constexpr int FD_KS = 32;        // continuation steps t = 1/KS .. 1
constexpr int FD_NEWT = 8;       // Newton iterations per step (early exit)
constexpr double FD_PAD = 1e30;  // eigenvalue of the padding slot of a short parity block

__device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
  const double s = 1.0 / (b.x * b.x + b.y * b.y);
  return cmake((a.x * b.x + a.y * b.y) * s, (a.y * b.x - a.x * b.y) * s);
}
__device__ __forceinline__ cplx csqrt_(cplx a) {   // principal branch
  const double r = hypot(a.x, a.y);
  double re = sqrt(0.5 * (r + fabs(a.x)));
  if (re == 0.0) return cmake(0, 0);
  double im = a.y / (2.0 * re);
  if (a.x < 0) { const double t = fabs(im); im = copysign(re, a.y); re = t; }
  return cmake(re, im);
}

// DCT-I mode j of the Neumann pencil on nc cells: mu_j and z_j = q_j(0) = 1/||c_j||_M1
__device__ __forceinline__ void fd_mode(int j, int nc, double& mu, double& z) {
  const double s = sinpi(0.5 * (double)j / nc);          // 1 - cos t = 2 sin^2(t/2)
  const double c = cospi((double)j / nc);
  mu = 6.0 * (double)nc * nc * (2.0 * s * s) / (2.0 + c);
  const double nrm2 = (4.0 + 2.0 * c) / 12.0 * ((j == 0 || j == nc) ? 2.0 : 1.0);
  z = 1.0 / sqrt(nrm2);
}
__host__ __device__ __forceinline__ int fd_count(int nc, int par) { return par ? (nc + 1) / 2 : nc / 2 + 1; }

// basis layout per sample (complex entries): V_e, V_o, VT_e, VT_o (P x P each,
// row-major, V[i][r] = component i (folded row) of eigenvector r), lam_e, lam_o (P),
// 1/nu_e, 1/nu_o (P)
__host__ __device__ __forceinline__ int64_t fd_mat_off(int P, int which, int par) {
  return (int64_t)(2 * which + par) * P * P;
}
__host__ __device__ __forceinline__ int64_t fd_lam_off(int P, int par) { return 4 * (int64_t)P * P + (int64_t)par * P; }
__host__ __device__ __forceinline__ int64_t fd_nu_off(int P, int par) { return 4 * (int64_t)P * P + 2 * (int64_t)P + (int64_t)par * P; }

// ---------------------------------------------------------------- setup kernels
// The eigenpairs depend on (k, nc) only -- not on eps -- so they are computed once
// per distinct k of a batch ("slot"); samples map to slots through bidx[b].
__device__ __forceinline__ cplx warp_csum(cplx v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}
__device__ __forceinline__ double warp_dsum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// roots of the secular equation: one warp per root (lanes split the sums over
// the poles), grid (root groups of 8, parity, slot)
__global__ void __launch_bounds__(256) k_fd_eig(int nc, const double* __restrict__ kslot, cplx* __restrict__ basis,
                                                int64_t BE, int* __restrict__ sflag) {
  extern __shared__ double fd_sm[];
  const int par = blockIdx.y, sl = blockIdx.z;
  const int p = fd_count(nc, par), P = nc / 2 + 1;
  double* d = fd_sm;                 // mu_q of this parity
  double* z2 = d + p;                // z_q^2
  for (int q = threadIdx.x; q < p; q += blockDim.x) {
    double zq;
    fd_mode(2 * q + par, nc, d[q], zq);
    z2[q] = zq * zq;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= p) return;
  const double k = kslot[sl];
  const cplx rho = cmake(0.0, -2.0 * k);
  cplx l = cmake(d[r], 0.0);
  const double scale = fmax(1.0, d[r]);
  for (int s = 1; s <= FD_KS; ++s) {
    const cplx tr = cscale(rho, (double)s / FD_KS);
    // intermediate points of the path only need to stay on their root's branch
    // (relative 1e-9); the end point t = 1 is polished to round-off
    const bool last = s == FD_KS;
    const double tol = last ? 1e-15 : 1e-9;
    for (int it = 0; it < (last ? 2 * FD_NEWT : FD_NEWT); ++it) {
      // g(l) = (d_r - l)(1 + t rho S) + t rho z_r^2, S = sum_{q != r} z_q^2 / (d_q - l)
      cplx S = cmake(0, 0), Sp = cmake(0, 0);
      for (int q = lane; q < p; q += 32) {
        if (q == r) continue;
        const cplx inv = cinv(cmake(d[q] - l.x, -l.y));
        const cplx t = cscale(inv, z2[q]);
        S = cadd(S, t);
        Sp = cadd(Sp, cmul(t, inv));
      }
      S = warp_csum(S);
      Sp = warp_csum(Sp);
      const cplx dr = cmake(d[r] - l.x, -l.y);
      const cplx one_trS = cadd(cmake(1, 0), cmul(tr, S));
      const cplx g = cadd(cmul(dr, one_trS), cscale(tr, z2[r]));
      const cplx gp = cadd(cmake(-one_trS.x, -one_trS.y), cmul(dr, cmul(tr, Sp)));
      const cplx step = cdiv(g, gp);
      l = csub(l, step);
      if (sqrt(cabs2(step)) <= tol * fmax(scale, sqrt(cabs2(l)))) break;   // uniform over the warp
    }
  }
  // residual of the converged root (relative to the terms of g)
  cplx S = cmake(0, 0);
  double Sabs = 0;
  for (int q = lane; q < p; q += 32) {
    if (q == r) continue;
    const cplx t = cscale(cinv(cmake(d[q] - l.x, -l.y)), z2[q]);
    S = cadd(S, t);
    Sabs += sqrt(cabs2(t));
  }
  S = warp_csum(S);
  Sabs = warp_dsum(Sabs);
  const cplx dr = cmake(d[r] - l.x, -l.y);
  const cplx g = cadd(cmul(dr, cadd(cmake(1, 0), cmul(rho, S))), cscale(rho, z2[r]));
  const double gs = sqrt(cabs2(dr)) * (1.0 + 2.0 * k * Sabs) + 2.0 * k * z2[r];
  if (lane == 0) {
    cplx* Bb = basis + (int64_t)sl * BE;
    Bb[fd_lam_off(P, par) + r] = l;
    if (!(isfinite(l.x) && isfinite(l.y)) || !(sqrt(cabs2(g)) <= 1e-9 * gs)) atomicOr(sflag + sl, 1);
    if (r == 0)
      for (int rr = p; rr < P; ++rr) {   // padding slot of the short (odd, nc even) block
        Bb[fd_lam_off(P, par) + rr] = cmake(FD_PAD, 0);
        Bb[fd_nu_off(P, par) + rr] = cmake(0, 0);
      }
  }
}

// distinct roots (a duplicate = a lost continuation path) and the normalisation
// v^T v = 1 of u_q = z_q / (d_q - lam): one warp per root
__global__ void __launch_bounds__(256) k_fd_norm(int nc, cplx* __restrict__ basis, int64_t BE, int* __restrict__ sflag) {
  extern __shared__ double fd_sm[];
  const int par = blockIdx.y, sl = blockIdx.z;
  const int p = fd_count(nc, par), P = nc / 2 + 1;
  double* d = fd_sm;
  double* z = d + p;
  cplx* lam = reinterpret_cast<cplx*>(z + p);
  cplx* Bb = basis + (int64_t)sl * BE;
  for (int q = threadIdx.x; q < p; q += blockDim.x) {
    fd_mode(2 * q + par, nc, d[q], z[q]);
    lam[q] = Bb[fd_lam_off(P, par) + q];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= p) return;
  const cplx l = lam[r];
  const double tol = 1e-9 * fmax(1.0, sqrt(cabs2(l)));
  bool dup = false;
  cplx nu2 = cmake(0, 0);
  for (int q = lane; q < p; q += 32) {
    if (q != r && sqrt(cabs2(csub(lam[q], l))) <= tol) dup = true;
    const cplx u = cscale(cinv(cmake(d[q] - l.x, -l.y)), z[q]);
    nu2 = cadd(nu2, cmul(u, u));
  }
  nu2 = warp_csum(nu2);
  dup = __any_sync(0xffffffffu, dup);
  if (lane == 0) {
    const cplx nu = csqrt_(nu2);
    if (dup || !(cabs2(nu) > 0) || !isfinite(nu.x) || !isfinite(nu.y)) atomicOr(sflag + sl, 1);
    Bb[fd_nu_off(P, par) + r] = cinv(nu);
  }
}

// V_par[i][r] = (1/nu_r) sum_q cos(j_q pi i / nc) z_q^2 / (mu_q - lam_r)  (folded rows
// i < P; zero for the padding column and the centre row of the odd block) and VT
__global__ void __launch_bounds__(256) k_fd_basis(int nc, cplx* __restrict__ basis, int64_t BE) {
  extern __shared__ double fd_sm[];
  const int par = blockIdx.y, sl = blockIdx.z;
  const int p = fd_count(nc, par), P = nc / 2 + 1;
  double* d = fd_sm;
  double* z2 = d + p;
  for (int q = threadIdx.x; q < p; q += blockDim.x) {
    double zq;
    fd_mode(2 * q + par, nc, d[q], zq);
    z2[q] = zq * zq;
  }
  __syncthreads();
  cplx* Bb = basis + (int64_t)sl * BE;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= P * P) return;
  const int i = idx / P, r = idx % P;
  cplx v = cmake(0, 0);
  if (r < p && !(par == 1 && 2 * i == nc)) {
    const cplx l = Bb[fd_lam_off(P, par) + r];
    const cplx inu = Bb[fd_nu_off(P, par) + r];
    const int two_nc = 2 * nc;
    for (int q = 0; q < p; ++q) {
      const int j = 2 * q + par;
      const double c = cospi((double)((int)(((int64_t)j * i) % two_nc)) / nc);
      cfma(v, cscale(cinv(cmake(d[q] - l.x, -l.y)), c * z2[q]), cmake(1, 0));
    }
    v = cmul(v, inu);
  }
  Bb[fd_mat_off(P, 0, par) + (int64_t)i * P + r] = v;
  Bb[fd_mat_off(P, 1, par) + (int64_t)r * P + i] = v;
}

// per sample: its slot's validation flag (-> 1), or a zero / non-finite diagonal
// entry of the transformed operator (-> 2, singular)
__global__ void k_fd_check(int dim, int nc, const double2* __restrict__ kc, const cplx* __restrict__ basis,
                           int64_t BE, const int* __restrict__ bidx, const int* __restrict__ sflag,
                           int* __restrict__ flag) {
  const int b = blockIdx.y, P = nc / 2 + 1;
  const int sl = bidx[b];
  if (sflag[sl]) {
    if (blockIdx.x == 0 && threadIdx.x == 0) flag[b] = 1;
    return;
  }
  const cplx* Bb = basis + (int64_t)sl * BE;
  const cplx shift = cmake(kc[b].x * kc[b].x, kc[b].y);
  const int64_t tot = (int64_t)(1 << dim) * (dim == 2 ? (int64_t)P * P : (int64_t)P * P * P);
  bool bad = false;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e;
    cplx D = cmake(-shift.x, -shift.y);
    const int nblk = 1 << dim;
    const int blk = (int)(r % nblk);
    r /= nblk;
    for (int a = 0; a < dim; ++a) {
      const int ia = (int)(r % P);
      r /= P;
      D = cadd(D, Bb[fd_lam_off(P, (blk >> a) & 1) + ia]);
    }
    const double m = cabs2(D);
    if (!(m > 1e-280) || !isfinite(m)) bad = true;
  }
  if (bad) atomicExch(flag + b, 2);
}

// ---------------------------------------------------------------- fold / unfold
__device__ __forceinline__ cplx ldx(const cplx* p) { return __ldg(p); }
// programmatic dependent launch inside the fold -> GEMM ... -> unfold chain (default on):
// a kernel signals once its last input is read / its main loop is done, the next one
// is launched while this one drains and blocks in fd_pdl_wait() until this one has
// completed and flushed; both are no-ops for launches without the attribute
__device__ __forceinline__ void fd_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void fd_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// 2D: rhs[y][x] (m x m) -> blocks [py*2+px][i][j] (P x P), i folded y, j folded x
__global__ void k_fd_fold2(int nc, const int* __restrict__ st, VArg rhs, cplx* __restrict__ W) {
  const int b = blockIdx.y;
  if (st && st[b]) return;
  const int P = nc / 2 + 1, m = nc + 1;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= P * P) return;
  const int i = idx / P, j = idx % P, i2 = nc - i, j2 = nc - j;
  const cplx* f = rhs.at(b);
  fd_pdl_wait();
  const cplx a = ldx(&f[(int64_t)i * m + j]), bq = ldx(&f[(int64_t)i * m + j2]);
  const cplx c = ldx(&f[(int64_t)i2 * m + j]), d = ldx(&f[(int64_t)i2 * m + j2]);
  fd_pdl_trigger();
  const bool xi = j < j2, yi = i < i2;   // false: centre line (no mirror)
  // fold along x
  const cplx sp0 = xi ? cadd(a, bq) : a, sm0 = xi ? csub(a, bq) : cmake(0, 0);   // row i
  const cplx sp1 = xi ? cadd(c, d) : c, sm1 = xi ? csub(c, d) : cmake(0, 0);     // row i2
  cplx* Wb = W + (int64_t)b * 4 * P * P + idx;
  const int64_t PP = (int64_t)P * P;
  Wb[0 * PP] = yi ? cadd(sp0, sp1) : sp0;              // (py, px) = (0, 0)
  Wb[1 * PP] = yi ? cadd(sm0, sm1) : sm0;              // (0, 1)
  Wb[2 * PP] = yi ? csub(sp0, sp1) : cmake(0, 0);      // (1, 0)
  Wb[3 * PP] = yi ? csub(sm0, sm1) : cmake(0, 0);      // (1, 1)
}
__global__ void k_fd_unfold2(int nc, const int* __restrict__ st, const cplx* __restrict__ W, VArg x) {
  const int b = blockIdx.y;
  if (st && st[b]) return;
  const int P = nc / 2 + 1, m = nc + 1;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= P * P) return;
  const int i = idx / P, j = idx % P, i2 = nc - i, j2 = nc - j;
  const int64_t PP = (int64_t)P * P;
  const cplx* Wb = W + (int64_t)b * 4 * PP + idx;
  fd_pdl_wait();
  const cplx z00 = Wb[0], z01 = Wb[PP], z10 = Wb[2 * PP], z11 = Wb[3 * PP];
  // unfold along y (P_y[i] +- Q_y[i]) then x
  const cplx r0p = cadd(z00, z10), r0m = cadd(z01, z11);   // row i : even-x part, odd-x part
  const cplx r1p = csub(z00, z10), r1m = csub(z01, z11);   // row i2
  cplx* o = x.at(b);
  o[(int64_t)i * m + j] = cadd(r0p, r0m);
  o[(int64_t)i * m + j2] = csub(r0p, r0m);
  o[(int64_t)i2 * m + j] = cadd(r1p, r1m);
  o[(int64_t)i2 * m + j2] = csub(r1p, r1m);
}

// 3D: rhs[z][y][x] -> blocks [pz*4+py*2+px][i][j][l]
__global__ void k_fd_fold3(int nc, const int* __restrict__ st, VArg rhs, cplx* __restrict__ W) {
  const int b = blockIdx.y;
  if (st && st[b]) return;
  const int P = nc / 2 + 1, m = nc + 1;
  const int64_t P3 = (int64_t)P * P * P;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= P3) return;
  const int i = (int)(idx / ((int64_t)P * P)), j = (int)((idx / P) % P), l = (int)(idx % P);
  const int I[2] = {i, nc - i}, J[2] = {j, nc - j}, L[2] = {l, nc - l};
  const bool in[3] = {l < nc - l, j < nc - j, i < nc - i};   // x, y, z: has a mirror
  const cplx* f = rhs.at(b);
  cplx v[8];   // v[cz*4 + cy*2 + cx] = f[I[cz]][J[cy]][L[cx]]
#pragma unroll
  for (int c = 0; c < 8; ++c)
    v[c] = ldx(&f[((int64_t)I[c >> 2] * m + J[(c >> 1) & 1]) * m + L[c & 1]]);
  // fold axis a in place: pairs (c, c | bit) -> (plus, minus) stored at (c, c | bit)
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int bit = 1 << a;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (!(c & bit)) {
        const cplx u = v[c], w = v[c | bit];
        v[c] = in[a] ? cadd(u, w) : u;
        v[c | bit] = in[a] ? csub(u, w) : cmake(0, 0);
      }
  }
  cplx* Wb = W + (int64_t)b * 8 * P3 + idx;
#pragma unroll
  for (int c = 0; c < 8; ++c) Wb[c * P3] = v[c];   // block index = pz*4 + py*2 + px = c
}
__global__ void k_fd_unfold3(int nc, const int* __restrict__ st, const cplx* __restrict__ W, VArg x) {
  const int b = blockIdx.y;
  if (st && st[b]) return;
  const int P = nc / 2 + 1, m = nc + 1;
  const int64_t P3 = (int64_t)P * P * P;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= P3) return;
  const int i = (int)(idx / ((int64_t)P * P)), j = (int)((idx / P) % P), l = (int)(idx % P);
  const int I[2] = {i, nc - i}, J[2] = {j, nc - j}, L[2] = {l, nc - l};
  const cplx* Wb = W + (int64_t)b * 8 * P3 + idx;
  cplx v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = Wb[c * P3];
  // unfold axis a: (plus, minus) -> (node, mirror) = (p + q, p - q)
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int bit = 1 << a;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (!(c & bit)) {
        const cplx u = v[c], w = v[c | bit];
        v[c] = cadd(u, w);
        v[c | bit] = csub(u, w);
      }
  }
  cplx* o = x.at(b);
#pragma unroll
  for (int c = 0; c < 8; ++c) o[((int64_t)I[c >> 2] * m + J[(c >> 1) & 1]) * m + L[c & 1]] = v[c];
}

// ---------------------------------------------------------------- batched complex GEMM (DMMA)
// C_z = A_z B_z for z = (sample b, block blk, slice sl); an operand is either
// data (base + (b*nblk + blk)*sblk + sl*ssl) or a basis matrix of sample b
// (which = 0: V, 1: V^T; parity from bit `axis` of blk).  Epilogue dmode 1 (2D)
// / 2 (3D): divide by D = sum of the axes' eigenvalues - (k^2 + i eps).
struct FDOp {
  const cplx* p; int64_t ld;
  int basis;        // -1 data, 0 V, 1 V^T
  int axis;
};
struct FDGemm {
  int M, N, K, P;
  FDOp A, B;
  cplx* C; int64_t ldc;
  int nblk, nsl;
  int64_t sblk, ssl;
  const cplx* basis; int64_t BE;
  const int* bidx;  // basis slot of sample b
  int dmode;        // 0 none, 1: rows axis 1 / cols axis 0 (2D), 2: rows axis 2 / cols (axis 1, axis 0) (3D)
  const double2* kc;
  const int* st;
};

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16z(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ const cplx* fd_operand(const FDGemm& g, const FDOp& o, int b, int blk, int sl) {
  if (o.basis < 0) return o.p + ((int64_t)b * g.nblk + blk) * g.sblk + (int64_t)sl * g.ssl;
  return g.basis + (int64_t)__ldg(&g.bidx[b]) * g.BE + fd_mat_off(g.P, o.basis, (blk >> o.axis) & 1);
}

#ifndef FD_BKC
#define FD_BKC 16
#endif
constexpr int FD_BK = FD_BKC;   // K-chunk per pipeline stage
#ifndef FD_3M
#define FD_3M 1
#endif
#ifndef FD_MINB48
#define FD_MINB48 2   // 48 x 48 tiles: 2 CTAs per SM (120 registers; 3 CTAs -> 96 registers + spills)
#endif
#ifndef FD_ST48
#define FD_ST48 2   // cp.async stages of the 48 x 48 tiles (3 = one barrier per K-chunk, two chunks in flight: measured slower, P = 134 coarse 111.8 -> 119.5 us)
#endif
#ifndef FD_ST32
#define FD_ST32 2   // other tiles (3 stages of 16-k chunks would cost a resident CTA; FD_BKC=12 keeps 5: A/B below)
#endif
template <int BM, int BN, int WR, int WC>
struct FDTile {
  static constexpr int NT = 32 * WR * WC;
  static constexpr int ST = BM == 48 ? FD_ST48 : FD_ST32;
  static constexpr int SA = (FD_BK % 8 == 4) ? FD_BK : FD_BK + 4;   // cplx row stride of the A stage: = 4 mod 8 (conflict-free fragment loads)
  static constexpr int SB = BN + 2;
  static constexpr int WM = BM / WR, WN = BN / WC, RB = WM / 8, CB = WN / 8;
  static constexpr size_t stage = (size_t)(BM * SA + FD_BK * SB);
  static constexpr size_t smem = ST * stage * sizeof(cplx);
};

template <int BM, int BN, int WR, int WC>
__global__ void __launch_bounds__(32 * WR * WC, BM == 32 ? 5 : (BM == 48 ? FD_MINB48 : (BM == 40 ? 4 : 2))) k_fd_gemm(FDGemm g) {
  using T = FDTile<BM, BN, WR, WC>;
  const int tiles_n = (g.N + BN - 1) / BN;
  const int i0 = (blockIdx.x / tiles_n) * BM, j0 = (blockIdx.x % tiles_n) * BN;
  int z = blockIdx.y;
  const int sl = z % g.nsl;
  z /= g.nsl;
  const int blk = z % g.nblk, b = z / g.nblk;
  if (g.st && g.st[b]) return;
  const cplx* A = fd_operand(g, g.A, b, blk, sl);
  const cplx* Bm = fd_operand(g, g.B, b, blk, sl);
  const int64_t lda = g.A.ld, ldb = g.B.ld;
  extern __shared__ double4 fd_smem[];
  cplx* sm = reinterpret_cast<cplx*>(fd_smem);
  auto load_stage = [&](int st_, int k0) {
    cplx* As = sm + st_ * T::stage;
    cplx* Bs = As + BM * T::SA;
    for (int e = threadIdx.x; e < BM * FD_BK; e += T::NT) {
      const int r = e / FD_BK, kk = e % FD_BK;
      const bool v = i0 + r < g.M && k0 + kk < g.K;
      cp_async16z(&As[r * T::SA + kk], v ? A + (int64_t)(i0 + r) * lda + k0 + kk : A, v);
    }
    for (int e = threadIdx.x; e < FD_BK * BN; e += T::NT) {
      const int kk = e / BN, c = e % BN;
      const bool v = k0 + kk < g.K && j0 + c < g.N;
      cp_async16z(&Bs[kk * T::SB + c], v ? Bm + (int64_t)(k0 + kk) * ldb + j0 + c : Bm, v);
    }
    cp_commit();
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = warp / WC, wc = warp % WC, gq = lane >> 2, q = lane & 3;
  // FD_3M: Gauss's three-multiplication complex product -- t1 = Ar Br, t2 = Ai Bi,
  // t3 = (Ar + Ai)(Br + Bi), Re = t1 - t2, Im = t3 - t1 - t2 -- 3 DMMAs per
  // complex multiply-add instead of 4 (FD_3M = 0: the 4-product form)
  double re[T::RB][T::CB][2], im[T::RB][T::CB][2], t3[T::RB][T::CB][2];
#pragma unroll
  for (int rb = 0; rb < T::RB; ++rb)
#pragma unroll
    for (int cb = 0; cb < T::CB; ++cb)
      re[rb][cb][0] = re[rb][cb][1] = im[rb][cb][0] = im[rb][cb][1] = t3[rb][cb][0] = t3[rb][cb][1] = 0.0;
  const int nk = (g.K + FD_BK - 1) / FD_BK;
  // 8-row / 8-column fragment blocks wholly beyond M / N (tile padding) and
  // k-steps wholly beyond K (the last chunk) are skipped: warp-uniform, and the
  // skipped products are exact zeros or never stored, so results are unchanged
  bool rbv[T::RB], cbv[T::CB];
#pragma unroll
  for (int rb = 0; rb < T::RB; ++rb) rbv[rb] = i0 + wr * T::WM + rb * 8 < g.M;
#pragma unroll
  for (int cb = 0; cb < T::CB; ++cb) cbv[cb] = j0 + wc * T::WN + cb * 8 < g.N;
  fd_pdl_wait();
  load_stage(0, 0);
  if (T::ST >= 3 && nk > 1) load_stage(1, FD_BK);
  for (int kt = 0; kt < nk; ++kt) {
    if (T::ST >= 3) {
      // three stages: chunk kt + 2 goes to the buffer chunk kt - 1 was read from,
      // free once every thread has passed this iteration's barrier
      if (kt + 1 < nk) cp_wait<1>(); else cp_wait<0>();
      __syncthreads();
      if (kt + 2 < nk) load_stage((kt + 2) % 3, (kt + 2) * FD_BK);
    } else {
      if (kt + 1 < nk) {
        load_stage((kt + 1) & 1, (kt + 1) * FD_BK);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
    }
    const cplx* As = sm + (T::ST >= 3 ? kt % 3 : (kt & 1)) * T::stage;
    const cplx* Bs = As + BM * T::SA;
    const int kv = g.K - kt * FD_BK;   // valid k of this chunk (>= FD_BK except the last)
#pragma unroll
    for (int ks = 0; ks < FD_BK / 4; ++ks) {
      if (ks * 4 >= kv) break;
      const int k = ks * 4 + q;
      cplx av[T::RB], bv[T::CB];
#pragma unroll
      for (int rb = 0; rb < T::RB; ++rb) av[rb] = As[(wr * T::WM + rb * 8 + gq) * T::SA + k];
#pragma unroll
      for (int cb = 0; cb < T::CB; ++cb) bv[cb] = Bs[k * T::SB + wc * T::WN + cb * 8 + gq];
#pragma unroll
      for (int rb = 0; rb < T::RB; ++rb)
#pragma unroll
        for (int cb = 0; cb < T::CB; ++cb) {
          if (!rbv[rb] || !cbv[cb]) continue;
          if (FD_3M) {
            dmma884(re[rb][cb][0], re[rb][cb][1], av[rb].x, bv[cb].x);                       // t1
            dmma884(im[rb][cb][0], im[rb][cb][1], av[rb].y, bv[cb].y);                       // t2
            dmma884(t3[rb][cb][0], t3[rb][cb][1], av[rb].x + av[rb].y, bv[cb].x + bv[cb].y);  // t3
          } else {
            dmma884(re[rb][cb][0], re[rb][cb][1], av[rb].x, bv[cb].x);    // Re += Ar Br
            dmma884(re[rb][cb][0], re[rb][cb][1], -av[rb].y, bv[cb].y);   // Re -= Ai Bi
            dmma884(im[rb][cb][0], im[rb][cb][1], av[rb].x, bv[cb].y);    // Im += Ar Bi
            dmma884(im[rb][cb][0], im[rb][cb][1], av[rb].y, bv[cb].x);    // Im += Ai Br
          }
        }
    }
    if (T::ST < 3) __syncthreads();
  }
  fd_pdl_trigger();
  cplx* C = g.C + ((int64_t)b * g.nblk + blk) * g.sblk + (int64_t)sl * g.ssl;
  const cplx* lamb = g.basis + (int64_t)__ldg(&g.bidx[b]) * g.BE;
  cplx shift = cmake(0, 0);
  if (g.dmode) shift = cmake(g.kc[b].x * g.kc[b].x, g.kc[b].y);
#pragma unroll
  for (int rb = 0; rb < T::RB; ++rb) {
    const int i = i0 + wr * T::WM + rb * 8 + gq;
    if (i >= g.M) continue;
    cplx li = cmake(0, 0);
    if (g.dmode == 1) li = lamb[fd_lam_off(g.P, (blk >> 1) & 1) + i];
    if (g.dmode == 2) li = lamb[fd_lam_off(g.P, (blk >> 2) & 1) + i];
#pragma unroll
    for (int cb = 0; cb < T::CB; ++cb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = j0 + wc * T::WN + cb * 8 + 2 * q + e;
        if (j >= g.N) continue;
        cplx v = FD_3M ? cmake(re[rb][cb][e] - im[rb][cb][e], t3[rb][cb][e] - re[rb][cb][e] - im[rb][cb][e])
                       : cmake(re[rb][cb][e], im[rb][cb][e]);
        if (g.dmode) {
          cplx D = csub(li, shift);
          if (g.dmode == 1) {
            D = cadd(D, lamb[fd_lam_off(g.P, blk & 1) + j]);
          } else {
            D = cadd(D, lamb[fd_lam_off(g.P, (blk >> 1) & 1) + j / g.P]);
            D = cadd(D, lamb[fd_lam_off(g.P, blk & 1) + j % g.P]);
          }
          v = cdiv(v, D);
        }
        C[(int64_t)i * g.ldc + j] = v;
      }
  }
}

// launch inside the FD chain: with programmatic stream serialisation (HH_FD_PDL=0 or
// HH_NO_PDL=1: plain launches).  Measured (profiles/r02/fd_pdl): coarse phase per batch
// iteration 28.1 -> 25.5 us (P = 9), 47.7 -> 46.8 (P = 34), 114.7 -> 111.3 (P = 101),
// 112.5 -> 111.0 (P = 134); sweep 87-89 -> 84-85 us, 3.473-3.483 -> 3.483-3.490e9 it*DOF/s
static const bool g_fd_pdl = !(getenv("HH_FD_PDL") && atoi(getenv("HH_FD_PDL")) == 0) && getenv("HH_NO_PDL") == nullptr;
template <typename... Args>
static hh_status fd_launch(void (*kern)(Args...), dim3 grid, int block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_fd_pdl ? 1 : 0;
  HH_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args...));
  return HH_OK;
}

template <int BM, int BN, int WR, int WC>
hh_status fd_gemm_launch(const FDGemm& g, int B, cudaStream_t s) {
  using T = FDTile<BM, BN, WR, WC>;
  HH_CUDA_TRY(smem_attr((const void*)k_fd_gemm<BM, BN, WR, WC>, T::smem));   // cached per device
  const int tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
  const int64_t zc = (int64_t)B * g.nblk * g.nsl;
  if (zc > 65535) { hh_set_error("fd_solve: batch x blocks x slices = %lld > 65535", (long long)zc); return HH_E_CONFIG; }
  return fd_launch(k_fd_gemm<BM, BN, WR, WC>, dim3(tiles, (unsigned)zc), T::NT, T::smem, s, g);
}
// tile choice: the least padded output area ceil(M/t) t x ceil(N/t) t over t = 32 / 40 / 48
// (ties -> the smaller tile: more CTAs); measured per grid size on the sweep's batches
// (scripts/probe_fd.py, profiles/r02/fd): the area rule picks the fastest of 32 / 48 at
// every size tried; 64 x 64 tiles never won.  40 x 40 tiles (5 warps of 8 x 40) are a
// candidate only where a GEMM dimension is <= 40: cfg3's P = 33 mode products (coarse
// 84.8 -> 78.9 us) and the sweep's P = 34 (56.8 -> 49.2 us); at P = 101 / 118 they lost
// to 32 x 32 (112.9 -> 118.4, 107.9 -> 111.9 us; profiles/r02/fd/tile40).
// HH_FD_TILE = 32 / 40 / 48 / 64 forces one (A/B).
// the tile fd_gemm launches for an M x N output (HH_FD_TILE forces one)
static int fd_tile_for(int M, int N) {
  static const int force = getenv("HH_FD_TILE") ? atoi(getenv("HH_FD_TILE")) : 0;
  static const bool use40 = !getenv("HH_FD_TILE40") || atoi(getenv("HH_FD_TILE40")) != 0;
  if (force) return force;
  const int tiles[3] = {32, 40, 48};
  int best = 0;
  int64_t ba = INT64_MAX;
  for (int t = 0; t < 3; ++t) {
    if (tiles[t] == 40 && (!use40 || std::min(M, N) > 40)) continue;   // 40: only where a dimension <= 40
    const int64_t a = (int64_t)((M + tiles[t] - 1) / tiles[t]) * tiles[t] * (((N + tiles[t] - 1) / tiles[t]) * tiles[t]);
    if (a < ba) { ba = a; best = t; }
  }
  return tiles[best];
}
hh_status fd_gemm(const FDGemm& g, int B, cudaStream_t s) {
  (void)B;
  const int tile = fd_tile_for(g.M, g.N);
  if (tile == 64) return fd_gemm_launch<64, 64, 4, 2>(g, B, s);
  if (tile == 48) return fd_gemm_launch<48, 48, 3, 2>(g, B, s);
  if (tile == 40) return fd_gemm_launch<40, 40, 5, 1>(g, B, s);
  return fd_gemm_launch<32, 32, 2, 2>(g, B, s);
}

}  // namespace

int fd_P(int nc) { return nc / 2 + 1; }
// 2D: CTAs one sample adds to each k_fd_gemm launch, and the CTAs of that tile one SM holds
void fd_gemm_ctas2d(int nc, int* per_sample, int* per_sm) {
  const int P = fd_P(nc), t = fd_tile_for(P, P), tl = (P + t - 1) / t;
  *per_sample = 4 * tl * tl;
  *per_sm = t == 32 ? 5 : (t == 48 ? FD_MINB48 : (t == 40 ? 4 : 2));
}
int64_t fd_basis_entries(int nc) {
  const int64_t P = fd_P(nc);
  return 4 * P * P + 4 * P;
}
int64_t fd_work_entries(int dim, int nc) {
  const int64_t P = fd_P(nc);
  return 2 * (int64_t)(1 << dim) * (dim == 2 ? P * P : P * P * P);
}
int fd_solve_launches(int dim) { return 2 + 2 * dim; }
double fd_solve_flops(int dim, int nc) {   // real flops of the 2d GEMMs (8 per complex multiply-add)
  const double P = fd_P(nc);
  return dim == 2 ? 4.0 * 4.0 * 8.0 * P * P * P : 6.0 * 8.0 * 8.0 * P * P * P * P;
}
int64_t fd_solve_bytes(int dim, int nc) {   // compulsory bytes: rhs + x, every pass's data, the bases
  const int64_t P = fd_P(nc), m = nc + 1;
  const int64_t Nc = dim == 2 ? m * m : m * m * m;
  const int64_t blk = (int64_t)(1 << dim) * (dim == 2 ? P * P : P * P * P);
  const int ng = 2 * dim;
  return 16 * (2 * Nc + 2 * blk + ng * 2 * blk + ng * 2 * P * P);
}

__global__ void k_fd_flag_all(int* flag, int B, int code) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) flag[b] = code;
}
hh_status fd_flag_all(int* flag, int B, int code, cudaStream_t s) {
  k_fd_flag_all<<<(B + 127) / 128, 128, 0, s>>>(flag, B, code);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status fd_setup(int dim, int nc, int B, int nslot, const double* kslot, const int* bidx, int* sflag,
                   const double2* kc, cplx* basis, int* flag, cudaStream_t s) {
  if (nc < 1 || nslot < 1) { hh_set_error("fd_setup: nc = %d, slots = %d", nc, nslot); return HH_E_CONFIG; }
  const int P = fd_P(nc);
  const int64_t BE = fd_basis_entries(nc);
  const size_t sm_eig = (size_t)P * 2 * sizeof(double);
  const size_t sm_norm = (size_t)P * (2 * sizeof(double) + sizeof(cplx));
  HH_CUDA_TRY(smem_attr((const void*)k_fd_eig, sm_eig));
  HH_CUDA_TRY(smem_attr((const void*)k_fd_norm, sm_norm));
  HH_CUDA_TRY(smem_attr((const void*)k_fd_basis, sm_eig));
  const dim3 roots((P + 7) / 8, 2, nslot);
  k_fd_eig<<<roots, 256, sm_eig, s>>>(nc, kslot, basis, BE, sflag);
  HH_CUDA_TRY(cudaGetLastError());
  k_fd_norm<<<roots, 256, sm_norm, s>>>(nc, basis, BE, sflag);
  HH_CUDA_TRY(cudaGetLastError());
  k_fd_basis<<<dim3((P * P + 255) / 256, 2, nslot), 256, sm_eig, s>>>(nc, basis, BE);
  HH_CUDA_TRY(cudaGetLastError());
  k_fd_check<<<dim3(std::min(64, (P * P * (1 << dim) + 255) / 256 + 1), B), 256, 0, s>>>(dim, nc, kc, basis, BE,
                                                                                         bidx, sflag, flag);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status fd_solve(int dim, int nc, int B, const int* st, const cplx* basis, const int* bidx, const double2* kc,
                   cplx* work, VArg rhs, VArg x, cudaStream_t s) {
  const int P = fd_P(nc);
  const int nblk = 1 << dim;
  const int64_t PD = dim == 2 ? (int64_t)P * P : (int64_t)P * P * P;
  cplx* W0 = work;
  cplx* W1 = work + (int64_t)B * nblk * PD;
  FDGemm g{};
  g.P = P; g.nblk = nblk; g.nsl = 1; g.sblk = PD; g.ssl = 0;
  g.basis = basis; g.BE = fd_basis_entries(nc); g.bidx = bidx; g.kc = kc; g.st = st;
  auto data = [](const cplx* p, int64_t ld) { FDOp o; o.p = p; o.ld = ld; o.basis = -1; o.axis = 0; return o; };
  auto bas = [&](int which, int axis) { FDOp o; o.p = nullptr; o.ld = P; o.basis = which; o.axis = axis; return o; };
  if (dim == 2) {
    const unsigned gx = (unsigned)((P * P + 255) / 256);
    HH_TRY(fd_launch(k_fd_fold2, dim3(gx, B), 256, 0, s, nc, st, rhs, W0));
    g.M = g.N = g.K = P; g.ldc = P;
    // Y = V_y^T F V_x (/ D), X = V_y H V_x^T
    g.A = data(W0, P); g.B = bas(0, 0); g.C = W1; g.dmode = 0; HH_TRY(fd_gemm(g, B, s));
    g.A = bas(1, 1); g.B = data(W1, P); g.C = W0; g.dmode = 1; HH_TRY(fd_gemm(g, B, s));
    g.A = bas(0, 1); g.B = data(W0, P); g.C = W1; g.dmode = 0; HH_TRY(fd_gemm(g, B, s));
    g.A = data(W1, P); g.B = bas(1, 0); g.C = W0; HH_TRY(fd_gemm(g, B, s));
    HH_TRY(fd_launch(k_fd_unfold2, dim3(gx, B), 256, 0, s, nc, st, (const cplx*)W0, x));
    return HH_OK;
  }
  const unsigned gx = (unsigned)((PD + 255) / 256);
  k_fd_fold3<<<dim3(gx, B), 256, 0, s>>>(nc, st, rhs, W0);
  HH_CUDA_TRY(cudaGetLastError());
  const int64_t P2 = (int64_t)P * P;
  // x-mode: (P^2 x P) . V_x
  g.M = (int)P2; g.N = P; g.K = P; g.ldc = P; g.nsl = 1; g.ssl = 0; g.dmode = 0;
  g.A = data(W0, P); g.B = bas(0, 0); g.C = W1; HH_TRY(fd_gemm(g, B, s));
  // y-mode: per z-slice V_y^T . (P x P)
  g.M = P; g.N = P; g.K = P; g.ldc = P; g.nsl = P; g.ssl = P2;
  g.A = bas(1, 1); g.B = data(W1, P); g.C = W0; HH_TRY(fd_gemm(g, B, s));
  // z-mode: V_z^T . (P x P^2), then / D
  g.M = P; g.N = (int)P2; g.K = P; g.ldc = P2; g.nsl = 1; g.ssl = 0; g.dmode = 2;
  g.A = bas(1, 2); g.B = data(W0, P2); g.C = W1; HH_TRY(fd_gemm(g, B, s));
  // inverse transform: V_z . , V_y . per slice, . V_x^T
  g.dmode = 0;
  g.A = bas(0, 2); g.B = data(W1, P2); g.C = W0; HH_TRY(fd_gemm(g, B, s));
  g.M = P; g.N = P; g.K = P; g.ldc = P; g.nsl = P; g.ssl = P2;
  g.A = bas(0, 1); g.B = data(W0, P); g.C = W1; HH_TRY(fd_gemm(g, B, s));
  g.M = (int)P2; g.N = P; g.K = P; g.ldc = P; g.nsl = 1; g.ssl = 0;
  g.A = data(W1, P); g.B = bas(1, 0); g.C = W0; HH_TRY(fd_gemm(g, B, s));
  k_fd_unfold3<<<dim3(gx, B), 256, 0, s>>>(nc, st, W0, x);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}
