// Local Fourier analysis of the 2D Q1 two-grid method (PAPER.md:205-258,
// symbols PAPER.md:273-334): rho_loc over a theta grid of T^low and the minimal
// convergent shift exponent sigma_c.
//
// For the harmonics theta^(00), theta^(11), theta^(10), theta^(01) of theta
// (cos(theta + pi) = -cos theta, so every symbol needs only
// c1 = cos t1, c2 = cos t2):
//   L_h   = (8 - 2c1 - 2c2 - 4c1c2)/3 - lambda h^2/36 (16 + 8c1 + 8c2 + 4c1c2)
//   L_2h  = same with cos 2t and lambda (2h)^2/36
//   S_h   = (1 - w) + w a (c1 + c2) + w b c1 c2,  a = (2/3 + 8 lh/36)/den,
//           b = (4/3 + 4 lh/36)/den, den = 8/3 - 16 lh/36, lh = lambda h^2
//   P     = [(1+c1)(1+c2), (1-c1)(1-c2), (1-c1)(1+c2), (1+c1)(1-c2)]^T,  R = P^T/4
//   T     = S^nu2 (I - P R L_h / L_2h) S^nu1
// T = D - a b^T with D = diag(s_i^(nu1+nu2)), a_i = s_i^nu2 P_i,
// b_i = P_i l_i s_i^nu1 / (4 L_2h): diagonal minus rank one, so
//   det(x I - T) = prod_i (x - d_i) + sum_i a_i b_i prod_{j != i} (x - d_j),
// whose four roots are found by Aberth iterations; rho(T) = max |root|.
//
// B200 design: ALU-bound (no memory traffic beyond the query list): one thread
// per theta point, a warp max and one 64-bit atomicMax per warp (rho >= 0, so
// the IEEE bit patterns order like the values).
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>
#include "hh_internal.cuh"

namespace {

constexpr int LFA_NT = 256;

// instrumentation: theta evaluations, Aberth iterations, kernel ms, launches
std::mutex g_stats_mu;
double g_stats[4] = {0, 0, 0, 0};

struct Q {
  double2 lam;   // k^2 + i beta k^sigma
  double h, omega;
  int nu1, nu2, m;
};

// 1/z with the correctly rounded reciprocal instruction sequence (no IEEE
// division slow path); z is never 0 here except at an exact root, guarded below
__device__ __forceinline__ cplx crcp(cplx a) {
  const double d = __drcp_rn(a.x * a.x + a.y * a.y);
  return make_double2(a.x * d, -a.y * d);
}
__device__ __forceinline__ cplx cdiv(cplx a, cplx b) { return cmul(a, crcp(b)); }
__device__ __forceinline__ cplx cpow_int(cplx a, int e) {
  cplx r = cmake(1, 0);
  for (int i = 0; i < e; ++i) r = cmul(r, a);
  return r;
}

// monic quartic x^4 + c[3] x^3 + c[2] x^2 + c[1] x + c[0]: value and derivative
__device__ __forceinline__ void poly_eval(const cplx* c, cplx z, cplx& p, cplx& dp) {
  p = cmake(1, 0);
  dp = cmake(0, 0);
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    dp = cadd(cmul(dp, z), p);
    p = cadd(cmul(p, z), c[i]);
  }
}

// spectral radius of T(theta); *its += Aberth iterations taken
__device__ double rho_T(const Q& q, double t1, double t2, int* its) {
  const double c1 = cos(t1), c2 = cos(t2);
  const double C1 = 2 * c1 * c1 - 1, C2 = 2 * c2 * c2 - 1;   // cos 2t
  const cplx lh = cscale(q.lam, q.h * q.h);
  const double sg1[4] = {1, -1, -1, 1}, sg2[4] = {1, -1, 1, -1};   // harmonic cosine signs
  // L_2h (one coarse harmonic)
  const cplx L2 = cmake((8 - 2 * C1 - 2 * C2 - 4 * C1 * C2) / 3.0 - lh.x * 4.0 / 36.0 * (16 + 8 * C1 + 8 * C2 + 4 * C1 * C2),
                        -lh.y * 4.0 / 36.0 * (16 + 8 * C1 + 8 * C2 + 4 * C1 * C2));
  const cplx den = cmake(8.0 / 3.0 - lh.x * 16.0 / 36.0, -lh.y * 16.0 / 36.0);
  const cplx sa = cdiv(cmake(2.0 / 3.0 + lh.x * 8.0 / 36.0, lh.y * 8.0 / 36.0), den);
  const cplx sb = cdiv(cmake(4.0 / 3.0 + lh.x * 4.0 / 36.0, lh.y * 4.0 / 36.0), den);
  const cplx inv4L2 = cinv(cscale(L2, 4.0));
  cplx d[4], ab[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double x1 = sg1[i] * c1, x2 = sg2[i] * c2;
    const double g = 16 + 8 * x1 + 8 * x2 + 4 * x1 * x2;
    const cplx l = cmake((8 - 2 * x1 - 2 * x2 - 4 * x1 * x2) / 3.0 - lh.x * g / 36.0, -lh.y * g / 36.0);
    cplx s = cmake(1 - q.omega, 0);
    cfma(s, cscale(sa, q.omega), cmake(x1 + x2, 0));
    cfma(s, cscale(sb, q.omega), cmake(x1 * x2, 0));
    // prolongation weights use the base cosines
    const double p = (i == 0) ? (1 + c1) * (1 + c2) : (i == 1) ? (1 - c1) * (1 - c2)
                   : (i == 2) ? (1 - c1) * (1 + c2) : (1 + c1) * (1 - c2);
    d[i] = cpow_int(s, q.nu1 + q.nu2);
    // a_i b_i = s^nu2 p * p l s^nu1 / (4 L2) = p^2 l s^(nu1+nu2) / (4 L2)
    ab[i] = cmul(cscale(cmul(l, d[i]), p * p), inv4L2);
  }
  // characteristic polynomial (monic): prod (x - d_i) + sum_i ab_i prod_{j != i} (x - d_j)
  cplx c[5] = {cmake(1, 0), cmake(0, 0), cmake(0, 0), cmake(0, 0), cmake(0, 0)};   // ascending, built up
#pragma unroll
  for (int i = 0; i < 4; ++i) {   // multiply by (x - d_i); degree i before
#pragma unroll
    for (int k = i + 1; k >= 1; --k) c[k] = csub(c[k - 1], cmul(d[i], c[k]));
    c[0] = cmul(cmake(-d[i].x, -d[i].y), c[0]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {   // + ab_i * cubic without (x - d_i)
    cplx e[4] = {cmake(1, 0), cmake(0, 0), cmake(0, 0), cmake(0, 0)};
#pragma unroll
    for (int jj = 0; jj < 3; ++jj) {
      const int j = jj < i ? jj : jj + 1;
#pragma unroll
      for (int k = jj + 1; k >= 1; --k) e[k] = csub(e[k - 1], cmul(d[j], e[k]));
      e[0] = cmul(cmake(-d[j].x, -d[j].y), e[0]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = cadd(c[k], cmul(ab[i], e[k]));
  }
  // Aberth iterations started next to the diagonal entries d_i (T is a rank-one
  // perturbation of diag(d)), each nudged off by a distinct small offset so
  // coincident d_i (symmetric theta) still give distinct starting points
  cplx z[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double sn, cs;
    sincos(1.5707963267948966 * k + 0.4, &sn, &cs);
    const double r0 = 1e-2 * (sqrt(cabs2(d[k])) + 1e-3);
    z[k] = cadd(d[k], cmake(r0 * cs, r0 * sn));
  }
  for (int it = 0; it < 200; ++it) {   // simultaneous (Jacobi) Aberth steps
    ++*its;
    cplx inv[6];                        // 1/(z_a - z_b) for the pairs (0,1) (0,2) (0,3) (1,2) (1,3) (2,3)
    inv[0] = crcp(csub(z[0], z[1])); inv[1] = crcp(csub(z[0], z[2])); inv[2] = crcp(csub(z[0], z[3]));
    inv[3] = crcp(csub(z[1], z[2])); inv[4] = crcp(csub(z[1], z[3])); inv[5] = crcp(csub(z[2], z[3]));
    cplx sum[4];
    sum[0] = cadd(cadd(inv[0], inv[1]), inv[2]);
    sum[1] = csub(cadd(inv[3], inv[4]), inv[0]);
    sum[2] = csub(inv[5], cadd(inv[1], inv[3]));
    sum[3] = cmake(-(inv[2].x + inv[4].x + inv[5].x), -(inv[2].y + inv[4].y + inv[5].y));
    double wmax = 0, zmax = 0;
    cplx w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      cplx p, dp;
      poly_eval(c, z[k], p, dp);
      w[k] = cmake(0, 0);
      if (cabs2(p) == 0 || cabs2(dp) == 0) continue;
      const cplx N = cdiv(p, dp);
      w[k] = cdiv(N, csub(cmake(1, 0), cmul(N, sum[k])));
      wmax = fmax(wmax, cabs2(w[k]));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      z[k] = csub(z[k], w[k]);
      zmax = fmax(zmax, cabs2(z[k]));
    }
    if (wmax <= 1e-28 * zmax) break;   // |w| <= 1e-14 |z|: the cubic step already landed
  }
  double r = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) r = fmax(r, sqrt(cabs2(z[k])));
  return r;
}

__global__ void __launch_bounds__(LFA_NT, 2) k_lfa_rho(const Q* __restrict__ qs,
                                                    unsigned long long* __restrict__ out,
                                                    unsigned long long* __restrict__ stats) {
  const Q q = qs[blockIdx.y];
  const int m = q.m;
  const int64_t total = (int64_t)m * m;
  const double step = 3.141592653589793 / m;
  double best = 0;
  int its = 0, evals = 0;
  for (int64_t e = blockIdx.x * (int64_t)LFA_NT + threadIdx.x; e < total; e += (int64_t)gridDim.x * LFA_NT) {
    const int i = (int)(e / m), j = (int)(e - (int64_t)i * m);
    const double t1 = -1.5707963267948966 + step * (i + 1), t2 = -1.5707963267948966 + step * (j + 1);
    if (fabs(t1) < 1e-12 && fabs(t2) < 1e-12) continue;   // theta = 0: L_2h singular (the set Lambda)
    best = fmax(best, rho_T(q, t1, t2, &its));
    ++evals;
  }
  for (int o = 16; o; o >>= 1) {
    its += __shfl_xor_sync(0xffffffffu, its, o);
    evals += __shfl_xor_sync(0xffffffffu, evals, o);
  }
  if ((threadIdx.x & 31) == 0 && evals) {
    atomicAdd(stats, (unsigned long long)evals);
    atomicAdd(stats + 1, (unsigned long long)its);
  }
  // warp maximum, one atomic per warp: no CTA barrier, so warps whose theta
  // points converged early leave without waiting for the slowest one
  for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best > 0)
    atomicMax(out + blockIdx.y, (unsigned long long)__double_as_longlong(best));
}

hh_status check_query(const hh_lfa_query& q) {
  if (q.m < 2 || q.m > 4096 || q.nu1 < 0 || q.nu2 < 0 || !(q.h > 0) || !(q.omega > 0 && q.omega <= 1)) {
    hh_set_error("lfa query: m in [2, 4096], nu >= 0, h > 0, omega in (0, 1] required");
    return HH_E_CONFIG;
  }
  return HH_OK;
}

Q make_q(const hh_lfa_query& in, double sigma) {
  Q q;
  q.lam = make_double2(in.k * in.k, in.beta * std::pow(in.k, sigma));   // reading C2
  q.h = in.h; q.omega = in.omega; q.nu1 = in.nu1; q.nu2 = in.nu2; q.m = in.m;
  return q;
}

// rho_loc of every query (at the given sigmas) on the device
hh_status rho_batch(const std::vector<Q>& qs, std::vector<double>& rho, cudaStream_t s) {
  const int n = (int)qs.size();
  rho.assign(n, 0.0);
  if (n == 0) return HH_OK;
  Q* dq = nullptr;
  unsigned long long* dr = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&dq, n * sizeof(Q), s);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&dr, (n + 2) * sizeof(unsigned long long), s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    if (dq) cudaFreeAsync(dq, s);
    hh_set_error("lfa: device allocation failed");
    return HH_E_OOM;
  }
  int mmax = 2;
  for (const Q& q : qs) mmax = std::max(mmax, q.m);
  const int bpq = (int)std::min<int64_t>(64, ((int64_t)mmax * mmax + LFA_NT - 1) / LFA_NT);
  HH_CUDA_TRY(cudaMemcpyAsync(dq, qs.data(), n * sizeof(Q), cudaMemcpyHostToDevice, s));
  HH_CUDA_TRY(cudaMemsetAsync(dr, 0, (n + 2) * sizeof(unsigned long long), s));
  cudaEvent_t ev[2];
  HH_CUDA_TRY(cudaEventCreate(&ev[0]));
  HH_CUDA_TRY(cudaEventCreate(&ev[1]));
  HH_CUDA_TRY(cudaEventRecord(ev[0], s));
  for (int q0 = 0; q0 < n; q0 += 65535) {
    const int cnt = std::min(65535, n - q0);
    k_lfa_rho<<<dim3(bpq, cnt), LFA_NT, 0, s>>>(dq + q0, dr + q0, dr + n);
  }
  HH_CUDA_TRY(cudaEventRecord(ev[1], s));
  HH_CUDA_TRY(cudaGetLastError());
  std::vector<unsigned long long> bits(n + 2);
  HH_CUDA_TRY(cudaMemcpyAsync(bits.data(), dr, (n + 2) * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(dq, s);
  cudaFreeAsync(dr, s);
  HH_CUDA_TRY(cudaStreamSynchronize(s));
  float ms = 0;
  cudaEventElapsedTime(&ms, ev[0], ev[1]);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  for (int i = 0; i < n; ++i) memcpy(&rho[i], &bits[i], sizeof(double));
  {
    std::lock_guard<std::mutex> lk(g_stats_mu);
    g_stats[0] += (double)bits[n];
    g_stats[1] += (double)bits[n + 1];
    g_stats[2] += ms;
    g_stats[3] += 1;
  }
  return HH_OK;
}

struct DeviceScope {   // run on `device`, restore the caller's device
  int prev = -1;
  hh_status st = HH_OK;
  explicit DeviceScope(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess || cudaSetDevice(device) != cudaSuccess) {
      cudaGetLastError();
      hh_set_error("lfa: cannot use CUDA device %d", device);
      st = HH_E_CUDA;
    }
  }
  ~DeviceScope() { if (prev >= 0) cudaSetDevice(prev); }
};

}  // namespace

extern "C" hh_status hh_lfa_rho(const hh_lfa_query* q, int32_t n, int32_t device, double* rho_out) {
  if (n < 0 || (n > 0 && (!q || !rho_out))) { hh_set_error("hh_lfa_rho: NULL argument"); return HH_E_ARG; }
  if (n == 0) return HH_OK;
  std::vector<Q> qs(n);
  for (int i = 0; i < n; ++i) {
    HH_TRY(check_query(q[i]));
    qs[i] = make_q(q[i], q[i].sigma);
  }
  DeviceScope ds(device);
  if (ds.st != HH_OK) return ds.st;
  cudaStream_t s;
  HH_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  std::vector<double> rho;
  const hh_status st = rho_batch(qs, rho, s);
  cudaStreamDestroy(s);
  if (st != HH_OK) return st;
  for (int i = 0; i < n; ++i) rho_out[i] = rho[i];
  return HH_OK;
}

extern "C" hh_status hh_lfa_sigma_c(const hh_lfa_query* q, int32_t n, int32_t device, double sigma_lo,
                                    double sigma_hi, double tol, double* sigma_c_out) {
  if (n < 0 || (n > 0 && (!q || !sigma_c_out))) { hh_set_error("hh_lfa_sigma_c: NULL argument"); return HH_E_ARG; }
  if (!(sigma_hi > sigma_lo) || !(tol > 0)) {
    hh_set_error("hh_lfa_sigma_c: need sigma_lo < sigma_hi and tol > 0");
    return HH_E_CONFIG;
  }
  if (n == 0) return HH_OK;
  for (int i = 0; i < n; ++i) HH_TRY(check_query(q[i]));
  DeviceScope ds(device);
  if (ds.st != HH_OK) return ds.st;
  cudaStream_t s;
  HH_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  std::vector<double> lo(n, sigma_lo), hi(n, sigma_hi), rho;
  std::vector<int> active(n, 1);
  hh_status st = HH_OK;
  {   // the ends: converged at sigma_lo, or not even at sigma_hi
    std::vector<Q> qs;
    for (int i = 0; i < n; ++i) { qs.push_back(make_q(q[i], sigma_lo)); qs.push_back(make_q(q[i], sigma_hi)); }
    st = rho_batch(qs, rho, s);
    for (int i = 0; i < n && st == HH_OK; ++i) {
      if (rho[2 * i] < 1.0) { sigma_c_out[i] = sigma_lo; active[i] = 0; }
      else if (!(rho[2 * i + 1] < 1.0)) { sigma_c_out[i] = NAN; active[i] = 0; }
    }
  }
  while (st == HH_OK) {   // bisection rounds, every active query at once
    std::vector<Q> qs;
    std::vector<int> idx;
    for (int i = 0; i < n; ++i)
      if (active[i] && hi[i] - lo[i] > tol) { qs.push_back(make_q(q[i], 0.5 * (lo[i] + hi[i]))); idx.push_back(i); }
    if (idx.empty()) break;
    st = rho_batch(qs, rho, s);
    for (size_t k = 0; k < idx.size() && st == HH_OK; ++k) {
      const int i = idx[k];
      const double mid = 0.5 * (lo[i] + hi[i]);
      if (rho[k] < 1.0) hi[i] = mid; else lo[i] = mid;
    }
  }
  cudaStreamDestroy(s);
  if (st != HH_OK) return st;
  for (int i = 0; i < n; ++i)
    if (active[i]) sigma_c_out[i] = hi[i];
  return HH_OK;
}

extern "C" hh_status hh_lfa_stats(int32_t reset, double* st4) {
  std::lock_guard<std::mutex> lk(g_stats_mu);
  if (st4) memcpy(st4, g_stats, sizeof(g_stats));
  if (reset) memset(g_stats, 0, sizeof(g_stats));
  return HH_OK;
}
