// Internal declarations of the B200 hot path (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>
#include "../../include/hh.h"

// ---------------------------------------------------------------- complex fp64
typedef double2 cplx;   // (re, im), 16 B: same bytes as torch.complex128

__host__ __device__ __forceinline__ cplx cmake(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ cplx cscale(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
// conj(a) * b
__host__ __device__ __forceinline__ cplx cconjmul(cplx a, cplx b) {
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
// acc += a * b
__host__ __device__ __forceinline__ void cfma(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}
// acc -= a * b
__host__ __device__ __forceinline__ void cfms(cplx& acc, cplx a, cplx b) {
  acc.x = fma(-a.x, b.x, fma(a.y, b.y, acc.x));
  acc.y = fma(-a.x, b.y, fma(-a.y, b.x, acc.y));
}
__host__ __device__ __forceinline__ cplx cinv(cplx a) {
  double d = 1.0 / (a.x * a.x + a.y * a.y);
  return make_double2(a.x * d, -a.y * d);
}
__host__ __device__ __forceinline__ double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }

// ---------------------------------------------------------------- errors
void hh_set_error(const char* fmt, ...);
#define HH_CUDA_TRY(expr)                                                          \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      hh_set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__,   \
                   __LINE__, cudaGetErrorString(_e));                              \
      return HH_E_CUDA;                                                            \
    }                                                                              \
  } while (0)
#define HH_TRY(expr)                   \
  do {                                 \
    hh_status _s = (expr);             \
    if (_s != HH_OK) return _s;        \
  } while (0)

// ---------------------------------------------------------------- level data
// Per-level (fine or coarse) geometry and element coefficients.
struct Level {
  int dim = 2;
  int n = 0;            // cells per side
  int64_t nodes = 0;    // (n+1)^dim
  int64_t elems = 0;    // n^dim
  double h = 0;
  bool het = false;
  double k_const = 0, eps_const = 0;
  double2* coef = nullptr;   // het: per element (k_e, eps_e), device
};

// ---------------------------------------------------------------- fine-level kernels
struct FineArgs {
  int n; double h; double omega;
  bool het; double k; double eps;      // constant-k case
  const double2* coef;                 // het: (k_e, eps_e) per element
};

// y = A x  (op: 0 -> A_0, 1 -> A_eps).  If sub_from != NULL: y = sub_from - A x.
hh_status fine_apply(const Level& L, int op, const cplx* x, cplx* y, const cplx* sub_from,
                     cudaStream_t s);
// Pre-smoothing + restriction (fused): u = S^nu (from 0) applied to f*fscale; rc = I^T (f - A_eps u)
hh_status fine_pre(const Level& L, int nu, double omega, const cplx* f, const double* fscale,
                   cplx* u, cplx* rc, cudaStream_t s);
// Prolongation + correction + post-smoothing (+ optional w = A_0 z)
hh_status fine_post(const Level& L, int nu, double omega, const cplx* f, const double* fscale,
                    const cplx* u, const cplx* ec, cplx* z, cplx* w, cudaStream_t s);
// Coarse stencil assembly: st[node*3^d + o] = A_eps^{(1)} entries
hh_status coarse_stencil(const Level& C, cplx* st, cudaStream_t s);

// ---------------------------------------------------------------- coarse ND solver
struct NDFactor;
hh_status nd_create(const Level& C, NDFactor** out, cudaStream_t s);
hh_status nd_factor(NDFactor* f, const cplx* stencil, cudaStream_t s);
hh_status nd_solve(NDFactor* f, const cplx* rhs, cplx* x, cudaStream_t s);
void nd_destroy(NDFactor* f);
int64_t nd_factor_bytes(const NDFactor* f);   // bytes streamed per solve (X, H, L blocks)
int nd_levels(const NDFactor* f);

// ---------------------------------------------------------------- krylov
struct KrylovWS {
  int64_t N = 0; int m = 0;
  cplx* V = nullptr;     // (m+1) x N  (stored unnormalised; vscale[i] scales V[i])
  cplx* Z = nullptr;     // m x N
  cplx* w = nullptr;     // N
  cplx* u = nullptr;     // N (pre-smoothed iterate)
  cplx* rc = nullptr;    // coarse rhs
  cplx* ec = nullptr;    // coarse solution
  // device scalars
  double* vscale = nullptr;   // m+1
  cplx* H = nullptr;          // (m+1) x m, column-major H[i + (m+1) j]
  double* cs = nullptr;       // m
  cplx* sn = nullptr;         // m
  cplx* g = nullptr;          // m+1
  cplx* y = nullptr;          // m
  cplx* partial = nullptr;    // nblk x (m+2)
  double* dscal = nullptr;    // misc device scalars [0]=bnorm, [1]=|g_{j+1}|, [2]=flag ...
  int nblk = 0;
};
