// FGMRES Arnoldi kernels (flexible right-preconditioned GMRES).
//
// Classical Gram-Schmidt in two batched passes (reading C11: one multi-dot
// pass h = V_j^H w, one update pass w' = w - V_j h with ||w'||^2 fused),
// complex Givens rotations and the convergence test |g_{j+1}| <= rtol ||b||
// (C13) evaluated on the device by the last CTA of each pass (last-block-done
// pattern: deterministic, no extra launch, no host round trip).
//
// V[i] is stored UNNORMALISED; vscale[i] = 1 / ||V[i]|| is applied by every
// consumer (the V-cycle reads f = vscale[j] V[j]), which saves a full
// read+write pass per iteration.
#include "hh_internal.cuh"

namespace {
constexpr int KT = 256;     // threads per CTA
constexpr int VG = 8;       // vectors per dot group

__device__ __forceinline__ cplx block_sum(cplx v, cplx* sh) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  cplx r = cmake(0, 0);
  if (threadIdx.x == 0)
    for (int w = 0; w < KT / 32; ++w) r = cadd(r, sh[w]);
  return r;   // valid in thread 0
}

__device__ __forceinline__ bool last_block(unsigned* counter) {
  __shared__ bool amLast;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(counter, 1u);
    amLast = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (amLast) __threadfence();
  return amLast;
}

// h_i = <v_i, w> = vscale_i * sum conj(V_i) w, i = 0..nv-1 -> H column (Hcol)
// If accumulate: Hcol[i] += h_i (re-orthogonalisation pass), else Hcol[i] = h_i.
__global__ void __launch_bounds__(KT) k_mdot(const cplx* __restrict__ V, int64_t N, int nv,
                                             const double* __restrict__ vscale,
                                             const cplx* __restrict__ w, cplx* __restrict__ part,
                                             unsigned* counter, cplx* __restrict__ Hcol,
                                             int accumulate, const int* __restrict__ stop) {
  if (stop && *stop) return;
  __shared__ cplx sh[KT / 32];
  const int64_t chunk = (N + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(N, lo + chunk);
  for (int g0 = 0; g0 < nv; g0 += VG) {
    cplx acc[VG];
#pragma unroll
    for (int q = 0; q < VG; ++q) acc[q] = cmake(0, 0);
    for (int64_t i = lo + threadIdx.x; i < hi; i += KT) {
      const cplx wi = w[i];
#pragma unroll
      for (int q = 0; q < VG; ++q)
        if (g0 + q < nv) {
          const cplx v = V[(int64_t)(g0 + q) * N + i];
          acc[q].x += v.x * wi.x + v.y * wi.y;
          acc[q].y += v.x * wi.y - v.y * wi.x;
        }
    }
#pragma unroll
    for (int q = 0; q < VG; ++q) {
      if (g0 + q >= nv) break;
      const cplx r = block_sum(acc[q], sh);
      if (threadIdx.x == 0) part[(int64_t)blockIdx.x * nv + g0 + q] = r;
    }
  }
  if (last_block(counter)) {
    for (int q = threadIdx.x; q < nv; q += KT) {
      cplx s = cmake(0, 0);
      for (int b = 0; b < (int)gridDim.x; ++b) s = cadd(s, part[(int64_t)b * nv + q]);
      s = cscale(s, vscale[q]);
      Hcol[q] = accumulate ? cadd(Hcol[q], s) : s;
    }
    if (threadIdx.x == 0) *counter = 0u;
  }
}

struct GivensState {
  cplx* H; int ldh;          // (m+1) x m column-major
  double* cs; cplx* sn; cplx* g;
  double* vscale;
  double* dscal;             // [0] bnorm, [1] |g_{j+1}|, [2] rtol*bnorm
  int* flags;                // [0] stop, [1] converged, [2] breakdown, [3] nan
  double* hist;              // per-iteration |g_{j+1}|/bnorm (device, indexed by total iteration)
};

// w' = w - sum_i (H_i vscale_i) V_i  -> Vout ; partial ||w'||^2 ; last block:
// h_{j+1,j} = ||w'||, vscale_{j+1}, Givens on column j, convergence flags.
__global__ void __launch_bounds__(KT) k_update(const cplx* __restrict__ V, int64_t N, int nv,
                                               const cplx* __restrict__ w, cplx* __restrict__ Vout,
                                               double* __restrict__ part, unsigned* counter,
                                               GivensState gs, int j, int total_it, int finalize) {
  if (gs.flags[0]) return;
  __shared__ cplx cf[128];
  __shared__ cplx sh[KT / 32];
  cplx* Hcol = gs.H + (int64_t)j * gs.ldh;
  for (int q = threadIdx.x; q < nv; q += KT) cf[q] = cscale(Hcol[q], gs.vscale[q]);
  __syncthreads();
  const int64_t chunk = (N + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(N, lo + chunk);
  double nrm = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += KT) {
    cplx a = w[i];
    for (int q = 0; q < nv; ++q) cfms(a, cf[q], V[(int64_t)q * N + i]);
    Vout[i] = a;
    nrm += a.x * a.x + a.y * a.y;
  }
  const cplx r = block_sum(cmake(nrm, 0), sh);
  if (threadIdx.x == 0) part[blockIdx.x] = r.x;
  if (!last_block(counter)) return;
  if (threadIdx.x != 0) return;
  double s = 0;
  for (int b = 0; b < (int)gridDim.x; ++b) s += part[b];
  *counter = 0u;
  const double hn = sqrt(s);
  if (!finalize) {             // first pass of CGS2: only record the norm
    gs.dscal[3] = hn;
    return;
  }
  // Givens on column j
  Hcol[j + 1] = cmake(hn, 0);
  gs.vscale[j + 1] = hn > 0 ? 1.0 / hn : 0.0;
  for (int i = 0; i < j; ++i) {
    const cplx hi = Hcol[i], hi1 = Hcol[i + 1];
    const double c = gs.cs[i];
    const cplx sn = gs.sn[i];
    cplx a = cscale(hi, c);
    cfma(a, sn, hi1);
    cplx b = cscale(hi1, c);
    cfms(b, cmake(sn.x, -sn.y), hi);
    Hcol[i] = a;
    Hcol[i + 1] = b;
  }
  const cplx a = Hcol[j], b = Hcol[j + 1];
  double c;
  cplx sn;
  const double aa = sqrt(cabs2(a)), bb = sqrt(cabs2(b));
  if (bb == 0.0) { c = 1.0; sn = cmake(0, 0); }
  else if (aa == 0.0) { c = 0.0; sn = cmake(1, 0); }
  else {
    const double t = sqrt(aa * aa + bb * bb);
    c = aa / t;
    sn = cscale(cmul(cscale(a, 1.0 / aa), cmake(b.x, -b.y)), 1.0 / t);
  }
  gs.cs[j] = c;
  gs.sn[j] = sn;
  cplx r0 = cscale(a, c);
  cfma(r0, sn, b);
  Hcol[j] = r0;
  Hcol[j + 1] = cmake(0, 0);
  const cplx gj = gs.g[j];
  cplx gj1 = cmul(cmake(-sn.x, sn.y), gj);   // -conj(s) g_j
  gs.g[j + 1] = gj1;
  gs.g[j] = cscale(gj, c);
  const double res = sqrt(cabs2(gj1));
  gs.dscal[1] = res;
  gs.hist[total_it] = res / gs.dscal[0];
  if (!(res == res) || !(hn == hn) || isinf(hn)) { gs.flags[3] = 1; gs.flags[0] = 1; }
  if (res <= gs.dscal[2]) gs.flags[1] = 1;
  if (hn == 0.0) gs.flags[2] = 1;
}

// y = H^{-1} g (upper triangular k x k), one warp, column-oriented back substitution
__global__ void k_trisolve(const cplx* __restrict__ H, int ldh, const cplx* __restrict__ g, int k,
                           cplx* __restrict__ y) {
  __shared__ cplx rhs[128];
  for (int i = threadIdx.x; i < k; i += 32) rhs[i] = g[i];
  __syncwarp();
  for (int i = k - 1; i >= 0; --i) {
    const cplx yi = cmul(rhs[i], cinv(H[i + (int64_t)i * ldh]));
    __syncwarp();
    for (int r = threadIdx.x; r < i; r += 32) cfms(rhs[r], H[r + (int64_t)i * ldh], yi);
    if (threadIdx.x == 0) y[i] = yi;
    __syncwarp();
  }
}

// x += sum_i y_i Z_i
__global__ void __launch_bounds__(KT) k_xupdate(const cplx* __restrict__ Z, int64_t N, int k,
                                                const cplx* __restrict__ y, cplx* __restrict__ x) {
  __shared__ cplx ys[128];
  for (int q = threadIdx.x; q < k; q += KT) ys[q] = y[q];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < N; i += (int64_t)gridDim.x * KT) {
    cplx a = x[i];
    for (int q = 0; q < k; ++q) cfma(a, ys[q], Z[(int64_t)q * N + i]);
    x[i] = a;
  }
}

// ||r||^2 -> out_norm (sqrt) ; last block also initialises the Arnoldi state
// for a new cycle: vscale[0] = 1/||r||, g[0] = ||r||; if set_bnorm: bnorm.
__global__ void __launch_bounds__(KT) k_norm(const cplx* __restrict__ r, int64_t N,
                                             double* __restrict__ part, unsigned* counter,
                                             double* __restrict__ out_norm, double* vscale0,
                                             cplx* g0, double* bnorm, double rtol) {
  __shared__ cplx sh[KT / 32];
  double nrm = 0;
  for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < N; i += (int64_t)gridDim.x * KT) {
    const cplx a = r[i];
    nrm += a.x * a.x + a.y * a.y;
  }
  const cplx s = block_sum(cmake(nrm, 0), sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s.x;
  if (!last_block(counter)) return;
  if (threadIdx.x) return;
  double t = 0;
  for (int b = 0; b < (int)gridDim.x; ++b) t += part[b];
  *counter = 0u;
  const double nr = sqrt(t);
  *out_norm = nr;
  if (vscale0) *vscale0 = nr > 0 ? 1.0 / nr : 0.0;
  if (g0) *g0 = cmake(nr, 0);
  if (bnorm) { bnorm[0] = nr; bnorm[2] = rtol * nr; }
}

}  // namespace

// ================================================================ host side
hh_status krylov_mdot(const cplx* V, int64_t N, int nv, const double* vscale, const cplx* w,
                      cplx* part, unsigned* counter, cplx* Hcol, int accumulate, const int* stop,
                      int nblk, cudaStream_t s) {
  k_mdot<<<nblk, KT, 0, s>>>(V, N, nv, vscale, w, part, counter, Hcol, accumulate, stop);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status krylov_update(const cplx* V, int64_t N, int nv, const cplx* w, cplx* Vout, double* part,
                        unsigned* counter, cplx* H, int ldh, double* cs, cplx* sn, cplx* g,
                        double* vscale, double* dscal, int* flags, double* hist, int j,
                        int total_it, int finalize, int nblk, cudaStream_t s) {
  GivensState gs{H, ldh, cs, sn, g, vscale, dscal, flags, hist};
  k_update<<<nblk, KT, 0, s>>>(V, N, nv, w, Vout, part, counter, gs, j, total_it, finalize);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status krylov_trisolve(const cplx* H, int ldh, const cplx* g, int k, cplx* y, cudaStream_t s) {
  k_trisolve<<<1, 32, 0, s>>>(H, ldh, g, k, y);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status krylov_xupdate(const cplx* Z, int64_t N, int k, const cplx* y, cplx* x, int nblk,
                         cudaStream_t s) {
  k_xupdate<<<nblk, KT, 0, s>>>(Z, N, k, y, x);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status krylov_norm(const cplx* r, int64_t N, double* part, unsigned* counter, double* out,
                      double* vscale0, cplx* g0, double* bnorm, double rtol, int nblk,
                      cudaStream_t s) {
  k_norm<<<nblk, KT, 0, s>>>(r, N, part, counter, out, vscale0, g0, bnorm, rtol);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}
