// FGMRES Arnoldi kernels, batched over samples (flexible
// right-preconditioned GMRES; Saad 1993).
//
// Classical Gram-Schmidt in two batched passes (reading C11: one multi-dot
// pass h = V_j^H w, one update pass w' = w - V_j h with ||w'||^2 fused),
// complex Givens rotations c = |a|/t, s = (a/|a|) conj(b)/t and the convergence
// test |g_{j+1}| <= rtol ||b|| (C13), all evaluated on the device by the last
// CTA of each sample (last-block-done: deterministic, no extra launch, no host
// round trip).  The Arnoldi index j lives in device memory so one captured
// iteration replays for every j.
//
// V[i] is stored UNNORMALISED; vscale[i] = 1 / ||V[i]|| is applied by every
// consumer (the V-cycle reads f = vscale[j] V[j]), which saves a full
// read+write pass per iteration.
#include <algorithm>
#include <vector>
#include "hh_internal.cuh"
#include "krylov.cuh"

namespace {
constexpr int KT = 256;     // threads per CTA
constexpr int KMAX_CF = KMAX_RESTART + 8;   // Arnoldi coefficients staged per pass (>= m + 1)

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

// this thread's share of sum_k dpart[k], k < gridDim.x (strided; combined by block_sum)
__device__ __forceinline__ double grid_partial_sum(const double* dpart) {
  double t = 0;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += KT) t += dpart[k];
  return t;
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

// last_block for a counter shared by `total` CTAs
__device__ __forceinline__ bool last_of(unsigned* counter, int total) {
  __shared__ bool amLast;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) amLast = (atomicAdd(counter, 1u) == (unsigned)total - 1);
  __syncthreads();
  if (amLast) __threadfence();
  return amLast;
}

// sum_r P[r * ld + q] for q = threadIdx.x < cnt (<= KT / 2), rows split over the
// two thread halves (even / odd r), fixed order; sh: KT / 2 cplx of scratch
__device__ __noinline__ cplx colsum(const cplx* P, int64_t ld, int rows, int cnt, cplx* sh) {
  const int q = threadIdx.x % (KT / 2), half = threadIdx.x / (KT / 2);
  cplx s0 = cmake(0, 0), s1 = cmake(0, 0);
  if (q < cnt) {
    int r = half;
    for (; r + 2 < rows; r += 4) {
      s0 = cadd(s0, P[(int64_t)r * ld + q]);
      s1 = cadd(s1, P[(int64_t)(r + 2) * ld + q]);
    }
    if (r < rows) s0 = cadd(s0, P[(int64_t)r * ld + q]);
  }
  const cplx s = cadd(s0, s1);
  __syncthreads();
  if (half == 1) sh[q] = s;
  __syncthreads();
  return half == 0 ? cadd(s, sh[q]) : cmake(0, 0);   // valid in threads q < cnt
}

__device__ __forceinline__ void owned_view(const KArgs& A, int b, int64_t& off, int64_t& len) {
  const int2 sl = slab_of(A.slab, b, A.n);
  off = (int64_t)A.G * A.plane;
  len = (int64_t)(sl.y - sl.x) * A.plane;
}

// h_i = <v_i, w> = vscale_i * sum conj(V_i) w, i = 0..j -> H column j.
// Work unit = (vector q, sub-chunk of this CTA's nodes); warps take units
// round-robin (balanced for any j), each lane keeps 8 predicated loads in
// flight (no serial tail loop); unit partials are combined in shared memory in
// a fixed order (deterministic).
constexpr int MD_UNITS = 1024;   // max units per CTA (nv <= 128, sub-chunks <= 8)
constexpr int MD_GROUP = 32;     // CTAs per first-level group of the column sums
// pass 2 (reorth): w = V[j+1] (the first pass's w'), result h2 -> y (folded into
// H column j by the second update's tail); reorth = 1: ||w||^2 rides along as
// the extra column nv of the partials (DGKS criterion).
__global__ void __launch_bounds__(KT, 4) k_mdot(KArgs A, int pass) {
  const int b = blockIdx.y;
  if (A.ks.status[b]) return;
  if (pass == 2 && !A.reo[b]) return;
  const int j = *A.jdev;
  const int nv = j + 1;
  const bool wn = pass == 1 && A.reorth == 1;
  int64_t off, N;
  owned_view(A, b, off, N);
  const int64_t NS = A.Nst;
  const cplx* V = A.V + (int64_t)b * A.Vbs + off;
  const cplx* w = pass == 2 ? V + (int64_t)(j + 1) * NS : A.w + (int64_t)b * NS + off;
  cplx* part = A.cpart + ((int64_t)b * gridDim.x + blockIdx.x) * A.ldp;
  const int64_t chunk = (N + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(N, lo + chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  extern __shared__ double4 smem_raw[];
  cplx* usum = reinterpret_cast<cplx*>(smem_raw);   // [MD_UNITS]
  cplx* ws = usum + MD_UNITS;                       // this CTA's chunk of w
  const int len = hi > lo ? (int)(hi - lo) : 0;
  double wsq = 0;
  for (int t = threadIdx.x; t < len; t += KT) {
    const cplx a = w[lo + t];
    ws[t] = a;
    wsq += a.x * a.x + a.y * a.y;
  }
  if (wn) {   // ||w||^2 partial of this CTA: warp shuffles, then warps in a fixed order
#pragma unroll
    for (int o = 16; o; o >>= 1) wsq += __shfl_xor_sync(0xffffffffu, wsq, o);
    if (lane == 0) usum[MD_UNITS - 1 - warp] = cmake(wsq, 0);
  }
  __syncthreads();
  double wsum = 0;
  if (wn && threadIdx.x == 0)
    for (int q = 0; q < KT / 32; ++q) wsum += usum[MD_UNITS - 1 - q].x;
  const int S = max(1, min(8, (4 * (KT / 32) + nv - 1) / nv));   // sub-chunks per vector
  const int sl = (len + S - 1) / S;
  const int units = nv * S;
  for (int u = warp; u < units; u += KT / 32) {
    const int q = u / S, sub = u - q * S;
    const int c0 = sub * sl, c1 = min(len, c0 + sl);
    const cplx* vq = V + (int64_t)q * NS + lo;
    cplx a0 = cmake(0, 0), a1 = cmake(0, 0);
    for (int i = c0 + lane; i < c1; i += 256) {
      cplx v[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) v[t] = (i + 32 * t < c1) ? __ldg(&vq[i + 32 * t]) : cmake(0, 0);
#pragma unroll
      for (int t = 0; t < 8; t += 2) {
        const cplx w0 = (i + 32 * t < c1) ? ws[i + 32 * t] : cmake(0, 0);
        const cplx w1 = (i + 32 * t + 32 < c1) ? ws[i + 32 * t + 32] : cmake(0, 0);
        a0.x = fma(v[t].x, w0.x, fma(v[t].y, w0.y, a0.x));
        a0.y = fma(v[t].x, w0.y, fma(-v[t].y, w0.x, a0.y));
        a1.x = fma(v[t + 1].x, w1.x, fma(v[t + 1].y, w1.y, a1.x));
        a1.y = fma(v[t + 1].x, w1.y, fma(-v[t + 1].y, w1.x, a1.y));
      }
    }
    cplx acc = cadd(a0, a1);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) usum[u] = acc;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < nv; q += KT) {
    cplx acc = cmake(0, 0);
    for (int sub = 0; sub < S; ++sub) acc = cadd(acc, usum[q * S + sub]);
    part[q] = acc;
  }
  if (wn && threadIdx.x == 0) part[nv] = cmake(wsum, 0);
  // Column sums over the CTAs in two deterministic levels: the last CTA of each
  // group of MD_GROUP CTAs folds the group's partial rows into the group's first
  // row, the last group finisher folds the group rows.  Each finisher reads
  // <= MD_GROUP (resp. ngroups) rows with coalesced, independent loads, so the
  // serial tail of a launch is two short reductions instead of one CTA reading
  // all nblk rows.
  const int cnt = nv + (wn ? 1 : 0);
  const int grp = blockIdx.x / MD_GROUP, ngrp = (gridDim.x + MD_GROUP - 1) / MD_GROUP;
  const int r0 = grp * MD_GROUP, nr = min((int)gridDim.x, r0 + MD_GROUP) - r0;
  cplx* P0 = A.cpart + (int64_t)b * gridDim.x * A.ldp;
  if (!last_of(A.gcounter + (int64_t)b * A.ldg + grp, nr)) return;
  cplx s = colsum(P0 + (int64_t)r0 * A.ldp, A.ldp, nr, cnt, usum);
  if (ngrp > 1) {
    if (threadIdx.x < cnt) P0[(int64_t)r0 * A.ldp + threadIdx.x] = s;
    if (threadIdx.x == 0) A.gcounter[(int64_t)b * A.ldg + grp] = 0u;
    if (!last_of(A.counter + b, ngrp)) return;
    s = colsum(P0, (int64_t)MD_GROUP * A.ldp, ngrp, cnt, usum);
    if (threadIdx.x == 0) A.counter[b] = 0u;
  } else if (threadIdx.x == 0) {
    A.gcounter[(int64_t)b * A.ldg + grp] = 0u;
  }
  const int q = threadIdx.x;
  if (q < cnt) {
    cplx* Hcol = A.H + (int64_t)b * A.HB + (int64_t)j * A.ldh;
    cplx* y = A.y + (int64_t)b * A.ldv;
    if (A.slabred) A.red[(int64_t)b * A.ldr + q] = s;
    else if (q == nv) A.wnorm2[b] = s.x;
    else if (pass == 2) y[q] = cscale(s, A.vscale[(int64_t)b * A.ldv + q]);
    else Hcol[q] = cscale(s, A.vscale[(int64_t)b * A.ldv + q]);
  }
}

// slabred: H column j = vscale * (sum over the entries of the partials)
__global__ void k_mdot_fin(KArgs A, int B, int pass) {
  const int b = blockIdx.x;
  if (A.ks.status[b]) return;
  if (pass == 2 && !A.reo[b]) return;
  const int j = *A.jdev;
  const bool wn = pass == 1 && A.reorth == 1;
  cplx* Hcol = A.H + (int64_t)b * A.HB + (int64_t)j * A.ldh;
  cplx* y = A.y + (int64_t)b * A.ldv;
  for (int q = threadIdx.x; q <= j + (wn ? 1 : 0); q += blockDim.x) {
    cplx s = cmake(0, 0);
    for (int e = 0; e < B; ++e) s = cadd(s, A.red[(int64_t)e * A.ldr + q]);
    if (q == j + 1) A.wnorm2[b] = s.x;
    else if (pass == 2) y[q] = cscale(s, A.vscale[(int64_t)b * A.ldv + q]);
    else Hcol[q] = cscale(s, A.vscale[(int64_t)b * A.ldv + q]);
  }
}

__device__ void givens_tail(const KArgs& A, int b, int j, double ssum);
__device__ void givens_core(const KArgs& A, int b, int j, double ssum, cplx* Hcol, const double* csp,
                            const cplx* snp);
__device__ void update_tail(const KArgs& A, int b, int j, double ssum, int pass);

// w' = w - sum_i (H_i vscale_i) V_i -> V[j+1] ; ||w'||^2 ; last block:
// h_{j+1,j} = ||w'||, vscale_{j+1}, Givens on column j, status.
// pass 2 (reorth): V[j+1] <- V[j+1] - sum_i (y_i vscale_i) V_i in place, with y = h2.
__global__ void __launch_bounds__(KT, 5) k_update(KArgs A, int pass) {
  const int b = blockIdx.y;
  if (A.ks.status[b]) return;
  if (pass == 2 && !A.reo[b]) return;
  __shared__ cplx cf[KMAX_CF];
  __shared__ cplx sh[KT / 32];
  const int j = *A.jdev;
  const int nv = j + 1;
  int64_t off, N;
  owned_view(A, b, off, N);
  const int64_t NS = A.Nst;
  const cplx* hsrc = pass == 2 ? A.y + (int64_t)b * A.ldv : A.H + (int64_t)b * A.HB + (int64_t)j * A.ldh;
  const double* vs = A.vscale + (int64_t)b * A.ldv;
  for (int q = threadIdx.x; q < KMAX_CF; q += KT) cf[q] = q < nv ? cscale(hsrc[q], vs[q]) : cmake(0, 0);
  __syncthreads();
  const cplx* V = A.V + (int64_t)b * A.Vbs + off;
  cplx* Vout = A.V + (int64_t)b * A.Vbs + (int64_t)(j + 1) * NS + off;
  const cplx* w = pass == 2 ? Vout : A.w + (int64_t)b * NS + off;
  const int64_t chunk = (N + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(N, lo + chunk);
  double nrm = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += KT) {
    cplx a = w[i], a2 = cmake(0, 0);
    for (int q = 0; q < nv; q += 8) {   // 8 independent (predicated) loads in flight
      cplx v[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) v[t] = (q + t < nv) ? __ldg(&V[(int64_t)(q + t) * NS + i]) : cmake(0, 0);
#pragma unroll
      for (int t = 0; t < 8; t += 2) {
        cfms(a, cf[q + t], v[t]);
        cfms(a2, cf[q + t + 1], v[t + 1]);
      }
    }
    a = cadd(a, a2);
    Vout[i] = a;
    nrm += a.x * a.x + a.y * a.y;
  }
  const cplx r = block_sum(cmake(nrm, 0), sh);
  double* dpart = A.dpart + (int64_t)b * gridDim.x;
  if (threadIdx.x == 0) dpart[blockIdx.x] = r.x;
  if (!last_block(A.counter + b)) return;
  const double ssum = block_sum(cmake(grid_partial_sum(dpart), 0), sh).x;   // thread 0
  // Tail (update_tail's decisions, then the Givens step) with H column j and
  // the previous rotations staged in shared memory by the whole CTA: the
  // rotation recurrence then runs on shared-memory operands instead of a chain
  // of dependent L2 round trips (one per previous rotation).
  __shared__ int go;
  __shared__ double scs[KMAX_RESTART];
  __shared__ cplx ssn[KMAX_RESTART];
  if (threadIdx.x == 0) {
    A.counter[b] = 0u;
    int g = 0;
    if (A.slabred) A.red2[b] = ssum;
    else if (pass == 2) { A.reo[b] = 0; g = 1; }
    else if (A.reorth == 2 || (A.reorth == 1 && ssum < 0.5 * A.wnorm2[b])) A.reo[b] = 1;   // second pass finishes the step
    else { if (A.reorth) A.reo[b] = 0; g = 1; }
    go = g;
  }
  __syncthreads();
  if (!go) return;
  cplx* Hcol = A.H + (int64_t)b * A.HB + (int64_t)j * A.ldh;
  const cplx* y2 = A.y + (int64_t)b * A.ldv;
  cplx* sH = cf;   // KMAX_CF >= j + 2
  for (int q = threadIdx.x; q <= j; q += KT) sH[q] = pass == 2 ? cadd(Hcol[q], y2[q]) : Hcol[q];
  for (int q = threadIdx.x; q < j; q += KT) {
    scs[q] = A.cs[(int64_t)b * A.ldv + q];
    ssn[q] = A.sn[(int64_t)b * A.ldv + q];
  }
  __syncthreads();
  if (threadIdx.x == 0) givens_core(A, b, j, ssum, sH, scs, ssn);
  __syncthreads();
  for (int q = threadIdx.x; q <= j + 1; q += KT) Hcol[q] = sH[q];
}

// slabred: ||w'||^2 = sum over the entries, then the Givens tail
__global__ void k_update_fin(KArgs A, int B, int pass) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || A.ks.status[b]) return;
  if (pass == 2 && !A.reo[b]) return;
  double ssum = 0;
  for (int e = 0; e < B; ++e) ssum += A.red2[e];
  update_tail(A, b, *A.jdev, ssum, pass);
}

// after the update pass: reorth = 1 decides the second pass by the DGKS
// criterion ||w'|| < ||w|| / sqrt 2 (oracle fgmres.py), reorth = 2
// always takes it; the second pass folds h2 into H column j, then Givens.
__device__ void update_tail(const KArgs& A, int b, int j, double ssum, int pass) {
  if (pass == 2) {
    cplx* Hcol = A.H + (int64_t)b * A.HB + (int64_t)j * A.ldh;
    const cplx* y = A.y + (int64_t)b * A.ldv;
    for (int q = 0; q <= j; ++q) Hcol[q] = cadd(Hcol[q], y[q]);
    A.reo[b] = 0;
    givens_tail(A, b, j, ssum);
    return;
  }
  if (A.reorth == 2 || (A.reorth == 1 && ssum < 0.5 * A.wnorm2[b])) {
    A.reo[b] = 1;   // the second pass finishes this step
    return;
  }
  if (A.reorth) A.reo[b] = 0;
  givens_tail(A, b, j, ssum);
}

// h_{j+1,j} = sqrt(ssum), vscale_{j+1}, Givens rotations on column j, status
__device__ void givens_tail(const KArgs& A, int b, int j, double ssum) {
  givens_core(A, b, j, ssum, A.H + (int64_t)b * A.HB + (int64_t)j * A.ldh, A.cs + (int64_t)b * A.ldv,
              A.sn + (int64_t)b * A.ldv);
}

// the Givens step on H column j at Hcol (global, or staged in shared memory by
// the caller, which writes it back); previous rotations read from csp / snp
__device__ void givens_core(const KArgs& A, int b, int j, double ssum, cplx* Hcol, const double* csp,
                            const cplx* snp) {
  const double hn = sqrt(ssum);
  double* vsw = A.vscale + (int64_t)b * A.ldv;
  double* cs = A.cs + (int64_t)b * A.ldv;
  cplx* sn = A.sn + (int64_t)b * A.ldv;
  cplx* g = A.g + (int64_t)b * A.ldv;
  Hcol[j + 1] = cmake(hn, 0);
  vsw[j + 1] = hn > 0 ? 1.0 / hn : 0.0;
  for (int i = 0; i < j; ++i) {       // previous rotations on column j
    const cplx hi0 = Hcol[i], hi1 = Hcol[i + 1];
    const double c = csp[i];
    const cplx s = snp[i];
    cplx a = cscale(hi0, c);
    cfma(a, s, hi1);
    cplx bb = cscale(hi1, c);
    cfms(bb, cmake(s.x, -s.y), hi0);
    Hcol[i] = a;
    Hcol[i + 1] = bb;
  }
  const cplx a = Hcol[j], bq = Hcol[j + 1];
  double c;
  cplx s;
  const double aa = sqrt(cabs2(a)), bb = sqrt(cabs2(bq));
  if (bb == 0.0) { c = 1.0; s = cmake(0, 0); }
  else if (aa == 0.0) { c = 0.0; s = cmake(1, 0); }
  else {
    const double t = sqrt(aa * aa + bb * bb);
    c = aa / t;
    s = cscale(cmul(cscale(a, 1.0 / aa), cmake(bq.x, -bq.y)), 1.0 / t);
  }
  cs[j] = c;
  sn[j] = s;
  cplx r0 = cscale(a, c);
  cfma(r0, s, bq);
  Hcol[j] = r0;
  Hcol[j + 1] = cmake(0, 0);
  const cplx gj = g[j];
  const cplx gj1 = cmul(cmake(-s.x, s.y), gj);   // -conj(s) g_j
  g[j + 1] = gj1;
  g[j] = cscale(gj, c);
  const double res = sqrt(cabs2(gj1));
  const int its = A.ks.its[b] + 1;
  A.ks.its[b] = its;
  A.ks.jend[b] = j + 1;
  A.ks.res[b] = res;
  const double bn = A.ks.bnorm[b];
  if (its < A.hist_len) A.ks.hist[(int64_t)b * A.hist_len + its] = res / bn;
  int stt = 0;
  if (!(res == res) || !(hn == hn) || isinf(hn)) stt = HHK_NAN;
  else if (A.fixed_iters > 0) { if (its >= A.fixed_iters) stt = HHK_FIXED; }
  else if (res <= A.rtol * bn) stt = HHK_CONVERGED;
  else if (its >= A.max_iters) stt = HHK_MAXIT;
  if (stt == 0 && hn == 0.0) stt = (res <= A.rtol * bn) ? HHK_CONVERGED : HHK_BREAKDOWN;
  A.ks.status[b] = stt;
}

__global__ void k_advance(int* jdev, int v) { *jdev = (v < 0) ? *jdev + 1 : v; }

// y = H^{-1} g (upper triangular jend x jend), one warp per sample; x += Z y
__global__ void k_trisolve(KArgs A) {
  const int b = blockIdx.x;
  const int k = A.ks.jend[b];
  if (k <= 0) return;
  __shared__ cplx rhs[KMAX_RESTART];
  const cplx* H = A.H + (int64_t)b * A.HB;
  const cplx* g = A.g + (int64_t)b * A.ldv;
  cplx* y = A.y + (int64_t)b * A.ldv;
  for (int i = threadIdx.x; i < k; i += 32) rhs[i] = g[i];
  __syncwarp();
  for (int i = k - 1; i >= 0; --i) {
    const cplx yi = cmul(rhs[i], cinv(H[i + (int64_t)i * A.ldh]));
    __syncwarp();
    for (int r = threadIdx.x; r < i; r += 32) cfms(rhs[r], H[r + (int64_t)i * A.ldh], yi);
    if (threadIdx.x == 0) y[i] = yi;
    __syncwarp();
  }
}

__global__ void __launch_bounds__(KT) k_xupdate(KArgs A, VArg xv) {
  const int b = blockIdx.y;
  const int k = A.ks.jend[b];
  if (k <= 0) return;
  __shared__ cplx ys[KMAX_RESTART];
  for (int q = threadIdx.x; q < k; q += KT) ys[q] = A.y[(int64_t)b * A.ldv + q];
  __syncthreads();
  int64_t off, N;
  owned_view(A, b, off, N);
  const cplx* Z = A.Z + (int64_t)b * A.Zbs + off;
  cplx* x = xv.at(b) + off;
  for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < N; i += (int64_t)gridDim.x * KT) {
    cplx a = x[i];
    for (int q = 0; q < k; ++q) cfma(a, ys[q], __ldg(&Z[(int64_t)q * A.Nst + i]));
    x[i] = a;
  }
}

__device__ void norm_tail(const KArgs& A, int b, int mode, double t);

// per-sample ||r||; mode 0: start (bnorm, V0 scale, g0); 1: restart; 2: true residual
__global__ void __launch_bounds__(KT) k_norm(KArgs A, VArg rv, int mode) {
  const int b = blockIdx.y;
  if (mode == 1 && A.ks.status[b]) return;
  __shared__ cplx sh[KT / 32];
  int64_t off, N;
  owned_view(A, b, off, N);
  const cplx* r = rv.at(b) + off;
  double nrm = 0;
  for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < N; i += (int64_t)gridDim.x * KT) {
    const cplx a = r[i];
    nrm += a.x * a.x + a.y * a.y;
  }
  const cplx s = block_sum(cmake(nrm, 0), sh);
  double* dpart = A.dpart + (int64_t)b * gridDim.x;
  if (threadIdx.x == 0) dpart[blockIdx.x] = s.x;
  if (!last_block(A.counter + b)) return;
  const double t = block_sum(cmake(grid_partial_sum(dpart), 0), sh).x;
  if (threadIdx.x) return;
  A.counter[b] = 0u;
  if (A.slabred) { A.red2[b] = t; return; }
  norm_tail(A, b, mode, t);
}

__global__ void k_norm_fin(KArgs A, int B, int mode) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || (mode == 1 && A.ks.status[b])) return;
  double t = 0;
  for (int e = 0; e < B; ++e) t += A.red2[e];
  norm_tail(A, b, mode, t);
}

__device__ void norm_tail(const KArgs& A, int b, int mode, double t) {
  const double nr = sqrt(t);
  if (mode == 2) { A.ks.rtrue[b] = nr; return; }
  A.vscale[(int64_t)b * A.ldv] = nr > 0 ? 1.0 / nr : 0.0;
  A.g[(int64_t)b * A.ldv] = cmake(nr, 0);
  A.ks.res[b] = nr;
  if (mode == 0) {
    A.ks.bnorm[b] = nr;
    A.ks.its[b] = 0;
    A.ks.jend[b] = 0;
    if (A.hist_len > 0) A.ks.hist[(int64_t)b * A.hist_len] = 1.0;
    A.ks.status[b] = (nr == 0.0) ? HHK_CONVERGED : 0;
  } else if (A.fixed_iters == 0 && nr <= A.rtol * A.ks.bnorm[b]) {
    A.ks.status[b] = HHK_CONVERGED;
  }
}

__global__ void k_clear_jend(KArgs A, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (A.ks.jend[b] > 0) A.ks.jlast[b] = A.ks.jend[b];
  A.ks.jend[b] = 0;
}

// |<v_a, v_c> - delta_ac| for every pair a <= c <= nv - 1 of entry b's basis
// (v_q = vscale_q V_q), one CTA per pair, fixed-order reduction
__global__ void __launch_bounds__(KT) k_orth(KArgs A, int b, int nv, double* out) {
  __shared__ cplx sh[KT / 32];
  int p = blockIdx.x, a = 0;
  while (p >= nv - a) { p -= nv - a; ++a; }
  const int c = a + p;
  int64_t off, N;
  owned_view(A, b, off, N);
  const cplx* Va = A.V + (int64_t)b * A.Vbs + (int64_t)a * A.Nst + off;
  const cplx* Vc = A.V + (int64_t)b * A.Vbs + (int64_t)c * A.Nst + off;
  cplx acc = cmake(0, 0);
  for (int64_t i = threadIdx.x; i < N; i += KT) {
    const cplx x = Va[i], y = Vc[i];
    acc.x = fma(x.x, y.x, fma(x.y, y.y, acc.x));
    acc.y = fma(x.x, y.y, fma(-x.y, y.x, acc.y));
  }
  const cplx s = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    const double* vs = A.vscale + (int64_t)b * A.ldv;
    const cplx g = cscale(s, vs[a] * vs[c]);
    out[blockIdx.x] = sqrt(cabs2(cmake(g.x - (a == c ? 1.0 : 0.0), g.y)));
  }
}

}  // namespace

// ================================================================ host side
hh_status krylov_mdot(const KArgs& A, int B, cudaStream_t s, int pass) {
  const size_t sm = (size_t)(MD_UNITS + (A.Nst + A.nblk - 1) / A.nblk) * sizeof(cplx);
  if (sm > 48 * 1024)
    HH_CUDA_TRY(smem_attr((const void*)k_mdot, sm));
  k_mdot<<<dim3(A.nblk, B), KT, sm, s>>>(A, pass);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}
hh_status krylov_update(const KArgs& A, int B, cudaStream_t s, int pass) {
  k_update<<<dim3(A.nblk, B), KT, 0, s>>>(A, pass);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}
hh_status krylov_advance(int* jdev, int v, cudaStream_t s) {
  k_advance<<<1, 1, 0, s>>>(jdev, v);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}
hh_status krylov_cycle_end(const KArgs& A, int B, VArg x, cudaStream_t s) {
  k_trisolve<<<B, 32, 0, s>>>(A);
  k_xupdate<<<dim3(A.nblk, B), KT, 0, s>>>(A, x);
  k_clear_jend<<<(B + 127) / 128, 128, 0, s>>>(A, B);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}
hh_status krylov_norm(const KArgs& A, int B, VArg r, int mode, cudaStream_t s) {
  k_norm<<<dim3(A.nblk, B), KT, 0, s>>>(A, r, mode);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}
hh_status krylov_mdot_fin(const KArgs& A, int B, cudaStream_t s, int pass) {
  k_mdot_fin<<<B, 128, 0, s>>>(A, B, pass);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}
hh_status krylov_update_fin(const KArgs& A, int B, cudaStream_t s, int pass) {
  k_update_fin<<<(B + 31) / 32, 32, 0, s>>>(A, B, pass);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}
hh_status krylov_norm_fin(const KArgs& A, int B, int mode, cudaStream_t s) {
  k_norm_fin<<<(B + 31) / 32, 32, 0, s>>>(A, B, mode);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status krylov_orth_loss(const KArgs& A, int b, double* loss, int* nvec, cudaStream_t s) {
  int jl = 0;
  HH_CUDA_TRY(cudaMemcpyAsync(&jl, A.ks.jlast + b, sizeof(int), cudaMemcpyDeviceToHost, s));
  HH_CUDA_TRY(cudaStreamSynchronize(s));
  std::vector<double> vs(jl + 1, 0.0);
  if (jl > 0)
    HH_CUDA_TRY(cudaMemcpy(vs.data(), A.vscale + (int64_t)b * A.ldv, (jl + 1) * sizeof(double),
                           cudaMemcpyDeviceToHost));
  int nv = jl + 1;
  while (nv > 0 && vs[nv - 1] == 0.0) --nv;   // a zero last vector (breakdown) is not a basis vector
  *nvec = nv;
  *loss = 0;
  if (nv <= 0) return HH_OK;
  const int np = nv * (nv + 1) / 2;
  double* d = nullptr;
  HH_CUDA_TRY(cudaMallocAsync(&d, np * sizeof(double), s));
  k_orth<<<np, KT, 0, s>>>(A, b, nv, d);
  HH_CUDA_TRY(cudaGetLastError());
  std::vector<double> h(np);
  HH_CUDA_TRY(cudaMemcpyAsync(h.data(), d, np * sizeof(double), cudaMemcpyDeviceToHost, s));
  HH_CUDA_TRY(cudaFreeAsync(d, s));
  HH_CUDA_TRY(cudaStreamSynchronize(s));
  for (double v : h) *loss = std::max(*loss, v);
  return HH_OK;
}
