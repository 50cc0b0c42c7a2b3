// Internal declarations of the B200 hot path (not part of the ABI).
//
// Everything is BATCHED: a batch holds B problems that share the grid (dim, n)
// and differ in coefficients (k, beta, sigma, or a full k_e field).  A single
// problem is a batch of one.  Sample b of a batch is blockIdx.z (stencil
// kernels) / blockIdx.y (Krylov kernels) / a flattened index (ND kernels).
// Per-sample status (0 = running) masks finished samples out of every launch.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>
#include "../../include/hh.h"

// ---------------------------------------------------------------- complex fp64
typedef double2 cplx;   // (re, im), 16 B: same bytes as torch.complex128

// largest FGMRES restart length m (hh_problem_desc.max_restart, hh_fgmres_opts.restart):
// the Krylov kernels stage m + 1 coefficients in fixed shared arrays
constexpr int KMAX_RESTART = 127;

__host__ __device__ __forceinline__ cplx cmake(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ cplx cscale(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
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

// ---------------------------------------------------------------- batched refs
// Vector argument: sample b, Krylov slot (*j + jo) -> p + b*bs + (*j+jo)*vs
struct VArg {
  cplx* p = nullptr;
  int64_t bs = 0, vs = 0;
  const int* j = nullptr;
  int jo = 0;
  __device__ __forceinline__ cplx* at(int b) const {
    return p + (int64_t)b * bs + (j ? (int64_t)(__ldg(j) + jo) * vs : 0);
  }
};
// Scalar argument (e.g. vscale[j]) -> p[b*bs + *j + jo], or 1 if p == NULL
struct SArg {
  const double* p = nullptr;
  int64_t bs = 0;
  const int* j = nullptr;
  int jo = 0;
  __device__ __forceinline__ double at(int b) const {
    return p ? p[(int64_t)b * bs + (j ? __ldg(j) + jo : 0)] : 1.0;
  }
};
inline VArg varg(cplx* p, int64_t bs, int64_t vs = 0, const int* j = nullptr, int jo = 0) {
  VArg a; a.p = p; a.bs = bs; a.vs = vs; a.j = j; a.jo = jo; return a;
}
inline SArg sarg(const double* p, int64_t bs, const int* j = nullptr, int jo = 0) {
  SArg a; a.p = p; a.bs = bs; a.j = j; a.jo = jo; return a;
}

// ---------------------------------------------------------------- levels
// Geometry + coefficients of one level for a batch of B entries.
//
// Slab layout (fine level): entry b owns the global planes [z0, z1) of the
// slowest axis (y in 2D, z in 3D; slab[b] = (z0, z1)) and stores the planes
// [z0 - G, z1 + G) (G ghost planes per side, filled by the halo exchange) in a
// buffer of `stride` nodes.  Kernels index vectors with GLOBAL node numbers
// through the virtual base  p - (z0 - G) * plane.  An independent sample is an
// entry with (z0, z1) = (0, n+1); the coarse level has slab == NULL, G = 0.
struct Level {
  int dim = 2;
  int n = 0;            // cells per side
  int64_t nodes = 0;    // (n+1)^dim (global)
  int64_t elems = 0;    // n^dim
  int64_t plane = 0;    // (n+1)^(dim-1)
  double h = 0;
  bool het = false;
  const double2* coef = nullptr;   // het: (k_e, eps_e) per element, global
  int64_t coef_bs = 0;             // entry stride of coef (0: shared by all entries)
  const double2* kc = nullptr;     // constant: [B] (k, eps)
  cplx* tmp = nullptr;             // 3D only: [B][2][stride] scratch owned by the engine
  const int2* slab = nullptr;      // device [B] (z0, z1), NULL = whole domain
  int G = 0;                       // ghost planes per side
  int maxloc = 0;                  // max owned planes over the entries (n+1 without slabs)
  int64_t stride = 0;              // entry stride of fine vectors: (maxloc + 2G) * plane
  cplx* dinv = nullptr;            // het fine level: D^{-1} = diag(A_eps)^{-1} per node (vector layout)
};

// Raise a kernel's dynamic shared-memory limit to at least `bytes`, never lower
// it: engines on several host threads launch the same kernel with different
// sizes, and a concurrent lower setting would make a larger launch fail.
cudaError_t smem_attr(const void* fn, size_t bytes);

__device__ __forceinline__ int2 slab_of(const int2* sl, int b, int n) {
  return sl ? sl[b] : make_int2(0, n + 1);
}

// fine-level kernels (fine2d.cu / fine3d.cu); st: per-sample status (NULL = all run)
hh_status fine_apply(const Level& L, int B, const int* st, int op, VArg x, VArg y, VArg sub,
                     cudaStream_t s);
hh_status fine_pre(const Level& L, int B, const int* st, int nu, double omega, VArg f, SArg fs,
                   VArg u, VArg rc, cudaStream_t s);
hh_status fine_post(const Level& L, int B, const int* st, int nu, double omega, VArg f, SArg fs,
                    VArg u, VArg ec, VArg z, VArg w, cudaStream_t s);
hh_status coarse_stencil(const Level& C, int B, cplx* st, cudaStream_t s);
// L.dinv = diag(A_eps)^{-1} at every stored node of every entry (setup; het levels)
hh_status fine_dinv(const Level& L, int B, cudaStream_t s);

// ---------------------------------------------------------------- coarse ND solver
struct NDPlan;                       // host+device tree data for one (dim, m); shareable
hh_status nd_plan_create(int dim, int m, NDPlan** out);
void nd_plan_destroy(NDPlan* p);
int64_t nd_front_entries(const NDPlan* p);        // complex entries per sample
int64_t nd_stream_bytes(const NDPlan* p);         // bytes streamed per solve per sample
int nd_levels(const NDPlan* p);
int nd_solve_launches(const NDPlan* p, int B, bool conc = false);      // kernel launches of one nd_solve
int64_t nd_work_entries(const NDPlan* p);         // zs + out entries per sample
// zero the dataflow-solve counters in the work of B samples (after allocation)
hh_status nd_flow_reset(const NDPlan* p, int B, cplx* work, cudaStream_t s);
int64_t nd_cbuf_entries(const NDPlan* p);         // pivot column buffer per sample
// F: [B][front_entries]; stencil: [B][Nc*3^d]; work: [B][work]; cbuf: [B][cbuf]
hh_status nd_factor(const NDPlan* p, int B, const cplx* stencil, cplx* F, cplx* cbuf, int* flag,
                    cudaStream_t s);
// shareF: every entry uses the one factor at F (slabs of one problem)
// conc: the solve shares the GPU with other streams (concurrent sweep workers):
// schedules are tuned and cached separately, and the dataflow kernels (whose
// waiting CTAs hold SM slots) are not used
// Dataflow schedule failure (a dependency wait that exceeded HH_ND_FLOW_POLLS polls):
// the waiting CTA marks sample b failed -- st[b] = HHK_NDFAIL when the Krylov
// status array is given, else *fail = 1 (a caller-owned device int) -- and every
// later wait of that sample gives up; the caller must then report an error,
// nd_flow_reset the counters and nd_flow_disable the schedule.
hh_status nd_solve(const NDPlan* p, int B, const int* st, const cplx* F, cplx* work, VArg rhs,
                   VArg x, cudaStream_t s, bool shareF = false, bool conc = false, int* fail = nullptr);
// ---- coarse solve by fast diagonalisation (fd.cu; constant k, separable coarse operator)
// basis: per factor copy fd_basis_entries(nc) complex entries (folded eigenvector
// matrices V, V^T per parity + eigenvalues); work: per entry fd_work_entries.
// fd_setup: flag[b] = 1 if the secular roots fail validation, 2 if the operator is
// singular (both leave flag 0 untouched otherwise; the caller zeroes it).
int fd_P(int nc);
void fd_gemm_ctas2d(int nc, int* per_sample, int* per_sm);
int64_t fd_basis_entries(int nc);
int64_t fd_work_entries(int dim, int nc);
int fd_solve_launches(int dim);
double fd_solve_flops(int dim, int nc);     // real flops per sample and solve
int64_t fd_solve_bytes(int dim, int nc);    // compulsory HBM bytes per sample and solve
// kslot: device [nslot] k of each distinct-k basis slot; bidx: device [B] slot of
// sample b; sflag: device [nslot] ints, zeroed by the caller; flag: per sample
hh_status fd_setup(int dim, int nc, int B, int nslot, const double* kslot, const int* bidx, int* sflag,
                   const double2* kc, cplx* basis, int* flag, cudaStream_t s);
hh_status fd_flag_all(int* flag, int B, int code, cudaStream_t s);   // fault injection (HH_FD_FAIL)
hh_status fd_solve(int dim, int nc, int B, const int* st, const cplx* basis, const int* bidx, const double2* kc,
                   cplx* work, VArg rhs, VArg x, cudaStream_t s);
// ---- distributed coarse solve (slab-aligned ND; SURVEY.md 8(e) second version)
struct Comm;
struct NDDistView {            // one rank's part, held by this process
  NDPlan* plan = nullptr;      // rank view (nd_plan_create_dist)
  cplx* F = nullptr;           // nd_front_entries(plan): this rank's [X | H] rows
  cplx* scratch = nullptr;     // nd_dist_scratch_entries(plan): pivot columns | workspace (shareable)
  cplx* S = nullptr;           // nd_dist_s_entries(plan): packed Schur complements
  cplx* work = nullptr;        // nd_work_entries(plan): solve vectors
  int* flag = nullptr;         // zero-pivot flag
};
// Zc: P + 1 coarse plane bounds of the slowest axis (slab k owns [Zc[k], Zc[k+1]))
hh_status nd_plan_create_dist(int dim, int m, const std::vector<int>& Zc, int rank, NDPlan** out);
// V: the rank views of this process (all P in-process, or one with an NCCL comm);
// st: the coarse stencil of the whole grid (each rank assembles its own fronts)
hh_status nd_dist_factor(std::vector<NDDistView>& V, const cplx* st, Comm* comm, cudaStream_t s);
// rhs / x: entry k = view k (full coarse vectors, rhs complete in every entry); on
// return x holds the solution on view k's own fronts and on every interface plane,
// i.e. on its own coarse planes [Zc[r], Zc[r+1]).  stage: nd_dist_stage_entries.
hh_status nd_dist_solve(std::vector<NDDistView>& V, const int* st, VArg rhs, VArg x, Comm* comm, cplx* stage,
                        cudaStream_t s);
int64_t nd_dist_stage_entries(const NDPlan* p);
int64_t nd_dist_scratch_entries(const NDPlan* p);
int64_t nd_dist_s_entries(const NDPlan* p);
int nd_dist_launches(const std::vector<NDDistView>& V);
// transport of the distributed solve (comm.cu): grouped NCCL point-to-point / broadcast
hh_status comm_group(bool start);
hh_status comm_send(Comm* c, const void* buf, size_t bytes, int peer, cudaStream_t s);
hh_status comm_recv(Comm* c, void* buf, size_t bytes, int peer, cudaStream_t s);
hh_status comm_bcast(Comm* c, void* buf, size_t bytes, int root, cudaStream_t s);

// true if nd_solve(p, B, ..., conc) runs the dataflow kernels
bool nd_solve_uses_flow(const NDPlan* p, int B, bool conc);
// never use the dataflow schedule for this tree again (after a failure)
void nd_flow_disable(const NDPlan* p);
// choose the solve schedule for batch size B by timing candidates on the real factor;
// multi != NULL (concurrent sweep workers): time every candidate on all the given
// streams at once (throughput under concurrency instead of isolated latency)
struct NDTuneCtx { const cplx* F; cplx* work; VArg rhs, x; cudaStream_t s; };
hh_status nd_autotune(const NDPlan* p, int B, const cplx* F, cplx* work, VArg rhs, VArg x,
                      cudaStream_t s, bool shareF = false, bool conc = false,
                      const std::vector<NDTuneCtx>* multi = nullptr);
