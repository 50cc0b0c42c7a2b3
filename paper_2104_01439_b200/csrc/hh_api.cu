// C ABI (include/hh.h): problem setup, operator apply, V-cycle, FGMRES solve
// and the sample sweep.  Every arithmetic step runs in the CUDA kernels of
// fine2d.cu / fine3d.cu / coarse_nd.cu / krylov.cu; this file only sequences
// launches on the handle's stream.
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>
#include "hh_internal.cuh"

// ------------------------------------------------------------------ errors
static thread_local char g_err[1024] = "";
void hh_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
extern "C" const char* hh_last_error(void) { return g_err; }
extern "C" const char* hh_version(void) { return "hh-b200 0.1 (sm_100a, complex fp64)"; }

// fine-level dispatch (2D / 3D)
hh_status fine_apply2d(const Level&, int, const cplx*, cplx*, const cplx*, cudaStream_t);
hh_status fine_pre2d(const Level&, int, double, const cplx*, const double*, cplx*, cplx*, cudaStream_t);
hh_status fine_post2d(const Level&, int, double, const cplx*, const double*, const cplx*,
                      const cplx*, cplx*, cplx*, cudaStream_t);
hh_status coarse_stencil2d(const Level&, cplx*, cudaStream_t);
hh_status fine_apply3d(const Level&, int, const cplx*, cplx*, const cplx*, cudaStream_t);
hh_status fine_pre3d(const Level&, int, double, const cplx*, const double*, cplx*, cplx*, cudaStream_t);
hh_status fine_post3d(const Level&, int, double, const cplx*, const double*, const cplx*,
                      const cplx*, cplx*, cplx*, cudaStream_t);
hh_status coarse_stencil3d(const Level&, cplx*, cudaStream_t);

hh_status fine_apply(const Level& L, int op, const cplx* x, cplx* y, const cplx* sub, cudaStream_t s) {
  return L.dim == 2 ? fine_apply2d(L, op, x, y, sub, s) : fine_apply3d(L, op, x, y, sub, s);
}
hh_status fine_pre(const Level& L, int nu, double om, const cplx* f, const double* fs, cplx* u,
                   cplx* rc, cudaStream_t s) {
  return L.dim == 2 ? fine_pre2d(L, nu, om, f, fs, u, rc, s) : fine_pre3d(L, nu, om, f, fs, u, rc, s);
}
hh_status fine_post(const Level& L, int nu, double om, const cplx* f, const double* fs,
                    const cplx* u, const cplx* ec, cplx* z, cplx* w, cudaStream_t s) {
  return L.dim == 2 ? fine_post2d(L, nu, om, f, fs, u, ec, z, w, s)
                    : fine_post3d(L, nu, om, f, fs, u, ec, z, w, s);
}
hh_status coarse_stencil(const Level& C, cplx* st, cudaStream_t s) {
  return C.dim == 2 ? coarse_stencil2d(C, st, s) : coarse_stencil3d(C, st, s);
}

// krylov.cu
hh_status krylov_mdot(const cplx*, int64_t, int, const double*, const cplx*, cplx*, unsigned*,
                      cplx*, int, const int*, int, cudaStream_t);
hh_status krylov_update(const cplx*, int64_t, int, const cplx*, cplx*, double*, unsigned*, cplx*,
                        int, double*, cplx*, cplx*, double*, double*, int*, double*, int, int, int,
                        int, cudaStream_t);
hh_status krylov_trisolve(const cplx*, int, const cplx*, int, cplx*, cudaStream_t);
hh_status krylov_xupdate(const cplx*, int64_t, int, const cplx*, cplx*, int, cudaStream_t);
hh_status krylov_norm(const cplx*, int64_t, double*, unsigned*, double*, double*, cplx*, double*,
                      double, int, cudaStream_t);

// ------------------------------------------------------------------ handle
enum { T_PRE = 0, T_COARSE, T_POST, T_KRYLOV, T_NT };

struct hh_problem {
  hh_problem_desc d{};
  Level F, C;
  cudaStream_t s = nullptr;
  cplx* stencil = nullptr;
  NDFactor* nd = nullptr;
  int m = 0;
  int64_t N = 0, Nc = 0;
  cplx *V = nullptr, *Z = nullptr, *w = nullptr, *u = nullptr, *rc = nullptr, *ec = nullptr;
  cplx *bdev = nullptr, *xdev = nullptr;
  double* vscale = nullptr;
  cplx *H = nullptr, *sn = nullptr, *g = nullptr, *y = nullptr, *cpart = nullptr;
  double *cs = nullptr, *dpart = nullptr, *dscal = nullptr, *hist = nullptr;
  int* flags = nullptr;
  unsigned* counter = nullptr;
  int nblk = 0;
  int hist_len = 0;
  double setup_s = 0;
  // timers
  bool timing = false;
  std::vector<cudaEvent_t> ev;
  std::vector<int> ev_kind;   // per pair (start index 2k) the phase
  int ev_used = 0;
  int64_t launches = 0;
  double acc_ms[T_NT] = {0, 0, 0, 0};
};

namespace {
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <typename T>
hh_status dalloc(T** p, size_t count) {
  if (cudaMalloc((void**)p, std::max<size_t>(1, count) * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    hh_set_error("cudaMalloc of %.3f GB failed", count * sizeof(T) / 1e9);
    return HH_E_OOM;
  }
  return HH_OK;
}

void tmark(hh_problem* p, int kind, bool start) {
  if (!p->timing) return;
  if (start) {
    if (p->ev_used + 2 > (int)p->ev.size()) {
      for (int i = 0; i < 256; ++i) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        p->ev.push_back(e);
      }
      p->ev_kind.resize(p->ev.size() / 2 + 1);
    }
    p->ev_kind[p->ev_used / 2] = kind;
    cudaEventRecord(p->ev[p->ev_used], p->s);
  } else {
    cudaEventRecord(p->ev[p->ev_used + 1], p->s);
    p->ev_used += 2;
  }
}

void flush_timers(hh_problem* p) {
  if (!p->ev_used) return;
  cudaStreamSynchronize(p->s);
  for (int i = 0; i < p->ev_used; i += 2) {
    float ms = 0;
    cudaEventElapsedTime(&ms, p->ev[i], p->ev[i + 1]);
    p->acc_ms[p->ev_kind[i / 2]] += ms;
  }
  p->ev_used = 0;
}

hh_status setup_level(Level& L, int dim, int n, double k_const, const double* k_elem, double beta,
                      double sigma) {
  L.dim = dim;
  L.n = n;
  L.h = 1.0 / n;
  L.nodes = 1;
  L.elems = 1;
  for (int d = 0; d < dim; ++d) { L.nodes *= (n + 1); L.elems *= n; }
  L.het = (k_elem != nullptr);
  L.k_const = k_const;
  L.eps_const = beta * std::pow(k_const, sigma);
  if (L.het) {
    std::vector<double2> c(L.elems);
    for (int64_t e = 0; e < L.elems; ++e) {
      const double k = k_elem[e];
      if (!(k >= 0) || !std::isfinite(k)) { hh_set_error("k_elem[%lld] = %g invalid", (long long)e, k); return HH_E_CONFIG; }
      c[e] = make_double2(k, beta * std::pow(k, sigma));
    }
    HH_TRY(dalloc(&L.coef, L.elems));
    HH_CUDA_TRY(cudaMemcpy(L.coef, c.data(), L.elems * sizeof(double2), cudaMemcpyHostToDevice));
  }
  return HH_OK;
}

hh_status vcycle_impl(hh_problem* p, const cplx* f, const double* fscale, cplx* z, cplx* w) {
  tmark(p, T_PRE, true);
  HH_TRY(fine_pre(p->F, p->d.nu_pre, p->d.omega, f, fscale, p->u, p->rc, p->s));
  tmark(p, T_PRE, false);
  tmark(p, T_COARSE, true);
  HH_TRY(nd_solve(p->nd, p->rc, p->ec, p->s));
  tmark(p, T_COARSE, false);
  tmark(p, T_POST, true);
  HH_TRY(fine_post(p->F, p->d.nu_post, p->d.omega, f, fscale, p->u, p->ec, z, w, p->s));
  tmark(p, T_POST, false);
  p->launches += 2 + 3 * nd_levels(p->nd);
  return HH_OK;
}
}  // namespace

extern "C" hh_status hh_setup_problem(const hh_problem_desc* d, hh_problem** out) {
  if (!d || !out) { hh_set_error("NULL argument"); return HH_E_ARG; }
  *out = nullptr;
  if (d->dim != 2 && d->dim != 3) { hh_set_error("dim must be 2 or 3 (got %d)", d->dim); return HH_E_CONFIG; }
  if (d->n_cells < 4 || d->n_cells % 2) { hh_set_error("n_cells must be even and >= 4 (got %d)", d->n_cells); return HH_E_CONFIG; }
  if (!(d->omega > 0 && d->omega <= 1)) { hh_set_error("omega must be in (0,1] (got %g)", d->omega); return HH_E_CONFIG; }
  if (d->nu_pre < 1 || d->nu_pre > 4 || d->nu_post < 1 || d->nu_post > 4) { hh_set_error("nu_pre/nu_post must be in 1..4"); return HH_E_CONFIG; }
  if (d->k_elem && !d->k_elem_coarse) { hh_set_error("k_elem_coarse required with k_elem"); return HH_E_CONFIG; }
  if (!d->k_elem && !(d->k_const >= 0)) { hh_set_error("k_const must be >= 0"); return HH_E_CONFIG; }
  if (d->max_restart < 1 || d->max_restart > 127) { hh_set_error("max_restart must be in 1..127"); return HH_E_CONFIG; }
  if (d->beta < 0 || !(d->beta == 0 || d->beta > 0)) { hh_set_error("beta must be >= 0"); return HH_E_CONFIG; }
  const double t0 = now_s();
  HH_CUDA_TRY(cudaSetDevice(d->device));
  hh_problem* p = new (std::nothrow) hh_problem();
  if (!p) return HH_E_OOM;
  p->d = *d;
  p->d.k_elem = nullptr;
  p->d.k_elem_coarse = nullptr;
  p->s = (cudaStream_t)d->stream;
  hh_status st;
#define CHK(x) do { st = (x); if (st != HH_OK) { hh_destroy_problem(p); return st; } } while (0)
  CHK(setup_level(p->F, d->dim, d->n_cells, d->k_const, d->k_elem, d->beta, d->sigma));
  CHK(setup_level(p->C, d->dim, d->n_cells / 2, d->k_const, d->k_elem_coarse, d->beta, d->sigma));
  p->N = p->F.nodes;
  p->Nc = p->C.nodes;
  const int S = d->dim == 2 ? 9 : 27;
  CHK(dalloc(&p->stencil, p->Nc * S));
  CHK(coarse_stencil(p->C, p->stencil, p->s));
  CHK(nd_create(p->C, &p->nd, p->s));
  {
    hh_status fs = nd_factor(p->nd, p->stencil, p->s);
    if (fs == HH_E_SINGULAR) {
      hh_set_error("zero pivot in the coarse factorisation (k=%g, eps=%g, h=%g)", d->k_const,
                   p->C.eps_const, p->C.h);
      hh_destroy_problem(p);
      return fs;
    }
    CHK(fs);
  }
  // Krylov workspace
  p->m = d->max_restart;
  const int m = p->m;
  CHK(dalloc(&p->V, (size_t)(m + 1) * p->N));
  CHK(dalloc(&p->Z, (size_t)m * p->N));
  CHK(dalloc(&p->w, p->N));
  CHK(dalloc(&p->u, p->N));
  CHK(dalloc(&p->bdev, p->N));
  CHK(dalloc(&p->xdev, p->N));
  CHK(dalloc(&p->rc, p->Nc));
  CHK(dalloc(&p->ec, p->Nc));
  CHK(dalloc(&p->vscale, m + 1));
  CHK(dalloc(&p->H, (size_t)(m + 1) * m));
  CHK(dalloc(&p->sn, m));
  CHK(dalloc(&p->cs, m));
  CHK(dalloc(&p->g, m + 1));
  CHK(dalloc(&p->y, m));
  p->nblk = (int)std::min<int64_t>(148 * 4, (p->N + 255) / 256);
  CHK(dalloc(&p->cpart, (size_t)p->nblk * (m + 1)));
  CHK(dalloc(&p->dpart, p->nblk));
  CHK(dalloc(&p->dscal, 8));
  CHK(dalloc(&p->flags, 4));
  CHK(dalloc(&p->counter, 1));
  p->hist_len = 4096;
  CHK(dalloc(&p->hist, p->hist_len));
  if (cudaMemsetAsync(p->counter, 0, sizeof(unsigned), p->s) != cudaSuccess) { hh_destroy_problem(p); return HH_E_CUDA; }
  if (cudaStreamSynchronize(p->s) != cudaSuccess) {
    hh_set_error("setup: %s", cudaGetErrorString(cudaGetLastError()));
    hh_destroy_problem(p);
    return HH_E_CUDA;
  }
#undef CHK
  p->setup_s = now_s() - t0;
  *out = p;
  return HH_OK;
}

extern "C" hh_status hh_layout(const hh_problem* p, int64_t* nf, int64_t* nc) {
  if (!p) { hh_set_error("NULL handle"); return HH_E_ARG; }
  if (nf) *nf = p->N;
  if (nc) *nc = p->Nc;
  return HH_OK;
}

extern "C" hh_status hh_apply_op(hh_problem* p, int32_t op, const void* x, void* y) {
  if (!p || !x || !y) { hh_set_error("NULL argument"); return HH_E_ARG; }
  if (x == y) { hh_set_error("apply_op: x and y must be distinct"); return HH_E_ARG; }
  if (op == HH_OP_A0 || op == HH_OP_AEPS)
    return fine_apply(p->F, op, (const cplx*)x, (cplx*)y, nullptr, p->s);
  if (op == HH_OP_AEPS_COARSE)
    return fine_apply(p->C, HH_OP_AEPS, (const cplx*)x, (cplx*)y, nullptr, p->s);
  hh_set_error("apply_op: unknown op %d", op);
  return HH_E_ARG;
}

extern "C" hh_status hh_vcycle(hh_problem* p, const void* f, void* z) {
  if (!p || !f || !z) { hh_set_error("NULL argument"); return HH_E_ARG; }
  return vcycle_impl(p, (const cplx*)f, nullptr, (cplx*)z, nullptr);
}

extern "C" hh_status hh_coarse_solve(hh_problem* p, const void* r, void* e) {
  if (!p || !r || !e) { hh_set_error("NULL argument"); return HH_E_ARG; }
  return nd_solve(p->nd, (const cplx*)r, (cplx*)e, p->s);
}

extern "C" hh_status hh_fgmres_solve(hh_problem* p, const void* bv, void* xv, const hh_fgmres_opts* o,
                                     hh_fgmres_report* rep, double* res_hist) {
  if (!p || !bv || !xv || !o || !rep) { hh_set_error("NULL argument"); return HH_E_ARG; }
  if (o->restart < 1 || o->restart > p->m) { hh_set_error("restart %d not in 1..%d", o->restart, p->m); return HH_E_CONFIG; }
  if (o->max_iters < 1 || o->max_iters >= p->hist_len || o->fixed_iters >= p->hist_len) { hh_set_error("max_iters out of range"); return HH_E_CONFIG; }
  const cplx* b = (const cplx*)bv;
  cplx* x = (cplx*)xv;
  cudaStream_t s = p->s;
  const int64_t N = p->N;
  const int m = o->restart;
  const int ldh = p->m + 1;
  memset(rep, 0, sizeof(*rep));
  cudaEvent_t e0, e1;
  HH_CUDA_TRY(cudaEventCreate(&e0));
  HH_CUDA_TRY(cudaEventCreate(&e1));
  HH_CUDA_TRY(cudaEventRecord(e0, s));
  HH_CUDA_TRY(cudaMemsetAsync(p->flags, 0, 4 * sizeof(int), s));
  HH_CUDA_TRY(cudaMemsetAsync(x, 0, N * sizeof(cplx), s));
  HH_CUDA_TRY(cudaMemsetAsync(p->H, 0, (size_t)ldh * p->m * sizeof(cplx), s));
  // ||b||, V[0] = b, vscale[0] = 1/||b||, g[0] = ||b||
  HH_TRY(krylov_norm(b, N, p->dpart, p->counter, p->dscal + 4, p->vscale, p->g, p->dscal, o->rtol,
                     p->nblk, s));
  HH_CUDA_TRY(cudaMemcpyAsync(p->V, b, N * sizeof(cplx), cudaMemcpyDeviceToDevice, s));
  double bnorm = 0;
  HH_CUDA_TRY(cudaMemcpyAsync(&bnorm, p->dscal, sizeof(double), cudaMemcpyDeviceToHost, s));
  HH_CUDA_TRY(cudaStreamSynchronize(s));
  p->launches += 1;
  if (bnorm == 0.0) {
    rep->converged = 1;
    rep->setup_s = p->setup_s;
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    return HH_OK;
  }
  int total = 0, restarts = 0;
  bool done = false;
  double lsq = 1.0;
  hh_status result = HH_OK;
  while (!done) {
    int j_end = 0;
    for (int j = 0; j < m; ++j) {
      cplx* Vj = p->V + (int64_t)j * N;
      cplx* Zj = p->Z + (int64_t)j * N;
      HH_TRY(vcycle_impl(p, Vj, p->vscale + j, Zj, p->w));
      tmark(p, T_KRYLOV, true);
      HH_TRY(krylov_mdot(p->V, N, j + 1, p->vscale, p->w, p->cpart, p->counter,
                         p->H + (int64_t)j * ldh, 0, nullptr, p->nblk, s));
      HH_TRY(krylov_update(p->V, N, j + 1, p->w, p->V + (int64_t)(j + 1) * N, p->dpart, p->counter,
                           p->H, ldh, p->cs, p->sn, p->g, p->vscale, p->dscal, p->flags, p->hist,
                           j, total + 1, 1, p->nblk, s));
      tmark(p, T_KRYLOV, false);
      p->launches += 2;
      ++total;
      j_end = j + 1;
      int fl[4];
      HH_CUDA_TRY(cudaMemcpyAsync(fl, p->flags, sizeof(fl), cudaMemcpyDeviceToHost, s));
      HH_CUDA_TRY(cudaStreamSynchronize(s));
      if (fl[3]) { hh_set_error("FGMRES: NaN/Inf in the Arnoldi recurrence"); result = HH_E_DIVERGED; done = true; break; }
      if (o->fixed_iters > 0) {
        if (total >= o->fixed_iters) { done = true; break; }
      } else if (fl[1] || total >= o->max_iters) {
        done = true;
        break;
      }
      if (fl[2]) { done = true; break; }   // happy breakdown
    }
    // y = H^{-1} g ; x += Z y
    HH_TRY(krylov_trisolve(p->H, ldh, p->g, j_end, p->y, s));
    HH_TRY(krylov_xupdate(p->Z, N, j_end, p->y, x, p->nblk, s));
    p->launches += 2;
    double res = 0;
    HH_CUDA_TRY(cudaMemcpyAsync(&res, p->dscal + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
    HH_CUDA_TRY(cudaStreamSynchronize(s));
    lsq = res / bnorm;
    if (done) break;
    // restart: V[0] = b - A_0 x
    ++restarts;
    HH_TRY(fine_apply(p->F, HH_OP_A0, x, p->V, b, s));
    HH_CUDA_TRY(cudaMemsetAsync(p->H, 0, (size_t)ldh * p->m * sizeof(cplx), s));
    HH_CUDA_TRY(cudaMemsetAsync(p->flags, 0, 4 * sizeof(int), s));
    HH_TRY(krylov_norm(p->V, N, p->dpart, p->counter, p->dscal + 1, p->vscale, p->g, nullptr, 0,
                       p->nblk, s));
    p->launches += 2;
    double rn = 0;
    HH_CUDA_TRY(cudaMemcpyAsync(&rn, p->dscal + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
    HH_CUDA_TRY(cudaStreamSynchronize(s));
    lsq = rn / bnorm;
    if (o->fixed_iters == 0 && rn <= o->rtol * bnorm) done = true;
  }
  // true residual ||b - A_0 x|| / ||b||
  HH_TRY(fine_apply(p->F, HH_OP_A0, x, p->w, b, s));
  HH_TRY(krylov_norm(p->w, N, p->dpart, p->counter, p->dscal + 5, nullptr, nullptr, nullptr, 0,
                     p->nblk, s));
  p->launches += 2;
  double rt = 0;
  HH_CUDA_TRY(cudaMemcpyAsync(&rt, p->dscal + 5, sizeof(double), cudaMemcpyDeviceToHost, s));
  HH_CUDA_TRY(cudaEventRecord(e1, s));
  HH_CUDA_TRY(cudaStreamSynchronize(s));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  flush_timers(p);
  rep->iterations = total;
  rep->restarts = restarts;
  rep->rel_res_lsq = lsq;
  rep->rel_res_true = rt / bnorm;
  rep->converged = o->fixed_iters > 0 ? (rep->rel_res_true <= o->rtol) : (lsq <= o->rtol);
  rep->rho = total > 0 ? std::pow(rep->rel_res_true, 1.0 / total) : NAN;
  rep->setup_s = p->setup_s;
  rep->solve_s = ms * 1e-3;
  if (res_hist) {
    std::vector<double> h(total + 1);
    HH_CUDA_TRY(cudaMemcpy(h.data(), p->hist, (total + 1) * sizeof(double), cudaMemcpyDeviceToHost));
    h[0] = 1.0;
    memcpy(res_hist, h.data(), (total + 1) * sizeof(double));
  }
  return result;
}

extern "C" hh_status hh_fgmres_solve_host(hh_problem* p, const void* b_host, void* x_host,
                                          const hh_fgmres_opts* o, hh_fgmres_report* r) {
  if (!p || !b_host || !x_host) { hh_set_error("NULL argument"); return HH_E_ARG; }
  HH_CUDA_TRY(cudaMemcpyAsync(p->bdev, b_host, p->N * sizeof(cplx), cudaMemcpyHostToDevice, p->s));
  HH_TRY(hh_fgmres_solve(p, p->bdev, p->xdev, o, r, nullptr));
  HH_CUDA_TRY(cudaMemcpyAsync(x_host, p->xdev, p->N * sizeof(cplx), cudaMemcpyDeviceToHost, p->s));
  HH_CUDA_TRY(cudaStreamSynchronize(p->s));
  return HH_OK;
}

extern "C" hh_status hh_sweep(const hh_problem_desc* common, const hh_fgmres_opts* o,
                              const hh_sample* smp, int32_t n, hh_sample_result* out) {
  if (!common || !o || (!smp && n) || (!out && n)) { hh_set_error("NULL argument"); return HH_E_ARG; }
  for (int i = 0; i < n; ++i) {
    hh_problem_desc d = *common;
    d.dim = 2;
    d.n_cells = smp[i].n_cells;
    d.k_const = smp[i].k;
    d.k_elem = d.k_elem_coarse = nullptr;
    d.beta = smp[i].beta;
    d.sigma = smp[i].sigma;
    if (d.max_restart < o->restart) d.max_restart = o->restart;
    hh_sample_result& r = out[i];
    memset(&r, 0, sizeof(r));
    r.id = smp[i].id;
    hh_problem* p = nullptr;
    hh_status st = hh_setup_problem(&d, &p);
    if (st != HH_OK) { r.status = st; continue; }
    // unit point source at the centre node (BASELINE configs[1], reading C7)
    const int64_t nn = d.n_cells + 1;
    const int64_t ctr = (d.n_cells / 2) + nn * (d.n_cells / 2);
    const cplx one = cmake(1.0, 0.0);
    st = HH_OK;
    if (cudaMemsetAsync(p->bdev, 0, p->N * sizeof(cplx), p->s) != cudaSuccess ||
        cudaMemcpyAsync(p->bdev + ctr, &one, sizeof(cplx), cudaMemcpyHostToDevice, p->s) != cudaSuccess)
      st = HH_E_CUDA;
    hh_fgmres_report rep{};
    if (st == HH_OK) st = hh_fgmres_solve(p, p->bdev, p->xdev, o, &rep, nullptr);
    r.status = st;
    r.iterations = rep.iterations;
    r.converged = rep.converged;
    r.rel_res_true = rep.rel_res_true;
    r.rho = rep.rho;
    r.setup_s = p->setup_s;
    r.solve_s = rep.solve_s;
    hh_destroy_problem(p);
  }
  return HH_OK;
}

extern "C" hh_status hh_destroy_problem(hh_problem* p) {
  if (!p) return HH_OK;
  cudaFree(p->F.coef); cudaFree(p->C.coef); cudaFree(p->stencil);
  nd_destroy(p->nd);
  cudaFree(p->V); cudaFree(p->Z); cudaFree(p->w); cudaFree(p->u); cudaFree(p->rc); cudaFree(p->ec);
  cudaFree(p->bdev); cudaFree(p->xdev); cudaFree(p->vscale); cudaFree(p->H); cudaFree(p->sn);
  cudaFree(p->g); cudaFree(p->y); cudaFree(p->cpart); cudaFree(p->cs); cudaFree(p->dpart);
  cudaFree(p->dscal); cudaFree(p->hist); cudaFree(p->flags); cudaFree(p->counter);
  for (auto e : p->ev) cudaEventDestroy(e);
  delete p;
  return HH_OK;
}

extern "C" hh_status hh_reset_timers(hh_problem* p, int32_t enable) {
  if (!p) return HH_E_ARG;
  flush_timers(p);
  p->timing = enable != 0;
  for (double& a : p->acc_ms) a = 0;
  p->launches = 0;
  return HH_OK;
}

extern "C" hh_status hh_read_timers(hh_problem* p, double* ms4, int64_t* launches) {
  if (!p) return HH_E_ARG;
  flush_timers(p);
  if (ms4) for (int i = 0; i < T_NT; ++i) ms4[i] = p->acc_ms[i];
  if (launches) *launches = p->launches;
  return HH_OK;
}
