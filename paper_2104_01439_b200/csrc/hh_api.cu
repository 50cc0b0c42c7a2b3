// C ABI (include/hh.h) and the batched engine behind it.
//
// Engine = one CUDA stream + reusable device workspace pools.  Batch = B
// problems of one grid (dim, n) set up together (coefficients, coarse stencil,
// ND factorisation) and solved in lockstep: every launch covers all B samples,
// finished samples are masked by their device status, and one FGMRES
// iteration (V-cycle + A_0 + CGS + Givens) is captured once as a CUDA graph
// and replayed with the Arnoldi index j kept in device memory.
// hh_problem = an engine + a batch of one; hh_sweep = a thread pool of
// engines draining a queue of equal-n batches.  Every arithmetic step runs in
// the kernels of fine2d.cu / fine3d.cu / coarse_nd.cu / krylov.cu.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <condition_variable>
#include <new>
#include <thread>
#include <tuple>
#include <vector>
#include "hh_internal.cuh"
#include "krylov.cuh"
#include "comm.cuh"

// ------------------------------------------------------------------ smem limits
cudaError_t smem_attr(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> set;
  if (bytes <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = set[{dev, fn}];
  if (bytes <= cur) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

// ------------------------------------------------------------------ errors
static thread_local char g_err[1024] = "";
void hh_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
extern "C" const char* hh_last_error(void) { return g_err; }
extern "C" const char* hh_version(void) { return "hh-b200 0.2 (sm_100a, complex fp64, batched)"; }

// fine-level dispatch (2D / 3D)
hh_status fine_apply2d(const Level&, int, const int*, int, VArg, VArg, VArg, cudaStream_t);
hh_status fine_pre2d(const Level&, int, const int*, int, double, VArg, SArg, VArg, VArg, cudaStream_t);
hh_status fine_post2d(const Level&, int, const int*, int, double, VArg, SArg, VArg, VArg, VArg,
                      VArg, cudaStream_t);
hh_status coarse_stencil2d(const Level&, int, cplx*, cudaStream_t);
hh_status fine_apply3d(const Level&, int, const int*, int, VArg, VArg, VArg, cudaStream_t);
hh_status fine_pre3d(const Level&, int, const int*, int, double, VArg, SArg, VArg, VArg, cudaStream_t);
hh_status fine_post3d(const Level&, int, const int*, int, double, VArg, SArg, VArg, VArg, VArg,
                      VArg, cudaStream_t);
hh_status coarse_stencil3d(const Level&, int, cplx*, cudaStream_t);
hh_status fine_dinv2d(const Level&, int, cudaStream_t);
hh_status fine_dinv3d(const Level&, int, cudaStream_t);
hh_status fine_dinv(const Level& L, int B, cudaStream_t s) {
  return L.dim == 2 ? fine_dinv2d(L, B, s) : fine_dinv3d(L, B, s);
}

hh_status fine_apply(const Level& L, int B, const int* st, int op, VArg x, VArg y, VArg sub,
                     cudaStream_t s) {
  return L.dim == 2 ? fine_apply2d(L, B, st, op, x, y, sub, s) : fine_apply3d(L, B, st, op, x, y, sub, s);
}
hh_status fine_pre(const Level& L, int B, const int* st, int nu, double om, VArg f, SArg fs, VArg u,
                   VArg rc, cudaStream_t s) {
  return L.dim == 2 ? fine_pre2d(L, B, st, nu, om, f, fs, u, rc, s)
                    : fine_pre3d(L, B, st, nu, om, f, fs, u, rc, s);
}
hh_status fine_post(const Level& L, int B, const int* st, int nu, double om, VArg f, SArg fs,
                    VArg u, VArg ec, VArg z, VArg w, cudaStream_t s) {
  return L.dim == 2 ? fine_post2d(L, B, st, nu, om, f, fs, u, ec, z, w, s)
                    : fine_post3d(L, B, st, nu, om, f, fs, u, ec, z, w, s);
}
hh_status coarse_stencil(const Level& C, int B, cplx* st, cudaStream_t s) {
  return C.dim == 2 ? coarse_stencil2d(C, B, st, s) : coarse_stencil3d(C, B, st, s);
}

namespace {
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ------------------------------------------------------------------ small kernels
// Over a whole (ghosted) fine vector of N entries: mode 0: x = 0; mode 1: x = src;
// mode 2: unit point source at GLOBAL node `idx` (placed if entry b owns it).
__global__ void k_vset(VArg x, VArg src, int64_t N, int mode, int64_t idx, const int* st,
                       const int2* slab, int n, int G, int64_t plane) {
  const int b = blockIdx.y;
  if (st && st[b]) return;
  cplx* xb = x.at(b);
  const cplx* sb = mode == 1 ? src.at(b) : nullptr;
  int64_t loc = -1;
  if (mode == 2) {
    const int2 sl = slab_of(slab, b, n);
    if (idx >= (int64_t)sl.x * plane && idx < (int64_t)sl.y * plane) loc = idx - (int64_t)(sl.x - G) * plane;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x)
    xb[i] = mode == 1 ? sb[i] : cmake((mode == 2 && i == loc) ? 1.0 : 0.0, 0.0);
}

// Shift-exponent map sigma_p(k, l) (Eq. shiftexp) with the
// fitted weights of Table 1, rows p = 1, 2, 3:
// (k_c0, k_c1, alpha_0, alpha_1)
__host__ __device__ inline double sigma_map(double k, double l, int p) {
  const double W[3][4] = {{0.4592788619853418, 2.5790032999702346, -0.6261637288068426, 1.7580549857142198},
                          {0.5736926870738827, 2.5729974893966001, -0.6615199737374460, 1.5966386518185063},
                          {0.6305770719029798, 2.4284320222555804, -0.4465407372367102, 0.1287828338493968}};
  const double* w = W[p - 1];
  const double kc = w[1] * exp(w[0] * l);
  const double al = w[3] * exp(w[2] * l);
  const double b = 2.0 - exp(-al * (k - kc));
  return fmin(fmax(b, 1.0), 2.0);
}

// eps_e = beta k_e^sigma, sigma = the fixed exponent or sigma_p(k_e, l) (map_p > 0)
__host__ __device__ inline double shift_of(double k, double beta, double sigma, int map_p, double l) {
  return beta * pow(k, map_p > 0 ? sigma_map(k, l, map_p) : sigma);
}

// heterogeneous coefficients: c[e] = (k_e, eps_e)
__global__ void k_coef(const double* __restrict__ k, int64_t n, double beta, double sigma, int map_p,
                       double l, double2* __restrict__ c) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double ke = k[e];
    c[e] = make_double2(ke, shift_of(ke, beta, sigma, map_p, l));
  }
}

hh_status vset(const Level& L, VArg x, VArg src, int B, int mode, int64_t idx, const int* st,
               cudaStream_t s) {
  const int64_t N = L.stride;
  const unsigned gx = (unsigned)std::min<int64_t>(1024, (N + 255) / 256);
  k_vset<<<dim3(gx, B), 256, 0, s>>>(x, src, N, mode, idx, st, L.slab, L.n, L.G, L.plane);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

// ------------------------------------------------------------------ pools
// Device block cache: buffers released by a destroyed handle / engine are kept
// (per device, by size) and handed to the next setup of the same shape instead
// of going back through cudaMalloc/cudaFree, which map/unmap pages and
// synchronise the device (hundreds of ms for a multi-GB Krylov basis).  The
// cache holds at most half the device memory; a failed cudaMalloc flushes it.
struct BlockCache {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> free_blocks;
  size_t cached = 0;
  void* take(int dev, size_t want, size_t* got) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = free_blocks.lower_bound({dev, want});
    if (it == free_blocks.end() || it->first.first != dev) return nullptr;
    if (it->first.second > want + want / 4 + (size_t(8) << 20)) return nullptr;   // too wasteful
    void* p = it->second;
    *got = it->first.second;
    cached -= it->first.second;
    free_blocks.erase(it);
    return p;
  }
  std::map<int, size_t> total;   // device memory size, queried once per device
  bool give(int dev, void* p, size_t bytes) {
    size_t tot = 0;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = total.find(dev);
      if (it != total.end()) tot = it->second;
    }
    if (!tot) {
      size_t fr = 0;
      if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) { cudaGetLastError(); return false; }
      std::lock_guard<std::mutex> lk(mu);
      total[dev] = tot;
    }
    std::lock_guard<std::mutex> lk(mu);
    if (cached + bytes > tot / 2) return false;
    free_blocks.insert({{dev, bytes}, p});
    cached += bytes;
    return true;
  }
  void flush(int dev) {
    std::lock_guard<std::mutex> lk(mu);
    for (auto it = free_blocks.begin(); it != free_blocks.end();) {
      if (it->first.first == dev) {
        cudaFree(it->second);
        cached -= it->first.second;
        it = free_blocks.erase(it);
      } else {
        ++it;
      }
    }
  }
};
BlockCache& block_cache() { static BlockCache* c = new BlockCache(); return *c; }   // never destroyed

struct Pool {
  void* p = nullptr;
  size_t bytes = 0;
  int dev = 0;
  hh_status ensure(size_t b) {
    if (b <= bytes && p) return HH_OK;
    release();
    const size_t want = (std::max<size_t>(b, 256) + 511) / 512 * 512;
    cudaGetDevice(&dev);
    size_t got = 0;
    if (void* c = block_cache().take(dev, want, &got)) {   // may be larger than asked
      p = c;
      bytes = got;
      return HH_OK;
    }
    if (cudaMalloc(&p, want) != cudaSuccess) {
      cudaGetLastError();
      block_cache().flush(dev);
      if (cudaMalloc(&p, want) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        hh_set_error("cudaMalloc of %.3f GB failed", want / 1e9);
        return HH_E_OOM;
      }
    }
    bytes = want;
    return HH_OK;
  }
  template <typename T> T* as() const { return (T*)p; }
  void release() {
    if (p && !block_cache().give(dev, p, bytes)) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

// ND plans are shared by every engine (tree depends on (dim, m) only)
// (per device: a plan holds device arrays of the device current at creation)
std::mutex g_plan_mu;
std::map<std::tuple<int, int, int>, NDPlan*> g_plans;   // (device, dim, m)
hh_status get_plan(int dim, int m, NDPlan** out) {
  int dev = 0;
  HH_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto it = g_plans.find({dev, dim, m});
  if (it != g_plans.end()) { *out = it->second; return HH_OK; }
  NDPlan* p = nullptr;
  HH_TRY(nd_plan_create(dim, m, &p));
  g_plans[{dev, dim, m}] = p;
  *out = p;
  return HH_OK;
}

// rank views of distributed (slab-aligned) coarse trees, per (device, dim, m, bounds, rank)
std::map<std::tuple<int, int, int, std::vector<int>, int>, NDPlan*> g_dplans;
hh_status get_dist_plan(int dim, int m, const std::vector<int>& Zc, int rank, NDPlan** out) {
  int dev = 0;
  HH_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto key = std::make_tuple(dev, dim, m, Zc, rank);
  auto it = g_dplans.find(key);
  if (it != g_dplans.end()) { *out = it->second; return HH_OK; }
  NDPlan* p = nullptr;
  HH_TRY(nd_plan_create_dist(dim, m, Zc, rank, &p));
  g_dplans[key] = p;
  *out = p;
  return HH_OK;
}

enum { T_PRE = 0, T_COARSE, T_POST, T_KRYLOV, T_NT };

struct BatchSpec {
  int dim = 2, n = 0, B = 1, nu_pre = 2, nu_post = 2, m = 100;
  double omega = 0.6;
  std::vector<double> k, beta, sigma;    // per entry (constant k)
  const double* kf = nullptr;            // het (one problem): host per-element k
  const double* kcoarse = nullptr;
  // slab decomposition: the B entries are the slabs [slab_first, slab_first + B) of
  // one problem cut into slabs_total slabs (reductions over the entries + comm)
  bool slabmode = false;
  int slabs_total = 1, slab_first = 0;
  Comm* comm = nullptr;
  int shift_map = 0;                     // > 0: sigma = sigma_p(k_e, log2 n) of Table 1 row p
  bool dist = false;                     // slab mode: distributed coarse solve (HH_COARSE_ND_DIST)
  int coarse = HH_COARSE_AUTO;           // requested HH_COARSE_* (AUTO: FD falls back to ND on failure)
  bool fd = false;                       // coarse solve by fast diagonalisation (fd.cu; constant k)
};

// AUTO's choice of the fast-diagonalisation coarse solve (fd.cu): constant k,
// no distributed factor, and a size where its dense transforms beat the ND
// factor (2D: 16 m^3 flops per solve against O(m^2 log m) bytes -- the GEMMs
// win up to nc ~ 512 on B200; 3D: 24 m^4 flops against the O(m^4)-byte, O(m^6)-flop
// factor -- always) with a resolved coarse grid (k h_c <= 2.5, where the secular
// continuation is validated; the ND factor takes the rest)
bool fd_wanted(int req, int dim, int nc, bool het, bool dist, double kmax) {
  if (het || dist) return false;
  if (req == HH_COARSE_FD) return true;
  if (req != HH_COARSE_AUTO) return false;
  if (!(kmax / nc <= 2.5)) return false;
  return dim == 3 ? nc <= 256 : nc <= 512;
}

// fine-vector layout of a batch: G ghost planes, entry stride, slab bounds
struct FineLayout {
  int G = 0, maxloc = 0;
  int64_t plane = 0, stride = 0;
  int64_t pad = 0;           // leading pad so that every owned view starts 256-B aligned
  std::vector<int2> slabs;   // per entry
  std::vector<int> all_z;    // bounds of every process' slab range (slab mode)
};

int64_t ipow(int64_t a, int d) { int64_t r = 1; while (d--) r *= a; return r; }

FineLayout fine_layout(const BatchSpec& sp) {
  FineLayout F;
  F.G = std::max(sp.nu_pre, sp.nu_post) + 1;
  F.plane = ipow(sp.n + 1, sp.dim - 1);
  if (sp.slabmode) {
    const std::vector<int> z = slab_bounds(sp.n, sp.slabs_total);
    for (int b = 0; b < sp.B; ++b) F.slabs.push_back(make_int2(z[sp.slab_first + b], z[sp.slab_first + b + 1]));
    const int per = sp.B;   // slabs per process
    for (int q = 0; q <= sp.slabs_total / per; ++q) F.all_z.push_back(z[std::min(q * per, sp.slabs_total)]);
  } else {
    for (int b = 0; b < sp.B; ++b) F.slabs.push_back(make_int2(0, sp.n + 1));
  }
  for (const int2& z : F.slabs) F.maxloc = std::max(F.maxloc, z.y - z.x);
  F.pad = (16 - (F.G * F.plane) % 16) % 16;
  F.stride = ((F.pad + (int64_t)(F.maxloc + 2 * F.G) * F.plane + 15) / 16) * 16;
  return F;
}

// Exclusive timing gate of the concurrent sweep engines: a sampled (timed)
// iteration runs with the GPU to itself -- the other engines finish their queued
// work and launch nothing until it is done -- so its per-phase CUDA-event times
// are kernel times, not time-shared wall times.  Plain iterations take the
// gate shared (only around their launch); a waiting exclusive request blocks new
// shared entries (no starvation).
struct ExclGate {
  std::mutex mu;
  std::condition_variable cv;
  int active = 0, waiting = 0;
  bool excl = false;
  void lock_shared() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return !excl && waiting == 0; });
    ++active;
  }
  void unlock_shared() {
    std::lock_guard<std::mutex> lk(mu);
    if (--active == 0) cv.notify_all();
  }
  void lock() {
    std::unique_lock<std::mutex> lk(mu);
    ++waiting;
    cv.wait(lk, [&] { return !excl && active == 0; });
    --waiting;
    excl = true;
  }
  void unlock() {
    std::lock_guard<std::mutex> lk(mu);
    excl = false;
    cv.notify_all();
  }
};

struct SampleOut {
  int status = 0, iterations = 0, converged = 0, restarts = 0;
  double rel_res_lsq = 0, rel_res_true = 0, rho = 0;
};

struct Engine {
  int device = 0;
  bool conc = false;         // runs beside other sweep workers (ND schedule choice)
  cudaStream_t s = nullptr;
  Pool V, Z, w, u, bv, xv, tmp3, rc, ec, stc, F, cbuf, work, kcf, kcc, coef_f, coef_c, ksmall,
      cpart, dpart, hist, kstage, slabp, hstage, ustage, dinvp, dscratch, dflag, dstage, fdb, fdm;
  // distributed coarse solve: one rank view per entry (factor, packed S, work per view)
  std::vector<NDDistView> dviews;
  std::vector<Pool> dF, dS, dW;
  int* h_status = nullptr;   // pinned
  int h_cap = 0;
  // batch
  BatchSpec spec;
  Level LF, LC;
  NDPlan* plan = nullptr;
  int B = 0, m = 0, nblk = 1, hist_len = 0;
  int64_t N = 0, Nc = 0;    // global fine / coarse nodes
  FineLayout FL;
  SlabCtx X;                // slab mode transport context
  int Bf = 0;               // coarse factor copies (1 in slab mode: shared by the slabs)
  KArgs ka;
  int* jdev = nullptr;
  int* nd_flag = nullptr;
  int* flow_fail = nullptr;  // dataflow coarse-solve failure flag of the status-less calls
  const int* fd_bidx = nullptr;   // FD: basis slot of every entry (device, in fdm)
  double setup_s = 0;
  // graph of one iteration
  cudaGraphExec_t gexec = nullptr;     // plain iteration
  cudaGraphExec_t gexec_t = nullptr;   // iteration with phase events
  int64_t iter_counter = 0;
  int timing_every = 1;                // sample one iteration in timing_every
  ExclGate* gate = nullptr;            // sweep: exclusive timed iterations (HH_SWEEP_EXCL_TIMING)
  std::vector<cudaStream_t> peers;     // the other engines' streams (drained before a timed iteration)
  void drop_graphs() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (gexec_t) cudaGraphExecDestroy(gexec_t);
    gexec = gexec_t = nullptr;
  }
  // timers
  bool timing = false;
  cudaEvent_t ev[2 * T_NT] = {};
  double acc_ms[T_NT] = {0, 0, 0, 0};
  double acc_bytes[T_NT] = {0, 0, 0, 0};      // timed (sampled) iterations
  double acc_bytes_all[T_NT] = {0, 0, 0, 0};  // every iteration (aggregate throughput)
  double acc_model[T_NT] = {0, 0, 0, 0};      // SURVEY 8(d) per-step model bytes, timed iterations
  double acc_model_all[T_NT] = {0, 0, 0, 0};  // ... every iteration
  double acc_launch[T_NT] = {0, 0, 0, 0};
  double acc_flops = 0, acc_flops_all = 0;    // coarse-solve flops (FD: tensor-core GEMMs), timed / every iteration
  int64_t launches = 0;
  int64_t launches_per_iter = 0;

  // return every pool to the device block cache (the engine itself is reused)
  void release_pools() {
    Pool* all[] = {&V, &Z, &w, &u, &bv, &xv, &tmp3, &rc, &ec, &stc, &F, &cbuf, &work, &kcf, &kcc,
                   &coef_f, &coef_c, &ksmall, &cpart, &dpart, &hist, &kstage, &slabp, &hstage, &ustage, &dinvp,
                   &dscratch, &dflag, &dstage, &fdb, &fdm};
    for (Pool* p : all) p->release();
    for (auto* vp : {&dF, &dS, &dW})
      for (Pool& p : *vp) p.release();
    dviews.clear();
  }
  ~Engine() {
    drop_graphs();
    release_pools();
    if (h_status) cudaFreeHost(h_status);
    for (auto& e : ev) if (e) cudaEventDestroy(e);
    if (s) cudaStreamDestroy(s);
  }
};

hh_status engine_init(Engine& E, int device) {
  E.device = device;
  HH_CUDA_TRY(cudaSetDevice(device));
  HH_CUDA_TRY(cudaStreamCreateWithFlags(&E.s, cudaStreamNonBlocking));
  for (auto& e : E.ev) HH_CUDA_TRY(cudaEventCreate(&e));
  return HH_OK;
}

// bytes of device workspace per sample for a (dim, n, m) batch
int64_t per_sample_bytes(int dim, int n, int m, const NDPlan* plan) {   // plan == NULL: FD coarse solve
  const int64_t N = ipow(n + 1, dim + 0) + 6 * ipow(n + 1, dim - 1), Nc = ipow(n / 2 + 1, dim);
  const int S = dim == 2 ? 9 : 27;
  int64_t b = (int64_t)(2 * m + 1 + 4 + (dim == 3 ? 2 : 0)) * N * 16;
  b += Nc * (2 + S) * 16;
  if (plan) b += (nd_front_entries(plan) + nd_cbuf_entries(plan) + nd_work_entries(plan)) * 16;
  else b += (fd_basis_entries(n / 2) + fd_work_entries(dim, n / 2)) * 16;
  return b;
}

constexpr int HIST_LEN = 4096;

// Krylov CTAs per sample: enough for ONE sample to fill the GPU (the tail of a
// batch is a single slow sample), chunks of <= 2048 nodes (the multi-dot stages
// its chunk of w in shared memory); independent of B, so batched == single.
int krylov_blocks(int64_t N) {
  const int64_t a = std::min<int64_t>(148 * 4, (N + 255) / 256);
  return (int)std::max<int64_t>(1, std::max<int64_t>(a, (N + 2047) / 2048));
}

size_t ksmall_bytes(int B, int m, int nblk) {
  const size_t ldv = m + 1, ldh = m + 1, ldg = (nblk + 31) / 32;
  auto r = [](size_t b) { return (b + 255) / 256 * 256; };
  return r(B * ldg * 4) + r(B * ldv * 8) * 2 + r(B * ldv * 16) * 3 + r((size_t)B * m * ldh * 16) + r(B * 8) * 3 +
         r(B * 4) * 3 + r(16) + r(B * 4) * 2 + r(B * (ldv + 1) * 16) + r(B * 8) + r(B * 8) + r(B * 4) * 2 +
         r(16);
}

// Grow the engine's pools to hold batch `sp` (no-op when already large enough).
// cudaMalloc/cudaFree synchronise the device, so the sweep reserves every
// engine for its largest batch before any worker starts.
hh_status reserve_pools(Engine& E, const BatchSpec& sp) {
  const int B = sp.B, dim = sp.dim, n = sp.n, m = sp.m;
  const FineLayout FL = fine_layout(sp);
  const int64_t N = FL.stride, Nc = ipow(n / 2 + 1, dim);
  const int Bf = sp.slabmode ? 1 : B;
  NDPlan* P = nullptr;
  if (!sp.dist && !sp.fd) HH_TRY(get_plan(dim, n / 2 + 1, &P));   // distributed: rank views (dist_setup)
  const int S = dim == 2 ? 9 : 27;
  const int nblk = krylov_blocks((int64_t)FL.maxloc * FL.plane);
  // fine vectors: B entries of N (ghosted, padded) nodes + 16 nodes of slack for the lead pad
  HH_TRY(E.V.ensure(((size_t)B * (m + 1) * N + 16) * 16));
  HH_TRY(E.Z.ensure(((size_t)B * m * N + 16) * 16));
  HH_TRY(E.w.ensure(((size_t)B * N + 16) * 16));
  HH_TRY(E.u.ensure(((size_t)B * N + 16) * 16));
  HH_TRY(E.bv.ensure(((size_t)B * N + 16) * 16));
  HH_TRY(E.xv.ensure(((size_t)B * N + 16) * 16));
  if (dim == 3) HH_TRY(E.tmp3.ensure(((size_t)B * 2 * N + 16) * 16));
  HH_TRY(E.rc.ensure((size_t)B * Nc * 16));
  HH_TRY(E.ec.ensure((size_t)B * Nc * 16));
  HH_TRY(E.stc.ensure((size_t)Bf * Nc * S * 16));
  if (P) HH_TRY(E.F.ensure((size_t)Bf * nd_front_entries(P) * 16));
  if (P) HH_TRY(E.cbuf.ensure((size_t)Bf * nd_cbuf_entries(P) * 16));
  HH_TRY(E.slabp.ensure((size_t)B * sizeof(int2)));
  if (sp.comm) HH_TRY(E.hstage.ensure((size_t)4 * FL.G * FL.plane * 16));
  if (P) {
    HH_TRY(E.work.ensure((size_t)B * nd_work_entries(P) * 16));
    HH_TRY(nd_flow_reset(P, B, E.work.as<cplx>(), E.s));
  }
  if (sp.fd) {   // eigenbases (one per factor copy) + two transform buffers per entry
    HH_TRY(E.fdb.ensure((size_t)Bf * fd_basis_entries(n / 2) * 16));
    HH_TRY(E.fdm.ensure((size_t)B * 16 + 64));   // bidx[B] | slot flags | slot k (section 7e)
    HH_TRY(E.work.ensure((size_t)B * fd_work_entries(dim, n / 2) * 16));
  }
  HH_TRY(E.kcf.ensure((size_t)B * 16));
  HH_TRY(E.kcc.ensure((size_t)B * 16));
  HH_TRY(E.cpart.ensure((size_t)B * nblk * (m + 2) * 16));
  HH_TRY(E.dpart.ensure((size_t)B * nblk * 8));
  HH_TRY(E.hist.ensure((size_t)B * HIST_LEN * 8));
  HH_TRY(E.ksmall.ensure(ksmall_bytes(B, m, nblk)));
  if (E.h_cap < B) {
    if (E.h_status) cudaFreeHost(E.h_status);
    E.h_status = nullptr;
    HH_CUDA_TRY(cudaMallocHost(&E.h_status, std::max(B, 4) * sizeof(int)));
    E.h_cap = std::max(B, 4);
  }
  return HH_OK;
}

// HH_PROFILE_SETUP=1: synchronise and print the setup phases (diagnostics only)
static const bool g_prof_setup = getenv("HH_PROFILE_SETUP") != nullptr;
static void prof_mark(Engine& E, const char* what, double& t) {
  if (!g_prof_setup) return;
  cudaStreamSynchronize(E.s);
  const double t1 = now_s();
  fprintf(stderr, "[hh setup] n=%d B=%d %-10s %9.3f ms\n", E.spec.n, E.B, what, 1e3 * (t1 - t));
  t = t1;
}

// distributed coarse solve: the rank views of this process' entries (slab k =
// rank slab_first + k) of the slab-aligned tree over the coarse planes of the
// fine slab bounds, with their factor / packed-S / work pools; the pivot-column
// + workspace scratch is shared by the views (they run one after another)
hh_status dist_setup(Engine& E, const BatchSpec& sp) {
  const int m = sp.n / 2 + 1, P = sp.slabs_total;
  const std::vector<int> z = slab_bounds(sp.n, P);
  std::vector<int> Zc(P + 1);
  for (int k = 0; k < P; ++k) Zc[k] = z[k] / 2;
  Zc[P] = m;
  E.dviews.assign(sp.B, NDDistView());
  E.dF.resize(sp.B);
  E.dS.resize(sp.B);
  E.dW.resize(sp.B);
  int64_t scratch = 1, stage = 1;
  for (int b = 0; b < sp.B; ++b) {
    NDPlan* p = nullptr;
    HH_TRY(get_dist_plan(sp.dim, m, Zc, sp.slab_first + b, &p));
    scratch = std::max(scratch, nd_dist_scratch_entries(p));
    stage = std::max(stage, nd_dist_stage_entries(p));
    HH_TRY(E.dF[b].ensure((size_t)std::max<int64_t>(1, nd_front_entries(p)) * 16));
    HH_TRY(E.dS[b].ensure((size_t)nd_dist_s_entries(p) * 16));
    HH_TRY(E.dW[b].ensure((size_t)nd_work_entries(p) * 16));
    E.dviews[b].plan = p;
    if (getenv("HH_DEBUG"))
      fprintf(stderr, "[hh dist] rank %d/%d: factor %.3f GB, packed S %.3f GB, work %.3f GB, scratch %.3f GB\n",
              sp.slab_first + b, P, 16e-9 * nd_front_entries(p), 16e-9 * nd_dist_s_entries(p),
              16e-9 * nd_work_entries(p), 16e-9 * nd_dist_scratch_entries(p));
  }
  HH_TRY(E.dscratch.ensure((size_t)scratch * 16));
  HH_TRY(E.dstage.ensure((size_t)stage * 16));
  HH_TRY(E.dflag.ensure((size_t)sp.B * sizeof(int)));
  for (int b = 0; b < sp.B; ++b) {
    NDDistView& v = E.dviews[b];
    v.F = E.dF[b].as<cplx>();
    v.S = E.dS[b].as<cplx>();
    v.work = E.dW[b].as<cplx>();
    v.scratch = E.dscratch.as<cplx>();
    v.flag = E.dflag.as<int>() + b;
  }
  E.plan = E.dviews[0].plan;
  return HH_OK;
}

hh_status batch_setup(Engine& E, const BatchSpec& sp) {
  const double t0 = now_s();
  double tp = t0;
  HH_CUDA_TRY(cudaSetDevice(E.device));
  E.drop_graphs();
  E.spec = sp;
  const int B = sp.B, dim = sp.dim, n = sp.n, m = sp.m;
  E.B = B; E.m = m;
  E.N = ipow(n + 1, dim);
  E.Nc = ipow(n / 2 + 1, dim);
  E.FL = fine_layout(sp);
  E.Bf = sp.slabmode ? 1 : B;
  const int64_t Nc = E.Nc;
  const int64_t NS = E.FL.stride;   // entry stride of fine vectors (ghosted)
  if (sp.slabmode)
    for (const int2& z : E.FL.slabs)
      if (z.y - z.x < E.FL.G || z.x % 2) {
        hh_set_error("slab [%d, %d) has fewer than G = %d planes (n = %d, %d slabs)", z.x, z.y, E.FL.G,
                     n, sp.slabs_total);
        return HH_E_CONFIG;
      }
  E.plan = nullptr;
  if (sp.dist) HH_TRY(dist_setup(E, sp));
  else if (!sp.fd) HH_TRY(get_plan(dim, n / 2 + 1, &E.plan));
  const NDPlan* P = E.plan;
  // pools
  HH_TRY(reserve_pools(E, sp));
  HH_CUDA_TRY(cudaMemcpyAsync(E.slabp.p, E.FL.slabs.data(), B * sizeof(int2), cudaMemcpyHostToDevice, E.s));
  // transport context (slab mode)
  E.X = SlabCtx();
  E.X.B = B;
  E.X.slab = E.slabp.as<int2>();
  E.X.h_slab = E.FL.slabs;
  E.X.all_z = E.FL.all_z;
  E.X.G = E.FL.G;
  E.X.maxloc = E.FL.maxloc;
  E.X.nc1 = n / 2 + 1;
  E.X.plane = E.FL.plane;
  E.X.cplane = ipow(n / 2 + 1, dim - 1);
  E.X.comm = sp.comm;
  if (sp.comm) {
    E.X.hsend = E.hstage.as<cplx>();
    E.X.hrecv = E.hstage.as<cplx>() + 2 * E.FL.G * E.FL.plane;
  }
  // per-level coefficients
  for (int lev = 0; lev < 2; ++lev) {
    Level& L = lev == 0 ? E.LF : E.LC;
    L.dim = dim;
    L.n = lev == 0 ? n : n / 2;
    L.h = 1.0 / L.n;
    L.nodes = ipow(L.n + 1, dim);
    L.elems = ipow(L.n, dim);
    L.plane = ipow(L.n + 1, dim - 1);
    L.het = sp.kf != nullptr;
    L.tmp = lev == 0 && dim == 3 ? E.tmp3.as<cplx>() + E.FL.pad : nullptr;
    L.coef = nullptr;
    L.coef_bs = 0;   // heterogeneous coefficients: one problem, shared by its entries
    L.kc = nullptr;
    if (lev == 0) {
      L.slab = E.slabp.as<int2>();
      L.G = E.FL.G;
      L.maxloc = E.FL.maxloc;
      L.stride = NS;
    } else {
      L.slab = nullptr;
      L.G = 0;
      L.maxloc = L.n + 1;
      L.stride = L.nodes;
    }
    if (L.het) {
      if (B != 1 && !sp.slabmode) { hh_set_error("heterogeneous batches must have B = 1"); return HH_E_CONFIG; }
      Pool& cp = lev == 0 ? E.coef_f : E.coef_c;
      HH_TRY(cp.ensure(L.elems * 16));
      HH_TRY(E.kstage.ensure(L.elems * 8));
      const double* kh = lev == 0 ? sp.kf : sp.kcoarse;
      for (int64_t e = 0; e < L.elems; ++e) {
        const double k = kh[e];
        if (!(k >= 0) || !std::isfinite(k)) {
          hh_set_error("k_elem[%lld] = %g invalid", (long long)e, k);
          return HH_E_CONFIG;
        }
      }
      // upload k_e only; (k_e, eps_e = beta k_e^sigma) is formed on the device (reading C2)
      HH_CUDA_TRY(cudaMemcpyAsync(E.kstage.p, kh, L.elems * 8, cudaMemcpyHostToDevice, E.s));
      {
        const unsigned g = (unsigned)std::min<int64_t>(148 * 8, (L.elems + 255) / 256);
        k_coef<<<g, 256, 0, E.s>>>(E.kstage.as<double>(), L.elems, sp.beta[0], sp.sigma[0], sp.shift_map,
                                   std::log2((double)n), cp.as<double2>());
        HH_CUDA_TRY(cudaGetLastError());
      }
      HH_CUDA_TRY(cudaStreamSynchronize(E.s));   // kh is caller memory (pageable)
      L.coef = cp.as<double2>();
    } else {
      Pool& kp = lev == 0 ? E.kcf : E.kcc;
      std::vector<double2> c(B);
      for (int b = 0; b < B; ++b)
        c[b] = make_double2(sp.k[b], shift_of(sp.k[b], sp.beta[b], sp.sigma[b], sp.shift_map, std::log2((double)n)));
      HH_CUDA_TRY(cudaMemcpyAsync(kp.p, c.data(), B * 16, cudaMemcpyHostToDevice, E.s));
      HH_CUDA_TRY(cudaStreamSynchronize(E.s));
      L.kc = kp.as<double2>();
    }
  }
  // Krylov small arrays: vscale, cs (double) ; sn, g, y (cplx) ; H ; state ; jdev ; flags ; counters
  const int ldv = m + 1, ldh = m + 1;
  // Krylov CTAs per sample: enough for ONE sample to fill the GPU (the tail of a
  // batch is a single slow sample); independent of B, so batched == single results
  E.nblk = krylov_blocks((int64_t)E.FL.maxloc * E.FL.plane);
  E.hist_len = HIST_LEN;
  size_t off = 0;
  auto carve = [&](size_t bytes) { size_t o = off; off += (bytes + 255) / 256 * 256; return o; };
  // (ksmall_bytes() below must mirror this layout)
  const int ldg = (E.nblk + 31) / 32;   // k_mdot group counters (MD_GROUP = 32)
  const size_t o_gc = carve((size_t)B * ldg * 4);
  const size_t o_vs = carve(B * ldv * 8), o_cs = carve(B * ldv * 8), o_sn = carve(B * ldv * 16),
               o_g = carve(B * ldv * 16), o_y = carve(B * ldv * 16), o_H = carve((size_t)B * m * ldh * 16),
               o_bn = carve(B * 8), o_res = carve(B * 8), o_rt = carve(B * 8), o_st = carve(B * 4),
               o_its = carve(B * 4), o_je = carve(B * 4), o_j = carve(16), o_fl = carve(B * 4),
               o_cnt = carve(B * 4), o_red = carve(B * (ldv + 1) * 16), o_red2 = carve(B * 8),
               o_wn = carve(B * 8), o_reo = carve(B * 4), o_jl = carve(B * 4), o_ff = carve(16);
  HH_TRY(E.ksmall.ensure(off));
  HH_TRY(E.cpart.ensure((size_t)B * E.nblk * (m + 2) * 16));
  HH_TRY(E.dpart.ensure((size_t)B * E.nblk * 8));
  HH_TRY(E.hist.ensure((size_t)B * E.hist_len * 8));
  char* base = E.ksmall.as<char>();
  KArgs& A = E.ka;
  A = KArgs();
  A.Nst = NS; A.n = n; A.G = E.FL.G; A.plane = E.FL.plane; A.slab = E.slabp.as<int2>();
  A.V = E.V.as<cplx>() + E.FL.pad; A.Vbs = (int64_t)(m + 1) * NS;
  A.Z = E.Z.as<cplx>() + E.FL.pad; A.Zbs = (int64_t)m * NS;
  A.w = E.w.as<cplx>() + E.FL.pad;
  A.slabred = sp.slabmode ? 1 : 0;
  A.red = (cplx*)(base + o_red); A.ldr = ldv + 1;
  A.red2 = (double*)(base + o_red2);
  A.H = (cplx*)(base + o_H); A.HB = (int64_t)m * ldh; A.ldh = ldh;
  A.vscale = (double*)(base + o_vs); A.cs = (double*)(base + o_cs);
  A.sn = (cplx*)(base + o_sn); A.g = (cplx*)(base + o_g); A.y = (cplx*)(base + o_y); A.ldv = ldv;
  A.cpart = E.cpart.as<cplx>(); A.ldp = m + 2;
  A.dpart = E.dpart.as<double>();
  A.counter = (unsigned*)(base + o_cnt);
  A.gcounter = (unsigned*)(base + o_gc); A.ldg = ldg;
  E.jdev = (int*)(base + o_j);
  A.jdev = E.jdev;
  A.nblk = E.nblk;
  A.hist_len = E.hist_len;
  A.ks.bnorm = (double*)(base + o_bn); A.ks.res = (double*)(base + o_res);
  A.ks.rtrue = (double*)(base + o_rt); A.ks.status = (int*)(base + o_st);
  A.ks.its = (int*)(base + o_its); A.ks.jend = (int*)(base + o_je); A.ks.hist = E.hist.as<double>();
  A.ks.jlast = (int*)(base + o_jl);
  A.wnorm2 = (double*)(base + o_wn); A.reo = (int*)(base + o_reo);
  E.nd_flag = (int*)(base + o_fl);
  E.flow_fail = (int*)(base + o_ff);
  HH_CUDA_TRY(cudaMemsetAsync(E.ksmall.p, 0, off, E.s));
  prof_mark(E, "pools+coef", tp);
  // precomputed D^{-1} of the heterogeneous fine operator (read by the smoothers)
  E.LF.dinv = nullptr;
  if (E.LF.het) {
    HH_TRY(E.dinvp.ensure(((size_t)B * NS + 16) * 16));
    E.LF.dinv = E.dinvp.as<cplx>() + E.FL.pad;
    HH_TRY(fine_dinv(E.LF, B, E.s));
  }
  // coarse operator + factorisation (slab mode: one copy, shared by the slabs)
  HH_TRY(coarse_stencil(E.LC, E.Bf, E.stc.as<cplx>(), E.s));
  int nflag = E.Bf;
  const int* flags = E.nd_flag;
  if (sp.dist) {   // each rank view factors its own fronts; S blocks move to the parents' owners
    HH_TRY(nd_dist_factor(E.dviews, E.stc.as<cplx>(), sp.comm, E.s));
    nflag = B;
    flags = E.dflag.as<int>();
    prof_mark(E, "factor", tp);
  } else if (sp.fd) {   // eigenpairs of the 1D pencil per factor copy (fd.cu)
    // one eigenbasis per distinct k (it does not depend on eps): slots
    std::vector<double> ks;
    std::vector<int> meta(B, 0);
    for (int b = 0; b < B; ++b) {
      const double kb = sp.k[sp.slabmode ? 0 : b];
      int sl = 0;
      while (sl < (int)ks.size() && ks[sl] != kb) ++sl;
      if (sl == (int)ks.size()) ks.push_back(kb);
      meta[b] = sl;
    }
    const int ns = (int)ks.size();
    const size_t o_fl = (size_t)B, o_k = ((o_fl + ns) * sizeof(int) + 7) / 8 * 8;
    std::vector<char> hb(o_k + ns * sizeof(double), 0);
    memcpy(hb.data(), meta.data(), B * sizeof(int));
    memcpy(hb.data() + o_k, ks.data(), ns * sizeof(double));
    HH_CUDA_TRY(cudaMemcpyAsync(E.fdm.p, hb.data(), hb.size(), cudaMemcpyHostToDevice, E.s));
    char* fm = E.fdm.as<char>();
    E.fd_bidx = (const int*)fm;
    HH_TRY(fd_setup(dim, n / 2, E.Bf, ns, (const double*)(fm + o_k), E.fd_bidx, (int*)fm + o_fl, E.LC.kc,
                    E.fdb.as<cplx>(), E.nd_flag, E.s));
    const char* ff = getenv("HH_FD_FAIL");   // fault injection (tests): validation failure
    if (ff && atoi(ff)) HH_TRY(fd_flag_all(E.nd_flag, E.Bf, 1, E.s));
    prof_mark(E, "fd basis", tp);
  } else {
    HH_TRY(nd_factor(P, E.Bf, E.stc.as<cplx>(), E.F.as<cplx>(), E.cbuf.as<cplx>(), E.nd_flag, E.s));
    prof_mark(E, "factor", tp);
    HH_CUDA_TRY(cudaMemsetAsync(E.rc.p, 0, (size_t)B * Nc * 16, E.s));
    HH_TRY(nd_autotune(P, B, E.F.as<cplx>(), E.work.as<cplx>(), varg(E.rc.as<cplx>(), Nc),
                       varg(E.ec.as<cplx>(), Nc), E.s, sp.slabmode, E.conc));
    prof_mark(E, "autotune", tp);
  }
  if (E.h_cap < nflag) {
    if (E.h_status) cudaFreeHost(E.h_status);
    E.h_status = nullptr;
    HH_CUDA_TRY(cudaMallocHost(&E.h_status, nflag * sizeof(int)));
    E.h_cap = nflag;
  }
  HH_CUDA_TRY(cudaMemcpyAsync(E.h_status, flags, nflag * sizeof(int), cudaMemcpyDeviceToHost, E.s));
  HH_CUDA_TRY(cudaStreamSynchronize(E.s));
  for (int b = 0; b < nflag; ++b)
    if (E.h_status[b]) {
      if (sp.fd && E.h_status[b] == 1) {   // secular roots failed validation
        if (sp.coarse == HH_COARSE_AUTO) {   // -> the nested-dissection factor
          BatchSpec nd = sp;
          nd.fd = false;
          return batch_setup(E, nd);
        }
        hh_set_error("HH_COARSE_FD: eigen-decomposition of the coarse pencil failed validation "
                     "(sample %d: k=%g, h_c=%g; use HH_COARSE_ND)", b, sp.k.empty() ? 0.0 : sp.k[b], E.LC.h);
        return HH_E_SINGULAR;
      }
      hh_set_error("%s (sample %d: k=%g, beta=%g, sigma=%g, h=%g)",
                   sp.fd ? "singular coarse operator (zero transformed diagonal entry)"
                         : "zero pivot in the coarse factorisation",
                   b, sp.k.empty() ? 0.0 : sp.k[b], sp.beta[b], sp.sigma[b], E.LC.h);
      return HH_E_SINGULAR;
    }
  E.setup_s = now_s() - t0;
  return HH_OK;
}

// vector views of the engine pools
VArg vV(Engine& E, int jo) {
  return varg(E.V.as<cplx>() + E.FL.pad, (int64_t)(E.m + 1) * E.FL.stride, E.FL.stride, E.jdev, jo);
}
VArg vZ(Engine& E) { return varg(E.Z.as<cplx>() + E.FL.pad, (int64_t)E.m * E.FL.stride, E.FL.stride, E.jdev, 0); }
VArg vfine(Engine& E, Pool& p) { return varg(p.as<cplx>() + E.FL.pad, E.FL.stride); }
bool slab_mode(const Engine& E) { return E.spec.slabmode; }
// coarse solve on all entries (shared factor in slab mode)
hh_status coarse_solve_all(Engine& E, const int* st, VArg rhs, VArg x) {
  if (E.spec.dist) {   // distributed: each entry solves its own fronts, then the owned planes go round
    HH_TRY(nd_dist_solve(E.dviews, st, rhs, x, E.spec.comm, E.dstage.as<cplx>(), E.s));
    return slab_coarse_allgather(E.X, x, E.s);
  }
  if (E.spec.fd)   // slab mode: one basis shared by the entries (the replicated coarse solve)
    return fd_solve(E.spec.dim, E.spec.n / 2, E.B, st, E.fdb.as<cplx>(), E.fd_bidx, E.LC.kc, E.work.as<cplx>(),
                    rhs, x, E.s);
  return nd_solve(E.plan, E.B, st, E.F.as<cplx>(), E.work.as<cplx>(), rhs, x, E.s, slab_mode(E), E.conc,
                  E.flow_fail);
}
// after a dataflow coarse-solve failure: zero the counters, never use the schedule again
hh_status flow_recover(Engine& E) {
  HH_TRY(nd_flow_reset(E.plan, E.B, E.work.as<cplx>(), E.s));
  HH_CUDA_TRY(cudaMemsetAsync(E.flow_fail, 0, sizeof(int), E.s));
  HH_CUDA_TRY(cudaStreamSynchronize(E.s));
  nd_flow_disable(E.plan);
  E.drop_graphs();
  return HH_OK;
}
// status-less calls (hh_vcycle, hh_coarse_solve): when the dataflow schedule ran,
// read its failure flag before returning (these calls then block)
hh_status flow_check(Engine& E, bool used) {
  if (!used) return HH_OK;
  int f = 0;
  HH_CUDA_TRY(cudaMemcpyAsync(&f, E.flow_fail, sizeof(int), cudaMemcpyDeviceToHost, E.s));
  HH_CUDA_TRY(cudaStreamSynchronize(E.s));
  if (!f) return HH_OK;
  HH_TRY(flow_recover(E));
  hh_set_error("coarse solve: a dataflow dependency wait timed out (schedule disabled; retry the call)");
  return HH_E_CUDA;
}
// Arnoldi reductions of the slab mode: partials -> (NCCL allreduce) -> finish on every entry
hh_status krylov_mdot_all(Engine& E, int pass) {
  HH_TRY(krylov_mdot(E.ka, E.B, E.s, pass));
  if (!slab_mode(E)) return HH_OK;
  HH_TRY(slab_allreduce(E.X, (double*)E.ka.red, (size_t)2 * E.ka.ldr * E.B, E.s));
  return krylov_mdot_fin(E.ka, E.B, E.s, pass);
}
hh_status krylov_update_all(Engine& E, int pass) {
  HH_TRY(krylov_update(E.ka, E.B, E.s, pass));
  if (!slab_mode(E)) return HH_OK;
  HH_TRY(slab_allreduce(E.X, E.ka.red2, (size_t)E.B, E.s));
  return krylov_update_fin(E.ka, E.B, E.s, pass);
}
hh_status krylov_norm_all(Engine& E, VArg r, int mode) {
  HH_TRY(krylov_norm(E.ka, E.B, r, mode, E.s));
  if (!slab_mode(E)) return HH_OK;
  HH_TRY(slab_allreduce(E.X, E.ka.red2, (size_t)E.B, E.s));
  return krylov_norm_fin(E.ka, E.B, mode, E.s);
}
hh_status halo(Engine& E, VArg v) { return slab_mode(E) ? slab_halo(E.X, v, E.s) : HH_OK; }
VArg vflat(Pool& p, int64_t bs) { return varg(p.as<cplx>(), bs); }

// one FGMRES iteration for the whole batch (graph-capturable)
hh_status enqueue_iteration(Engine& E, bool timing) {
  const int* st = E.ka.ks.status;
  cudaStream_t s = E.s;
  const SArg fs = sarg(E.ka.vscale, E.ka.ldv, E.jdev, 0);
  if (timing) HH_CUDA_TRY(cudaEventRecordWithFlags(E.ev[0], s, cudaEventRecordExternal));
  HH_TRY(halo(E, vV(E, 0)));                     // ghost planes of f = v_j (slab mode)
  HH_TRY(fine_pre(E.LF, E.B, st, E.spec.nu_pre, E.spec.omega, vV(E, 0), fs, vfine(E, E.u),
                  vflat(E.rc, E.Nc), s));
  if (slab_mode(E)) HH_TRY(slab_coarse_allgather(E.X, vflat(E.rc, E.Nc), s));
  if (timing) HH_CUDA_TRY(cudaEventRecordWithFlags(E.ev[1], s, cudaEventRecordExternal));
  if (timing) HH_CUDA_TRY(cudaEventRecordWithFlags(E.ev[2], s, cudaEventRecordExternal));
  HH_TRY(coarse_solve_all(E, st, vflat(E.rc, E.Nc), vflat(E.ec, E.Nc)));
  if (timing) HH_CUDA_TRY(cudaEventRecordWithFlags(E.ev[3], s, cudaEventRecordExternal));
  if (timing) HH_CUDA_TRY(cudaEventRecordWithFlags(E.ev[4], s, cudaEventRecordExternal));
  HH_TRY(halo(E, vfine(E, E.u)));                // ghost planes of the pre-smoothed u
  HH_TRY(fine_post(E.LF, E.B, st, E.spec.nu_post, E.spec.omega, vV(E, 0), fs, vfine(E, E.u),
                   vflat(E.ec, E.Nc), vZ(E), vfine(E, E.w), s));
  if (timing) HH_CUDA_TRY(cudaEventRecordWithFlags(E.ev[5], s, cudaEventRecordExternal));
  if (timing) HH_CUDA_TRY(cudaEventRecordWithFlags(E.ev[6], s, cudaEventRecordExternal));
  HH_TRY(krylov_mdot_all(E, 1));
  HH_TRY(krylov_update_all(E, 1));
  if (E.ka.reorth) {   // second CGS pass (samples with reo[b] = 1 only)
    HH_TRY(krylov_mdot_all(E, 2));
    HH_TRY(krylov_update_all(E, 2));
  }
  if (timing) HH_CUDA_TRY(cudaEventRecordWithFlags(E.ev[7], s, cudaEventRecordExternal));
  HH_TRY(krylov_advance(E.jdev, -1, s));
  return HH_OK;
}

int64_t launches_per_iteration(const Engine& E) {
  const int fine = E.spec.dim == 2 ? 2 : (E.spec.nu_pre + 2 + 1 + E.spec.nu_post + 1);
  int slab = 0;
  if (slab_mode(E)) {
    const bool multi = E.X.comm && E.X.comm->nranks > 1;
    slab = 2 * ((E.B > 1 ? 1 : 0) + (multi ? 2 : 0)) + (E.B > 1 ? 1 : 0) + 2;
  }
  const int kry = E.ka.reorth ? 4 + (slab_mode(E) ? 2 * (2 + (E.X.comm && E.X.comm->nranks > 1 ? 2 : 0)) : 0) : 0;
  const int nd = E.spec.fd ? fd_solve_launches(E.spec.dim)
                           : (E.spec.dist ? nd_dist_launches(E.dviews) + 2 : nd_solve_launches(E.plan, E.B, E.conc));
  return fine + nd + 3 + slab + kry;
}

// two captured variants of one iteration: plain, and with phase events (sampled timing)
hh_status run_iteration(Engine& E, bool timed) {
  cudaGraphExec_t& ge = timed ? E.gexec_t : E.gexec;
  if (!ge) {
    cudaGraph_t g;
    HH_CUDA_TRY(cudaStreamBeginCapture(E.s, cudaStreamCaptureModeThreadLocal));
    hh_status st = enqueue_iteration(E, timed);
    cudaError_t ce = cudaStreamEndCapture(E.s, &g);
    if (st != HH_OK) return st;
    HH_CUDA_TRY(ce);
    HH_CUDA_TRY(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
  }
  HH_CUDA_TRY(cudaGraphLaunch(ge, E.s));
  E.launches += launches_per_iteration(E);
  return HH_OK;
}

void harvest_timers(Engine& E) {
  float ms = 0;
  for (int k = 0; k < T_NT; ++k)
    if (cudaEventElapsedTime(&ms, E.ev[2 * k], E.ev[2 * k + 1]) == cudaSuccess) E.acc_ms[k] += ms;
    else cudaGetLastError();
}

// HBM bytes of one iteration per running sample, two counts:
//  out   = compulsory bytes of OUR fused kernels (each reads its inputs and writes
//          its outputs once: pre/post are single passes over the fine grid);
//  model = SURVEY.md 8(d)'s per-step model, in which every Jacobi step, the
//          residual + restriction, the prolongation + correction and the A_0
//          apply are separate passes (vectors 16 B/node, coefficients c = 16 B
//          (A_eps) / c0 = 8 B (A_0) per element when heterogeneous, coarse share
//          16/2^d B per fine node).  The model counts are the "algorithmic" bytes
//          of the roofline; the fused kernels move fewer, so their model-byte rate
//          can exceed what HBM alone would allow.
void phase_bytes(const Engine& E, int j, double* out, double* model) {
  const double N = (double)E.N, Nc = (double)E.Nc;
  const double ce = E.LF.het ? 16.0 * (double)E.LF.elems : 0.0;   // A_eps coefficients
  const double c0 = E.LF.het ? 8.0 * (double)E.LF.elems : 0.0;    // A_0 coefficients
  const double cshare = 16.0 * Nc;
  const int nu1 = E.spec.nu_pre, nu2 = E.spec.nu_post;
  out[T_PRE] = 32.0 * N + 16.0 * Nc + ce;                  // f, u, r_c (+ coef)
  out[T_POST] = 64.0 * N + 16.0 * Nc + ce;                 // f, u, e_c, z, w (+ coef)
  double nb = 0;
  if (E.spec.fd)
    nb = (double)fd_solve_bytes(E.spec.dim, E.spec.n / 2) - 32.0 * Nc;
  else if (E.spec.dist)   // every view streams its own fronts (per problem: the sum over the ranks)
    for (const NDDistView& v : E.dviews) nb += (double)nd_stream_bytes(v.plan);
  else
    nb = (double)nd_stream_bytes(E.plan);
  out[T_COARSE] = nb + 32.0 * Nc;
  out[T_KRYLOV] = (2.0 * (j + 1) + 3.0) * 16.0 * N;        // mdot + update
  if (E.ka.reorth == 2) out[T_KRYLOV] *= 2.0;              // second pass every step
  // Jacobi from zero 32 + c, Jacobi 48 + c, residual + restrict 32 + c + share
  model[T_PRE] = (32.0 * N + ce) + (nu1 - 1) * (48.0 * N + ce) + (32.0 * N + ce + cshare);
  // prolong + correct + Jacobi 48 + c + share, Jacobi 48 + c, apply A_0 32 + c0
  model[T_POST] = (48.0 * N + ce + cshare) + (nu2 - 1) * (48.0 * N + ce) + (32.0 * N + c0);
  model[T_COARSE] = out[T_COARSE];
  model[T_KRYLOV] = (32.0 * (j + 1) + 48.0) * N;           // CGS 32j + 80 B/node (j counted from 1)
  if (E.ka.reorth == 2) model[T_KRYLOV] *= 2.0;
}
double coarse_flops(const Engine& E) {   // per running sample and coarse solve (FD GEMMs; 0 for ND)
  return E.spec.fd ? fd_solve_flops(E.spec.dim, E.spec.n / 2) : 0.0;
}
void account_bytes(Engine& E, int running, int j) {
  double pb[T_NT], mb[T_NT];
  phase_bytes(E, j, pb, mb);
  E.acc_flops += running * coarse_flops(E);
  for (int t = 0; t < T_NT; ++t) {
    E.acc_bytes[t] += running * pb[t];
    E.acc_model[t] += running * mb[t];
    E.acc_launch[t] += 1;
  }
}
void account_bytes_all(Engine& E, int running, int j) {
  double pb[T_NT], mb[T_NT];
  phase_bytes(E, j, pb, mb);
  E.acc_flops_all += running * coarse_flops(E);
  for (int t = 0; t < T_NT; ++t) {
    E.acc_bytes_all[t] += running * pb[t];
    E.acc_model_all[t] += running * mb[t];
  }
}

int count_running(Engine& E) {
  int r = 0;
  for (int b = 0; b < E.B; ++b) r += (E.h_status[b] == HHK_RUN);
  return r;
}

hh_status sync_status(Engine& E) {
  HH_CUDA_TRY(cudaMemcpyAsync(E.h_status, E.ka.ks.status, E.B * sizeof(int), cudaMemcpyDeviceToHost, E.s));
  HH_CUDA_TRY(cudaStreamSynchronize(E.s));
  return HH_OK;
}

// FGMRES(m) for every sample of the batch: b, x are [B] device vectors
// use_x0: xvec holds the initial guess x0 (r_0 = b - A_0 x0, PAPER.md:416 u^(0));
// otherwise x0 = 0 (BASELINE configs) and xvec is cleared.
hh_status batch_solve(Engine& E, VArg bvec, VArg xvec, const hh_fgmres_opts& o,
                      std::vector<SampleOut>& out, double* hist_host, bool use_x0 = false) {
  const int B = E.B;
  const int m = o.restart;
  if (m < 1 || m > E.m) { hh_set_error("restart %d not in 1..%d", m, E.m); return HH_E_CONFIG; }
  if (o.max_iters < 1 || o.max_iters >= E.hist_len || o.fixed_iters >= E.hist_len || o.fixed_iters < 0) {
    hh_set_error("max_iters/fixed_iters out of range");
    return HH_E_CONFIG;
  }
  if (o.reorth < 0 || o.reorth > 2) { hh_set_error("reorth must be 0, 1 or 2 (got %d)", o.reorth); return HH_E_CONFIG; }
  if (!(o.rtol >= 0)) { hh_set_error("rtol must be >= 0"); return HH_E_CONFIG; }
  cudaStream_t s = E.s;
  KArgs& A = E.ka;
  A.rtol = o.rtol;
  A.max_iters = o.max_iters;
  A.fixed_iters = o.fixed_iters;
  A.reorth = o.reorth;
  E.drop_graphs();   // KArgs (rtol, caps, reorth) are captured by value
  const int check = std::max(1, o.check_every);
  if (!use_x0) HH_TRY(vset(E.LF, xvec, VArg(), B, 0, 0, nullptr, s));
  HH_CUDA_TRY(cudaMemsetAsync(A.H, 0, (size_t)B * A.HB * sizeof(cplx), s));
  HH_CUDA_TRY(cudaMemsetAsync(A.reo, 0, (size_t)B * sizeof(int), s));
  HH_TRY(vset(E.LF, varg(A.V, A.Vbs), bvec, B, 1, 0, nullptr, s));       // V[0] = b
  HH_TRY(krylov_norm_all(E, bvec, 0));                                    // ||b||, status
  if (use_x0) {   // V[0] = r_0 = b - A_0 x0; the threshold stays relative to ||b|| (C14)
    HH_TRY(halo(E, xvec));
    HH_TRY(fine_apply(E.LF, B, A.ks.status, HH_OP_A0, xvec, varg(A.V, A.Vbs), bvec, s));
    HH_TRY(krylov_norm_all(E, varg(A.V, A.Vbs), 1));
    E.launches += 2;
  }
  HH_TRY(sync_status(E));
  std::vector<int> restarts(B, 0);
  int running = count_running(E);
  while (running > 0) {
    HH_TRY(krylov_advance(E.jdev, 0, s));
    for (int j = 0; j < m; ++j) {
      // sampled instrumentation: every timing_every-th iteration runs the graph
      // variant with phase events; its bytes use the exact running count
      const bool timed = E.timing && (E.iter_counter++ % E.timing_every == 0);
      if (timed) {
        HH_TRY(sync_status(E));
        running = count_running(E);
        if (!running) break;
      }
      if (E.gate && timed) {   // the GPU to itself: peers drained, no new peer launches
        E.gate->lock();
        for (cudaStream_t ps : E.peers) cudaStreamSynchronize(ps);
      } else if (E.gate) {
        E.gate->lock_shared();
      }
      const hh_status ist = run_iteration(E, timed);
      cudaError_t sst = cudaSuccess;
      if (timed && ist == HH_OK) sst = cudaStreamSynchronize(s);
      if (E.gate && timed) E.gate->unlock();
      else if (E.gate) E.gate->unlock_shared();
      HH_TRY(ist);
      HH_CUDA_TRY(sst);
      if (E.timing) account_bytes_all(E, running, j);
      if (timed) {
        harvest_timers(E);
        account_bytes(E, running, j);
      }
      if ((j + 1) % check == 0 || j == m - 1) {
        HH_TRY(sync_status(E));
        running = count_running(E);
        if (!running) break;
      }
    }
    HH_TRY(krylov_cycle_end(A, B, xvec, s));
    E.launches += 3;
    HH_TRY(sync_status(E));
    running = count_running(E);
    if (!running) break;
    // restart the still-running samples: V[0] = b - A_0 x
    for (int b = 0; b < B; ++b) if (E.h_status[b] == HHK_RUN) restarts[b]++;
    HH_CUDA_TRY(cudaMemsetAsync(A.H, 0, (size_t)B * A.HB * sizeof(cplx), s));
    HH_TRY(halo(E, xvec));
    HH_TRY(fine_apply(E.LF, B, A.ks.status, HH_OP_A0, xvec, varg(A.V, A.Vbs), bvec, s));
    HH_TRY(krylov_norm_all(E, varg(A.V, A.Vbs), 1));
    E.launches += 2;
    HH_TRY(sync_status(E));
    running = count_running(E);
  }
  // true residuals ||b - A_0 x||
  HH_TRY(halo(E, xvec));
  HH_TRY(fine_apply(E.LF, B, nullptr, HH_OP_A0, xvec, vfine(E, E.w), bvec, s));
  HH_TRY(krylov_norm_all(E, vfine(E, E.w), 2));
  E.launches += 2;
  std::vector<double> bn(B), res(B), rt(B);
  std::vector<int> its(B), stt(B);
  HH_CUDA_TRY(cudaMemcpyAsync(bn.data(), A.ks.bnorm, B * 8, cudaMemcpyDeviceToHost, s));
  HH_CUDA_TRY(cudaMemcpyAsync(res.data(), A.ks.res, B * 8, cudaMemcpyDeviceToHost, s));
  HH_CUDA_TRY(cudaMemcpyAsync(rt.data(), A.ks.rtrue, B * 8, cudaMemcpyDeviceToHost, s));
  HH_CUDA_TRY(cudaMemcpyAsync(its.data(), A.ks.its, B * 4, cudaMemcpyDeviceToHost, s));
  HH_CUDA_TRY(cudaMemcpyAsync(stt.data(), A.ks.status, B * 4, cudaMemcpyDeviceToHost, s));
  HH_CUDA_TRY(cudaStreamSynchronize(s));
  out.assign(B, SampleOut());
  bool ndfail = false;
  for (int b = 0; b < B; ++b) {
    SampleOut& r = out[b];
    r.iterations = its[b];
    r.restarts = restarts[b];
    r.rel_res_lsq = bn[b] > 0 ? res[b] / bn[b] : 0.0;
    r.rel_res_true = bn[b] > 0 ? rt[b] / bn[b] : 0.0;
    r.rho = its[b] > 0 ? std::pow(r.rel_res_true, 1.0 / its[b]) : NAN;
    r.converged = o.fixed_iters > 0 ? (r.rel_res_true <= o.rtol) : (stt[b] == HHK_CONVERGED);
    r.status = stt[b] == HHK_NAN ? HH_E_DIVERGED : (stt[b] == HHK_BREAKDOWN ? HH_E_BREAKDOWN : HH_OK);
    if (stt[b] == HHK_NDFAIL) {   // never a silent wrong result: the sample fails loudly
      r.status = HH_E_CUDA;
      r.converged = 0;
      ndfail = true;
    }
  }
  if (ndfail) {
    HH_TRY(flow_recover(E));
    hh_set_error("coarse solve: a dataflow dependency wait timed out (schedule disabled; rerun the sample)");
  }
  if (hist_host && (B == 1 || slab_mode(E))) {
    std::vector<double> h(its[0] + 1);
    HH_CUDA_TRY(cudaMemcpy(h.data(), A.ks.hist, (its[0] + 1) * 8, cudaMemcpyDeviceToHost));
    h[0] = 1.0;
    memcpy(hist_host, h.data(), (its[0] + 1) * 8);
  }
  return HH_OK;
}

// wait for the user stream before work on the engine stream, and vice versa
hh_status enter(Engine& E, cudaStream_t user) {
  cudaEvent_t e;
  HH_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  HH_CUDA_TRY(cudaEventRecord(e, user));
  HH_CUDA_TRY(cudaStreamWaitEvent(E.s, e, 0));
  cudaEventDestroy(e);
  return HH_OK;
}
hh_status leave(Engine& E, cudaStream_t user) {
  cudaEvent_t e;
  HH_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  HH_CUDA_TRY(cudaEventRecord(e, E.s));
  HH_CUDA_TRY(cudaStreamWaitEvent(user, e, 0));
  cudaEventDestroy(e);
  return HH_OK;
}
}  // namespace

// ================================================================== ABI
// Engines of destroyed handles are kept (per device, at most 4) and handed to
// the next setup: destroying an engine (graph execs, events, stream, pinned
// buffers, pools) costs 2-170 ms of driver work, re-creating it as much.
static std::mutex g_engine_mu;
static std::vector<Engine*> g_engine_cache;

static Engine* engine_take(int device) {
  std::lock_guard<std::mutex> lk(g_engine_mu);
  for (size_t i = 0; i < g_engine_cache.size(); ++i)
    if (g_engine_cache[i]->device == device) {
      Engine* e = g_engine_cache[i];
      g_engine_cache.erase(g_engine_cache.begin() + i);
      return e;
    }
  return nullptr;
}

static void engine_give(Engine* e) {
  const double t0 = now_s();
  e->drop_graphs();
  const double t1 = now_s();
  e->release_pools();   // memory goes back to the block cache (flushed on OOM)
  if (g_prof_setup)
    fprintf(stderr, "[hh destroy] drop_graphs %.3f ms release_pools %.3f ms\n", 1e3 * (t1 - t0),
            1e3 * (now_s() - t1));
  {
    std::lock_guard<std::mutex> lk(g_engine_mu);
    if (g_engine_cache.size() < 4) {
      e->timing = false;
      g_engine_cache.push_back(e);
      return;
    }
  }
  delete e;
}

struct hh_problem {
  hh_problem_desc d{};
  Engine* ep = nullptr;
  cudaStream_t user = nullptr;
  Comm* comm = nullptr;
  int64_t n_local = 0;      // user-vector length: owned nodes of this handle's slabs
  ~hh_problem() {
    comm_destroy(comm);
    if (ep) engine_give(ep);
  }
};

extern "C" hh_status hh_nccl_unique_id(void* id128) {
  if (!id128) { hh_set_error("NULL argument"); return HH_E_ARG; }
  return comm_unique_id(id128);
}

extern "C" hh_status hh_slab_bounds(int32_t n_cells, int32_t nslabs, int32_t* z) {
  if (!z || nslabs < 1 || n_cells < 4 || n_cells % 2) { hh_set_error("bad argument"); return HH_E_ARG; }
  const std::vector<int> b = slab_bounds(n_cells, nslabs);
  for (int i = 0; i <= nslabs; ++i) z[i] = b[i];
  return HH_OK;
}

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
  if (!(d->beta >= 0)) { hh_set_error("beta must be >= 0"); return HH_E_CONFIG; }
  if (d->shift_map < 0 || d->shift_map > 3) { hh_set_error("shift_map must be 0..3"); return HH_E_CONFIG; }
  if (d->coarse_solver < HH_COARSE_AUTO || d->coarse_solver > HH_COARSE_FD) {
    hh_set_error("coarse_solver must be HH_COARSE_AUTO, HH_COARSE_ND, HH_COARSE_ND_DIST or HH_COARSE_FD");
    return HH_E_CONFIG;
  }
  if (d->coarse_solver == HH_COARSE_FD && d->k_elem) {
    hh_set_error("HH_COARSE_FD needs a constant k (the coarse operator must be separable)");
    return HH_E_CONFIG;
  }
  const int nloc = std::max(1, d->nslabs_local);
  const bool use_nccl = d->nccl_id != nullptr;
  if (d->coarse_solver == HH_COARSE_ND_DIST && !(use_nccl ? d->nranks > 1 : nloc > 1)) {
    hh_set_error("HH_COARSE_ND_DIST needs a slab decomposition (nslabs_local > 1 or nranks > 1)");
    return HH_E_CONFIG;
  }
  if (use_nccl && (d->nranks < 1 || d->rank < 0 || d->rank >= d->nranks || nloc != 1)) {
    hh_set_error("NCCL slab mode needs 0 <= rank < nranks and nslabs_local <= 1");
    return HH_E_CONFIG;
  }
  hh_problem* p = new (std::nothrow) hh_problem();
  if (!p) return HH_E_OOM;
  p->d = *d;
  p->d.k_elem = p->d.k_elem_coarse = nullptr;
  p->d.nccl_id = nullptr;
  p->user = (cudaStream_t)d->stream;
  hh_status st = HH_OK;
  p->ep = engine_take(d->device);
  if (!p->ep) {
    p->ep = new (std::nothrow) Engine();
    if (!p->ep) { delete p; return HH_E_OOM; }
    st = engine_init(*p->ep, d->device);
    if (st != HH_OK) { delete p->ep; p->ep = nullptr; }
  }
  if (st == HH_OK && use_nccl) st = comm_create(d->nccl_id, d->rank, d->nranks, d->device, &p->comm);
  if (st == HH_OK) {
    BatchSpec sp;
    sp.dim = d->dim; sp.n = d->n_cells; sp.nu_pre = d->nu_pre; sp.nu_post = d->nu_post;
    sp.m = d->max_restart; sp.omega = d->omega;
    sp.slabmode = use_nccl || nloc > 1;
    sp.B = use_nccl ? 1 : nloc;
    sp.slabs_total = use_nccl ? d->nranks : nloc;
    sp.slab_first = use_nccl ? d->rank : 0;
    sp.comm = p->comm;
    sp.k.assign(sp.B, d->k_const); sp.beta.assign(sp.B, d->beta); sp.sigma.assign(sp.B, d->sigma);
    sp.kf = d->k_elem; sp.kcoarse = d->k_elem_coarse;
    sp.shift_map = d->shift_map;
    sp.dist = d->coarse_solver == HH_COARSE_ND_DIST;
    sp.coarse = d->coarse_solver;
    sp.fd = fd_wanted(d->coarse_solver, d->dim, d->n_cells / 2, d->k_elem != nullptr, sp.dist, d->k_const);
    st = enter(*p->ep, p->user);
    if (st == HH_OK) st = batch_setup(*p->ep, sp);
  }
  if (st != HH_OK) { delete p; return st; }
  for (const int2& z : p->ep->FL.slabs) p->n_local += (int64_t)(z.y - z.x) * p->ep->FL.plane;
  *out = p;
  return HH_OK;
}

extern "C" hh_status hh_layout(const hh_problem* p, int64_t* nf, int64_t* nc) {
  if (!p) { hh_set_error("NULL handle"); return HH_E_ARG; }
  if (nf) *nf = p->n_local;
  if (nc) *nc = p->ep->Nc;
  return HH_OK;
}

extern "C" hh_status hh_local_layout(const hh_problem* p, int64_t* n_local_nodes, int64_t* first_plane,
                                     int64_t* n_planes) {
  if (!p) { hh_set_error("NULL handle"); return HH_E_ARG; }
  const std::vector<int2>& z = p->ep->FL.slabs;
  if (n_local_nodes) *n_local_nodes = p->n_local;
  if (first_plane) *first_plane = z.front().x;
  if (n_planes) *n_planes = z.back().y - z.front().x;
  return HH_OK;
}

namespace {
// user vector (this handle's owned nodes) <-> ghosted engine vector of every entry
hh_status user_in(Engine& E, const void* u, Pool& dst) {
  return slab_user_copy(E.X, vfine(E, dst), const_cast<void*>(u), 0, E.s);
}
hh_status user_out(Engine& E, Pool& src, void* u) { return slab_user_copy(E.X, vfine(E, src), u, 1, E.s); }
}  // namespace

extern "C" hh_status hh_apply_op(hh_problem* p, int32_t op, const void* x, void* y) {
  if (!p || !x || !y) { hh_set_error("NULL argument"); return HH_E_ARG; }
  if (x == y) { hh_set_error("apply_op: x and y must be distinct"); return HH_E_ARG; }
  Engine& E = *p->ep;
  HH_TRY(enter(E, p->user));
  if (op == HH_OP_A0 || op == HH_OP_AEPS) {
    HH_TRY(user_in(E, x, E.xv));
    HH_TRY(halo(E, vfine(E, E.xv)));
    HH_TRY(fine_apply(E.LF, E.B, nullptr, op, vfine(E, E.xv), vfine(E, E.w), VArg(), E.s));
    HH_TRY(user_out(E, E.w, y));
  } else if (op == HH_OP_AEPS_COARSE) {
    HH_TRY(fine_apply(E.LC, 1, nullptr, HH_OP_AEPS, varg((cplx*)x, 0), varg((cplx*)y, 0), VArg(), E.s));
  } else {
    hh_set_error("apply_op: unknown op %d", op);
    return HH_E_ARG;
  }
  return leave(E, p->user);
}

extern "C" hh_status hh_vcycle(hh_problem* p, const void* f, void* z) {
  if (!p || !f || !z) { hh_set_error("NULL argument"); return HH_E_ARG; }
  Engine& E = *p->ep;
  HH_TRY(enter(E, p->user));
  HH_TRY(user_in(E, f, E.bv));
  HH_TRY(halo(E, vfine(E, E.bv)));
  HH_TRY(fine_pre(E.LF, E.B, nullptr, E.spec.nu_pre, E.spec.omega, vfine(E, E.bv), SArg(),
                  vfine(E, E.u), vflat(E.rc, E.Nc), E.s));
  if (slab_mode(E)) HH_TRY(slab_coarse_allgather(E.X, vflat(E.rc, E.Nc), E.s));
  HH_TRY(coarse_solve_all(E, nullptr, vflat(E.rc, E.Nc), vflat(E.ec, E.Nc)));
  HH_TRY(halo(E, vfine(E, E.u)));
  HH_TRY(fine_post(E.LF, E.B, nullptr, E.spec.nu_post, E.spec.omega, vfine(E, E.bv), SArg(),
                   vfine(E, E.u), vflat(E.ec, E.Nc), vfine(E, E.xv), VArg(), E.s));
  HH_TRY(user_out(E, E.xv, z));
  HH_TRY(flow_check(E, !E.spec.dist && !E.spec.fd && nd_solve_uses_flow(E.plan, E.B, E.conc)));
  return leave(E, p->user);
}

extern "C" hh_status hh_coarse_solve(hh_problem* p, const void* r, void* e) {
  if (!p || !r || !e) { hh_set_error("NULL argument"); return HH_E_ARG; }
  Engine& E = *p->ep;
  HH_TRY(enter(E, p->user));
  if (E.spec.dist) {   // r -> every entry, distributed solve + owned-plane allgather, entry 0 -> e
    for (int b = 0; b < E.B; ++b)
      HH_CUDA_TRY(cudaMemcpyAsync(E.rc.as<cplx>() + (int64_t)b * E.Nc, r, E.Nc * 16, cudaMemcpyDeviceToDevice, E.s));
    HH_TRY(coarse_solve_all(E, nullptr, vflat(E.rc, E.Nc), vflat(E.ec, E.Nc)));
    HH_CUDA_TRY(cudaMemcpyAsync(e, E.ec.p, E.Nc * 16, cudaMemcpyDeviceToDevice, E.s));
    return leave(E, p->user);
  }
  if (E.spec.fd) {
    HH_TRY(fd_solve(E.spec.dim, E.spec.n / 2, 1, nullptr, E.fdb.as<cplx>(), E.fd_bidx, E.LC.kc, E.work.as<cplx>(),
                    varg((cplx*)r, 0), varg((cplx*)e, 0), E.s));
    return leave(E, p->user);
  }
  HH_TRY(nd_solve(E.plan, 1, nullptr, E.F.as<cplx>(), E.work.as<cplx>(), varg((cplx*)r, 0),
                  varg((cplx*)e, 0), E.s, true, false, E.flow_fail));
  HH_TRY(flow_check(E, nd_solve_uses_flow(E.plan, 1, false)));
  return leave(E, p->user);
}

static void fill_report(const hh_problem* p, const SampleOut& o, double solve_s, hh_fgmres_report* r) {
  r->iterations = o.iterations;
  r->restarts = o.restarts;
  r->converged = o.converged;
  r->rel_res_lsq = o.rel_res_lsq;
  r->rel_res_true = o.rel_res_true;
  r->rho = o.rho;
  r->setup_s = p->ep->setup_s;
  r->solve_s = solve_s;
}

extern "C" hh_status hh_fgmres_solve(hh_problem* p, const void* bv, void* xv, const hh_fgmres_opts* o,
                                     hh_fgmres_report* rep, double* res_hist) {
  if (!p || !bv || !xv || !o || !rep) { hh_set_error("NULL argument"); return HH_E_ARG; }
  Engine& E = *p->ep;
  memset(rep, 0, sizeof(*rep));
  HH_TRY(enter(E, p->user));
  cudaEvent_t e0, e1;
  HH_CUDA_TRY(cudaEventCreate(&e0));
  HH_CUDA_TRY(cudaEventCreate(&e1));
  HH_CUDA_TRY(cudaEventRecord(e0, E.s));
  std::vector<SampleOut> out;
  hh_status st = user_in(E, bv, E.bv);
  if (st == HH_OK) st = user_in(E, xv, E.xv);   // x0
  if (st == HH_OK) st = batch_solve(E, vfine(E, E.bv), vfine(E, E.xv), *o, out, res_hist, true);
  if (st == HH_OK) st = user_out(E, E.xv, xv);
  HH_CUDA_TRY(cudaEventRecord(e1, E.s));
  HH_CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (st != HH_OK) return st;
  fill_report(p, out[0], ms * 1e-3, rep);
  HH_TRY(leave(E, p->user));
  if (out[0].status != HH_OK) {
    if (out[0].status != HH_E_CUDA)
      hh_set_error(out[0].status == HH_E_DIVERGED ? "FGMRES: NaN/Inf in the Arnoldi recurrence"
                                                  : "FGMRES: breakdown with residual above tolerance");
    return (hh_status)out[0].status;
  }
  return HH_OK;
}

extern "C" hh_status hh_fgmres_solve_host(hh_problem* p, const void* b_host, void* x_host,
                                          const hh_fgmres_opts* o, hh_fgmres_report* r) {
  if (!p || !b_host || !x_host) { hh_set_error("NULL argument"); return HH_E_ARG; }
  Engine& E = *p->ep;
  HH_TRY(enter(E, p->user));
  HH_TRY(E.ustage.ensure((size_t)p->n_local * 16));
  HH_CUDA_TRY(cudaMemcpyAsync(E.ustage.p, b_host, p->n_local * 16, cudaMemcpyHostToDevice, E.s));
  HH_TRY(user_in(E, E.ustage.p, E.bv));
  HH_CUDA_TRY(cudaMemcpyAsync(E.ustage.p, x_host, p->n_local * 16, cudaMemcpyHostToDevice, E.s));
  HH_TRY(user_in(E, E.ustage.p, E.xv));   // x0
  std::vector<SampleOut> out;
  const double t0 = now_s();
  HH_TRY(batch_solve(E, vfine(E, E.bv), vfine(E, E.xv), *o, out, nullptr, true));
  HH_TRY(user_out(E, E.xv, E.ustage.p));
  HH_CUDA_TRY(cudaMemcpyAsync(x_host, E.ustage.p, p->n_local * 16, cudaMemcpyDeviceToHost, E.s));
  HH_CUDA_TRY(cudaStreamSynchronize(E.s));
  fill_report(p, out[0], now_s() - t0, r);
  return (hh_status)out[0].status;
}

extern "C" hh_status hh_arnoldi_orthogonality(hh_problem* p, double* max_loss, int32_t* nvec) {
  if (!p || !max_loss) { hh_set_error("NULL argument"); return HH_E_ARG; }
  Engine& E = *p->ep;
  if (slab_mode(E)) { hh_set_error("arnoldi_orthogonality: not available for slab-decomposed handles"); return HH_E_STATE; }
  HH_CUDA_TRY(cudaSetDevice(E.device));
  HH_TRY(enter(E, p->user));
  int nv = 0;
  HH_TRY(krylov_orth_loss(E.ka, 0, max_loss, &nv, E.s));
  if (nvec) *nvec = nv;
  return leave(E, p->user);
}

extern "C" hh_status hh_destroy_problem(hh_problem* p) {
  if (!p) return HH_OK;
  cudaSetDevice(p->ep->device);
  cudaStreamSynchronize(p->ep->s);
  delete p;
  return HH_OK;
}

extern "C" hh_status hh_reset_timers(hh_problem* p, int32_t enable) {
  if (!p) return HH_E_ARG;
  p->ep->timing = enable != 0;
  for (int i = 0; i < T_NT; ++i)
    p->ep->acc_ms[i] = p->ep->acc_bytes[i] = p->ep->acc_launch[i] = p->ep->acc_bytes_all[i] =
        p->ep->acc_model[i] = p->ep->acc_model_all[i] = 0;
  p->ep->acc_flops = p->ep->acc_flops_all = 0;
  p->ep->launches = 0;
  return HH_OK;
}

extern "C" hh_status hh_read_timers(hh_problem* p, double* st12, int64_t* launches) {
  if (!p) return HH_E_ARG;
  if (st12)
    for (int i = 0; i < T_NT; ++i) {
      st12[i] = p->ep->acc_ms[i];
      st12[4 + i] = p->ep->acc_bytes[i];
      st12[8 + i] = p->ep->acc_launch[i];
      st12[12 + i] = p->ep->acc_bytes_all[i];
      st12[16 + i] = p->ep->acc_model[i];
      st12[20 + i] = p->ep->acc_model_all[i];
    }
  if (launches) *launches = p->ep->launches;
  return HH_OK;
}

// ================================================================== sweep
static std::mutex g_sweep_mu;
static bool g_sweep_timing = false;
static double g_sweep_st[6 * T_NT] = {0};
static double g_sweep_flops[2] = {0, 0};
static int64_t g_sweep_launches = 0;
// persistent sweep engines per device; a sweep holds its device's lock for the
// whole call, so concurrent hh_sweep calls never share an engine
static std::map<int, std::vector<std::unique_ptr<Engine>>> g_sweep_engines;
static std::map<int, std::unique_ptr<std::mutex>> g_sweep_dev_mu;
static std::mutex& sweep_device_mutex(int dev) {
  std::lock_guard<std::mutex> lk(g_sweep_mu);
  auto& m = g_sweep_dev_mu[dev];
  if (!m) m.reset(new std::mutex());
  return *m;
}

extern "C" hh_status hh_sweep_timers(int32_t reset_enable, double* st12, int64_t* launches) {
  std::lock_guard<std::mutex> lk(g_sweep_mu);
  if (st12)
    for (int i = 0; i < 6 * T_NT; ++i) st12[i] = g_sweep_st[i];
  if (launches) *launches = g_sweep_launches;
  if (reset_enable >= 0) {
    g_sweep_timing = reset_enable != 0;
    for (double& a : g_sweep_st) a = 0;
    g_sweep_flops[0] = g_sweep_flops[1] = 0;
    g_sweep_launches = 0;
  }
  return HH_OK;
}

// Batched solves of independent 2D constant-k samples (shared by hh_sweep and
// hh_shift_search): rhs == NULL -> unit point source at the centre node (C7),
// else rhs[i] = HOST complex128 right-hand side of sample i ((n+1)^2 nodes).
static hh_status sweep_run(const hh_problem_desc* common, const hh_fgmres_opts* o,
                           const hh_sample* smp, int32_t n, const void* const* rhs,
                           hh_sample_result* out) {
  if (!common || !o || (n && (!smp || !out))) { hh_set_error("NULL argument"); return HH_E_ARG; }
  if (n < 0) { hh_set_error("negative sample count"); return HH_E_ARG; }
  if (n == 0) return HH_OK;
  // the checks of hh_setup_problem (the Krylov kernels stage restart + 1 coefficients)
  if (o->restart < 1 || o->restart > KMAX_RESTART) {
    hh_set_error("restart must be in 1..%d (got %d)", KMAX_RESTART, o->restart);
    return HH_E_CONFIG;
  }
  if (common->max_restart > KMAX_RESTART) {
    hh_set_error("max_restart must be <= %d (got %d)", KMAX_RESTART, common->max_restart);
    return HH_E_CONFIG;
  }
  if (!(common->omega > 0 && common->omega <= 1)) { hh_set_error("omega must be in (0,1] (got %g)", common->omega); return HH_E_CONFIG; }
  if (common->nu_pre < 1 || common->nu_pre > 4 || common->nu_post < 1 || common->nu_post > 4) {
    hh_set_error("nu_pre/nu_post must be in 1..4");
    return HH_E_CONFIG;
  }
  if (common->shift_map < 0 || common->shift_map > 3) { hh_set_error("shift_map must be 0..3"); return HH_E_CONFIG; }
  if (common->coarse_solver != HH_COARSE_AUTO && common->coarse_solver != HH_COARSE_ND &&
      common->coarse_solver != HH_COARSE_FD) {
    hh_set_error("sweep: coarse_solver must be HH_COARSE_AUTO, HH_COARSE_ND or HH_COARSE_FD");
    return HH_E_CONFIG;
  }
  const int m = std::max(o->restart, common->max_restart > 0 ? common->max_restart : o->restart);
  for (int i = 0; i < n; ++i) {
    memset(&out[i], 0, sizeof(out[i]));
    out[i].id = smp[i].id;
    if (smp[i].n_cells < 4 || smp[i].n_cells % 2 || !(smp[i].k >= 0) || !(smp[i].beta >= 0)) {
      hh_set_error("sweep sample %lld: invalid (n=%d, k=%g, beta=%g)", (long long)smp[i].id,
                   smp[i].n_cells, smp[i].k, smp[i].beta);
      return HH_E_CONFIG;
    }
  }
  HH_CUDA_TRY(cudaSetDevice(common->device));
  std::lock_guard<std::mutex> dev_lock(sweep_device_mutex(common->device));
  // group by grid size; within a group, order by shift strength eps = beta k^sigma
  // (stronger shift -> more FGMRES iterations) so samples of
  // similar iteration counts share a lockstep batch; batches are bounded by a
  // per-engine memory budget and by a node budget (B * N <= HH_SWEEP_NODES)
  // that splits the large grids over several streams.
  std::map<int, std::vector<int>> groups;
  for (int i = 0; i < n; ++i) groups[smp[i].n_cells].push_back(i);
  const char* es = getenv("HH_SWEEP_STREAMS");
  // 6 engine streams: full sweep 1.51 s (3: 1.53, 8: 1.51; 2: 1.68-1.72, 1: 1.82-2.02 s),
  // and the 1/N shards of a multi-GPU sweep need the extra concurrency most (one
  // 8-way shard: 218 ms with 6 streams, 243 ms with 3; profiles/r02/shards)
  const int nstreams = std::max(1, es ? atoi(es) : 6);
  const char* eb = getenv("HH_SWEEP_MAX_BATCH");
  const int maxB = std::max(1, eb ? atoi(eb) : 256);
  const char* en = getenv("HH_SWEEP_NODES");
  const double node_budget = en ? atof(en) : 2.4e6;   // A/B: 1.2e6 -> 2.4e6 = +1.5% (profiles/r02/sweep_ab)
  // device memory size, queried once per device (cudaMemGetInfo takes driver locks
  // that can stall for tens of ms)
  static std::mutex tot_mu;
  static std::map<int, size_t> tot_cache;
  size_t totb = 0;
  {
    std::lock_guard<std::mutex> lk(tot_mu);
    auto it = tot_cache.find(common->device);
    if (it != tot_cache.end()) totb = it->second;
  }
  if (!totb) {
    size_t freeb = 0;
    HH_CUDA_TRY(cudaMemGetInfo(&freeb, &totb));
    std::lock_guard<std::mutex> lk(tot_mu);
    tot_cache[common->device] = totb;
  }
  const double budget = 0.60 * (double)totb / nstreams;   // engines persist: budget on total HBM
  std::vector<std::vector<int>> batches;
  std::map<int, bool> group_fd;
  for (auto& kv : groups) {
    std::vector<int>& gi = kv.second;
    std::stable_sort(gi.begin(), gi.end(), [&](int a, int b) {
      return smp[a].beta * std::pow(smp[a].k, smp[a].sigma) > smp[b].beta * std::pow(smp[b].k, smp[b].sigma);
    });
    double kmax = 0;
    for (int i : gi) kmax = std::max(kmax, smp[i].k);
    const bool fd = fd_wanted(common->coarse_solver, 2, kv.first / 2, false, false, kmax);
    group_fd[kv.first] = fd;
    NDPlan* plan = nullptr;
    if (!fd) HH_TRY(get_plan(2, kv.first / 2 + 1, &plan));
    const int64_t per = per_sample_bytes(2, kv.first, m, plan);
    const double Nn = (double)(kv.first + 1) * (kv.first + 1);
    const int bmem = (int)std::max<int64_t>(1, std::min<int64_t>(maxB, (int64_t)(budget / per)));
    int bmax = std::max(1, std::min(bmem, (int)(node_budget / Nn)));
    // HH_SWEEP_FD_WAVE=1 (A/B): size FD batches to whole waves of the GEMM tiles -- a batch
    // whose CTAs overshoot W full waves by less than 0.8 of a wave shrinks to W waves
    static const bool fd_wave = getenv("HH_SWEEP_FD_WAVE") && atoi(getenv("HH_SWEEP_FD_WAVE")) != 0;
    if (fd && fd_wave) {
      int per_sample = 1, per_sm = 1, sms = 148;
      fd_gemm_ctas2d(kv.first / 2, &per_sample, &per_sm);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, common->device);
      const double slots = (double)sms * per_sm;
      const int cnt0 = (int)gi.size(), nb0 = (cnt0 + bmax - 1) / bmax;
      const int bact = (cnt0 + nb0 - 1) / nb0;   // the batches' actual size (the group is split evenly)
      const double waves = bact * (double)per_sample / slots;
      const int W = (int)waves;
      if (W >= 1 && waves - W > 0.02 && waves - W < 0.8) bmax = std::max(1, (int)(W * slots / per_sample));
    }
    const int cnt = (int)gi.size();
    const int nb = (cnt + bmax - 1) / bmax;
    for (int k = 0; k < nb; ++k) {
      std::vector<int> bt;
      for (int i = k * cnt / nb; i < (k + 1) * cnt / nb; ++i) bt.push_back(gi[i]);
      batches.push_back(bt);
    }
  }
  // largest work first
  std::sort(batches.begin(), batches.end(), [&](const std::vector<int>& a, const std::vector<int>& b) {
    return (int64_t)smp[a[0]].n_cells * smp[a[0]].n_cells * a.size() >
           (int64_t)smp[b[0]].n_cells * smp[b[0]].n_cells * b.size();
  });
  // spec of every batch
  std::vector<BatchSpec> specs(batches.size());
  for (size_t bi = 0; bi < batches.size(); ++bi) {
    BatchSpec& sp = specs[bi];
    const std::vector<int>& bt = batches[bi];
    sp.dim = 2; sp.n = smp[bt[0]].n_cells; sp.B = (int)bt.size();
    sp.nu_pre = common->nu_pre; sp.nu_post = common->nu_post; sp.omega = common->omega; sp.m = m;
    sp.coarse = common->coarse_solver;
    sp.fd = group_fd[sp.n];
    for (int i : bt) { sp.k.push_back(smp[i].k); sp.beta.push_back(smp[i].beta); sp.sigma.push_back(smp[i].sigma); }
  }
  const int nt = std::min<int>(nstreams, (int)batches.size());
  // persistent engines: every allocation happens here, before the workers start
  // (cudaMalloc/cudaFree synchronise the whole device)
  std::vector<Engine*> engines;
  {
    std::lock_guard<std::mutex> lk(g_sweep_mu);
    auto& pool = g_sweep_engines[common->device];
    while ((int)pool.size() < nt) {
      pool.emplace_back(new Engine());
      HH_TRY(engine_init(*pool.back(), common->device));
    }
    for (int t = 0; t < nt; ++t) engines.push_back(pool[t].get());
  }
  for (Engine* E : engines) E->conc = nt > 1;
  // exclusive timed iterations when several engines share the GPU (default on;
  // HH_SWEEP_EXCL_TIMING=0: timed iterations time-share like the rest)
  static ExclGate gates[64];
  static const bool excl_timing = !getenv("HH_SWEEP_EXCL_TIMING") || atoi(getenv("HH_SWEEP_EXCL_TIMING")) != 0;
  for (Engine* E : engines) {
    E->gate = (excl_timing && nt > 1 && g_sweep_timing) ? &gates[common->device % 64] : nullptr;
    E->peers.clear();
    for (Engine* O : engines)
      if (O != E) E->peers.push_back(O->s);
  }
  for (Engine* E : engines)
    for (const BatchSpec& sp : specs) HH_TRY(reserve_pools(*E, sp));
  // ND solve schedule per (grid, batch size), timed once on an idle GPU (zero
  // factor: the schedule depends on sizes only), then cached in the shared tree
  // (HH_ND_TUNE_CONC=1: time the candidates on all worker streams at once --
  // throughput under concurrency -- instead of in isolation; measured slower:
  // 2.97 vs 2.80 s per sweep step)
  {
    static const bool tune_conc = getenv("HH_ND_TUNE_CONC") && atoi(getenv("HH_ND_TUNE_CONC")) != 0;
    Engine& E = *engines[0];
    for (const BatchSpec& sp : specs) {
      if (sp.fd) continue;   // no schedule to tune
      NDPlan* P = nullptr;
      HH_TRY(get_plan(2, sp.n / 2 + 1, &P));
      const int64_t Nc = ipow(sp.n / 2 + 1, 2);
      std::vector<NDTuneCtx> multi;
      for (Engine* Ek : engines) {
        HH_CUDA_TRY(cudaMemsetAsync(Ek->F.p, 0, (size_t)sp.B * nd_front_entries(P) * 16, Ek->s));
        HH_CUDA_TRY(cudaMemsetAsync(Ek->rc.p, 0, (size_t)sp.B * Nc * 16, Ek->s));
        HH_TRY(nd_flow_reset(P, sp.B, Ek->work.as<cplx>(), Ek->s));
        multi.push_back({Ek->F.as<cplx>(), Ek->work.as<cplx>(), varg(Ek->rc.as<cplx>(), Nc),
                         varg(Ek->ec.as<cplx>(), Nc), Ek->s});
        if (!(tune_conc && E.conc)) break;
      }
      for (Engine* Ek : engines) HH_CUDA_TRY(cudaStreamSynchronize(Ek->s));
      HH_TRY(nd_autotune(P, sp.B, E.F.as<cplx>(), E.work.as<cplx>(), varg(E.rc.as<cplx>(), Nc),
                         varg(E.ec.as<cplx>(), Nc), E.s, false, E.conc,
                         (tune_conc && E.conc && multi.size() > 1) ? &multi : nullptr));
    }
    HH_CUDA_TRY(cudaStreamSynchronize(E.s));
  }
  std::atomic<int> next(0);
  std::atomic<int> failed(0);
  std::string err;
  std::mutex err_mu;
  const bool timing = g_sweep_timing;
  auto worker = [&](Engine* Ep) {
    Engine& E = *Ep;
    if (cudaSetDevice(common->device) != cudaSuccess) { failed = 1; return; }
    E.timing = timing;
    for (double& a : E.acc_ms) a = 0;
    for (double& a : E.acc_bytes) a = 0;
    for (double& a : E.acc_bytes_all) a = 0;
    for (double& a : E.acc_model) a = 0;
    for (double& a : E.acc_model_all) a = 0;
    for (double& a : E.acc_launch) a = 0;
    E.acc_flops = E.acc_flops_all = 0;
    E.launches = 0;
    if (const char* te = getenv("HH_TIMING_EVERY")) E.timing_every = std::max(1, atoi(te));
    // sweep: sample 1 iteration in 16, run with the GPU to itself (ExclGate): the
    // phase times are kernel times; costs ~3% of the timed-region throughput
    // (1 in 8: 5.5%; profiles/r02/fd/excl_ab), nothing outside the timed region
    else E.timing_every = 16;
    const double w0 = now_s();
    int nbat = 0;
    double busy = 0;
    for (;;) {
      const int bi = next.fetch_add(1);
      if (bi >= (int)batches.size() || failed) break;
      const std::vector<int>& bt = batches[bi];
      const BatchSpec& sp = specs[bi];
      const double b0 = now_s();
      ++nbat;
      hh_status st = batch_setup(E, sp);
      std::vector<SampleOut> res;
      double t_solve = 0;
      if (st == HH_OK) {
        const int half = sp.n / 2;
        const int64_t ctr = half + (int64_t)(sp.n + 1) * half;   // unit point source at the centre (C7)
        if (!rhs) {
          st = vset(E.LF, vfine(E, E.bv), VArg(), sp.B, 2, ctr, nullptr, E.s);
        } else {
          cplx* base = E.bv.as<cplx>() + E.FL.pad + (int64_t)E.FL.G * E.FL.plane;   // owned view, entry 0
          for (size_t k = 0; k < bt.size() && st == HH_OK; ++k)
            if (cudaMemcpyAsync(base + (int64_t)k * E.FL.stride, rhs[bt[k]], E.N * 16, cudaMemcpyHostToDevice,
                                E.s) != cudaSuccess) {
              cudaGetLastError();
              hh_set_error("sweep: rhs upload failed");
              st = HH_E_CUDA;
            }
        }
        const double t0 = now_s();
        if (st == HH_OK) st = batch_solve(E, vfine(E, E.bv), vfine(E, E.xv), *o, res, nullptr);
        t_solve = now_s() - t0;
      }
      if (st != HH_OK) {
        std::lock_guard<std::mutex> lk(err_mu);
        err = hh_last_error();
        for (int i : bt) out[i].status = st;
        if (st != HH_E_SINGULAR) failed = 1;
        continue;
      }
      for (size_t k = 0; k < bt.size(); ++k) {
        hh_sample_result& r = out[bt[k]];
        r.status = res[k].status;
        r.iterations = res[k].iterations;
        r.converged = res[k].converged;
        r.rel_res_true = res[k].rel_res_true;
        r.rho = res[k].rho;
        r.setup_s = E.setup_s;
        r.solve_s = t_solve;
      }
      busy += now_s() - b0;
    }
    if (getenv("HH_DEBUG") && atoi(getenv("HH_DEBUG")) >= 3)
      fprintf(stderr, "[hh sweep] worker %p: %d batches, busy %.3f s, finished at %.3f s\n", (void*)Ep, nbat,
              busy, now_s() - w0);
    std::lock_guard<std::mutex> lk(g_sweep_mu);
    for (int t = 0; t < T_NT; ++t) {
      g_sweep_st[t] += E.acc_ms[t];
      g_sweep_st[4 + t] += E.acc_bytes[t];
      g_sweep_st[12 + t] += E.acc_bytes_all[t];
      g_sweep_st[8 + t] += E.acc_launch[t];
      g_sweep_st[16 + t] += E.acc_model[t];
      g_sweep_st[20 + t] += E.acc_model_all[t];
    }
    g_sweep_flops[0] += E.acc_flops;
    g_sweep_flops[1] += E.acc_flops_all;
    g_sweep_launches += E.launches;
  };
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) th.emplace_back(worker, engines[t]);
  for (auto& t : th) t.join();
  if (failed) { hh_set_error("%s", err.c_str()); return HH_E_CUDA; }
  return HH_OK;
}

extern "C" hh_status hh_coarse_kind(const hh_problem* p, int32_t* kind) {
  if (!p || !kind) { hh_set_error("NULL argument"); return HH_E_ARG; }
  const BatchSpec& sp = p->ep->spec;
  *kind = sp.fd ? HH_COARSE_FD : (sp.dist ? HH_COARSE_ND_DIST : HH_COARSE_ND);
  return HH_OK;
}

extern "C" hh_status hh_coarse_flops(hh_problem* p, double* flops2) {
  if (!flops2) { hh_set_error("NULL argument"); return HH_E_ARG; }
  if (p) {
    flops2[0] = p->ep->acc_flops;
    flops2[1] = p->ep->acc_flops_all;
    return HH_OK;
  }
  std::lock_guard<std::mutex> lk(g_sweep_mu);
  flops2[0] = g_sweep_flops[0];
  flops2[1] = g_sweep_flops[1];
  return HH_OK;
}

extern "C" hh_status hh_sweep(const hh_problem_desc* common, const hh_fgmres_opts* o,
                              const hh_sample* smp, int32_t n, hh_sample_result* out) {
  return sweep_run(common, o, smp, n, nullptr, out);
}

// ================================================================== shift search
// Golden-section search of the near-optimal shift exponent (PAPER.md:404-421,
// Sec. 5 step 5): for each sample minimise rho(sigma) = (r_end / r_0)^(1/end)
// of an FGMRES solve of A_0 u = f preconditioned by the V-cycle on
// A(k, beta k^sigma), over sigma in [lo, hi] to a bracket width <= tol.
// Classic two-interior-point reduction with ratio 1/phi; tie f(c) == f(d) keeps
// the right bracket [c, b].  All samples advance in lockstep rounds; every
// round's evaluations are one batched sweep.  A failed solve scores rho = 1.
extern "C" hh_status hh_shift_search(const hh_problem_desc* common, const hh_fgmres_opts* o,
                                     const hh_search_sample* smp, int32_t n, const void* const* rhs,
                                     double sigma_lo, double sigma_hi, double tol,
                                     hh_search_result* out) {
  if (!common || !o || (n && (!smp || !out || !rhs))) { hh_set_error("NULL argument"); return HH_E_ARG; }
  if (!(sigma_lo < sigma_hi) || !(tol > 0)) { hh_set_error("need sigma_lo < sigma_hi and tol > 0"); return HH_E_CONFIG; }
  if (n == 0) return HH_OK;
  const double invphi = (std::sqrt(5.0) - 1.0) / 2.0;
  struct St { double a, b, c, d, fc, fd, best_s, best_f; int evals, its; bool active; };
  std::vector<St> S(n);
  for (int i = 0; i < n; ++i) {
    St& t = S[i];
    t.a = sigma_lo; t.b = sigma_hi;
    t.c = t.b - invphi * (t.b - t.a);
    t.d = t.a + invphi * (t.b - t.a);
    t.fc = t.fd = 0; t.best_s = t.c; t.best_f = 2; t.evals = 0; t.its = 0;
    t.active = (t.b - t.a) > tol;
    memset(&out[i], 0, sizeof(out[i]));
    out[i].id = smp[i].id;
  }
  auto evaluate = [&](const std::vector<std::pair<int, double>>& pts, std::vector<double>& f) -> hh_status {
    const int m = (int)pts.size();
    std::vector<hh_sample> q(m);
    std::vector<const void*> r(m);
    for (int k = 0; k < m; ++k) {
      const hh_search_sample& z = smp[pts[k].first];
      q[k].id = k; q[k].n_cells = z.n_cells; q[k].k = z.k; q[k].beta = z.beta; q[k].sigma = pts[k].second;
      r[k] = rhs[pts[k].first];
    }
    std::vector<hh_sample_result> res(m);
    HH_TRY(sweep_run(common, o, q.data(), m, r.data(), res.data()));
    f.resize(m);
    for (int k = 0; k < m; ++k) {
      const bool ok = res[k].status == HH_OK && std::isfinite(res[k].rho);
      f[k] = ok ? res[k].rho : 1.0;
      St& t = S[pts[k].first];
      t.evals++;
      t.its += res[k].iterations;
      if (f[k] < t.best_f) { t.best_f = f[k]; t.best_s = pts[k].second; }
    }
    return HH_OK;
  };
  // round 0: both interior points
  {
    std::vector<std::pair<int, double>> pts;
    for (int i = 0; i < n; ++i) { pts.push_back({i, S[i].c}); pts.push_back({i, S[i].d}); }
    std::vector<double> f;
    HH_TRY(evaluate(pts, f));
    for (int i = 0; i < n; ++i) { S[i].fc = f[2 * i]; S[i].fd = f[2 * i + 1]; }
  }
  for (;;) {
    std::vector<std::pair<int, double>> pts;
    std::vector<int> side;
    for (int i = 0; i < n; ++i) {
      St& t = S[i];
      if (!t.active) continue;
      if (t.fc < t.fd) {   // minimum in [a, d]
        t.b = t.d; t.d = t.c; t.fd = t.fc;
        t.c = t.b - invphi * (t.b - t.a);
        side.push_back(0);
        pts.push_back({i, t.c});
      } else {             // minimum in [c, b]
        t.a = t.c; t.c = t.d; t.fc = t.fd;
        t.d = t.a + invphi * (t.b - t.a);
        side.push_back(1);
        pts.push_back({i, t.d});
      }
    }
    if (pts.empty()) break;
    std::vector<double> f;
    HH_TRY(evaluate(pts, f));
    for (size_t k = 0; k < pts.size(); ++k) {
      St& t = S[pts[k].first];
      (side[k] == 0 ? t.fc : t.fd) = f[k];
      t.active = (t.b - t.a) > tol;
    }
  }
  for (int i = 0; i < n; ++i) {
    out[i].sigma_hat = 0.5 * (S[i].a + S[i].b);
    out[i].sigma_best = S[i].best_s;
    out[i].rho_best = S[i].best_f;
    out[i].evaluations = S[i].evals;
    out[i].iterations_total = S[i].its;
    out[i].status = HH_OK;
  }
  return HH_OK;
}
