// Slab decomposition transport (north_star: "Large single solves
// use a slab decomposition, with NCCL halo exchange over NVLink for the stencil
// and allreduce for Arnoldi inner products").
//
// The fine grid is cut into slabs of whole planes of the slowest axis (y in 2D,
// z in 3D) with even boundaries, so the coarse planes (2Z) split the same way.
// One solve = S slabs; a process holds either all S slabs as the entries of one
// batch (in-process slabs: the exchanges are device copies between entries, the
// reductions sum over the entries) or ONE slab with an NCCL communicator over
// the S processes (one per GPU).  Three exchange steps exist:
//   halo      : G owned boundary planes of a fine vector -> the neighbours' ghost planes
//   allgather : the owned planes of the restricted residual r_c -> every slab
//               (the coarse solve is replicated, SURVEY 8(e) "first version")
//   allreduce : the multi-dot partials and the squared norms of the Arnoldi step
// NCCL is loaded at run time (dlopen of libnccl.so.2, normally the copy torch
// already loaded), so the library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>
#include <mutex>
#include "comm.cuh"

// ------------------------------------------------------------------ NCCL API
namespace {
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { api.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror(); return; }
    bool good = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<typename std::remove_reference<decltype(fn)>::type>(dlsym(h, name));
      if (!fn) { good = false; api.err = std::string("NCCL symbol missing: ") + name; }
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.Broadcast, "ncclBroadcast");
    sym(api.GetErrorString, "ncclGetErrorString");
    api.ok = good;
  });
  return api;
}

#define HH_NCCL_TRY(expr)                                                                \
  do {                                                                                   \
    ncclResult_t _r = (expr);                                                            \
    if (_r != ncclSuccess) {                                                             \
      hh_set_error("NCCL error %d (%s) at %s:%d", (int)_r, nccl().GetErrorString(_r),     \
                   __FILE__, __LINE__);                                                  \
      return HH_E_NCCL;                                                                  \
    }                                                                                    \
  } while (0)

// ------------------------------------------------------------------ kernels
// in-process halo: entry b's first / last G owned planes -> ghost planes of b-1 / b+1
__global__ void k_halo_local(VArg v, const int2* __restrict__ slab, int G, int64_t plane, int B) {
  const int b = blockIdx.y;
  const int2 sl = slab[b];
  const int64_t cnt = (int64_t)G * plane;
  cplx* me = v.at(b);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (b > 0) {   // my first owned planes -> upper ghost of b-1 (starts at its local plane G + owned)
      const int2 sp = slab[b - 1];
      v.at(b - 1)[(int64_t)(G + sp.y - sp.x) * plane + i] = me[(int64_t)G * plane + i];
    }
    if (b < B - 1) {   // my last owned planes -> lower ghost of b+1 (local planes 0..G-1)
      v.at(b + 1)[i] = me[(int64_t)(sl.y - sl.x) * plane + i];
    }
  }
}

// NCCL halo staging: pack the boundary planes of the first / last entry (mode 0),
// unpack the received planes into their ghost planes (mode 1)
__global__ void k_halo_stage(VArg v, const int2* __restrict__ slab, int G, int64_t plane, int B,
                             cplx* __restrict__ snd, cplx* __restrict__ rcv, int lo, int hi, int mode) {
  const int64_t cnt = (int64_t)G * plane;
  const int2 sl = slab[B - 1];
  const int64_t own = (int64_t)(sl.y - sl.x);
  cplx* first = v.at(0);
  cplx* last = v.at(B - 1);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (mode == 0) {
      if (lo) snd[i] = first[cnt + i];                 // first owned planes -> rank - 1
      if (hi) snd[cnt + i] = last[own * plane + i];    // last owned planes  -> rank + 1
    } else {
      if (lo) first[i] = rcv[i];                                 // lower ghost <- rank - 1
      if (hi) last[(G + own) * plane + i] = rcv[cnt + i];        // upper ghost <- rank + 1
    }
  }
}

// in-process allgather of the owned coarse planes: entry e's planes [z0/2, ..) -> every entry
__global__ void k_cgather_local(VArg rc, const int2* __restrict__ slab, int64_t cplane, int nc1, int B) {
  const int e = blockIdx.y;   // source entry
  const int2 sl = slab[e];
  const int Z0 = sl.x / 2, Z1 = min(nc1, (sl.y + 1) / 2);
  const int64_t o0 = (int64_t)Z0 * cplane, cnt = (int64_t)(Z1 - Z0) * cplane;
  const cplx* src = rc.at(e) + o0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const cplx v = src[i];
    for (int b = 0; b < B; ++b)
      if (b != e) rc.at(b)[o0 + i] = v;
  }
}

// user (concatenated owned parts of the entries) <-> entry owned views
__global__ void k_user_copy(VArg ent, cplx* __restrict__ user, const int2* __restrict__ slab,
                            int G, int64_t plane, int to_user) {
  const int b = blockIdx.y;
  const int2 sl = slab[b];
  const int2 s0 = slab[0];
  const int64_t uoff = (int64_t)(sl.x - s0.x) * plane, cnt = (int64_t)(sl.y - sl.x) * plane;
  cplx* me = ent.at(b) + (int64_t)G * plane;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (to_user) user[uoff + i] = me[i];
    else me[i] = user[uoff + i];
  }
}
}  // namespace

// ------------------------------------------------------------------ host API
std::vector<int> slab_bounds(int n, int S) {
  std::vector<int> z(S + 1);
  const int half = n / 2;
  for (int k = 0; k < S; ++k) z[k] = 2 * (int)(((int64_t)k * half) / S);
  z[S] = n + 1;
  return z;
}

hh_status comm_unique_id(void* out128) {
  NcclApi& a = nccl();
  if (!a.ok) { hh_set_error("%s", a.err.c_str()); return HH_E_NCCL; }
  ncclUniqueId id;
  HH_NCCL_TRY(a.GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out128, &id, 128);
  return HH_OK;
}

hh_status comm_create(const void* id128, int rank, int nranks, int device, Comm** out) {
  NcclApi& a = nccl();
  if (!a.ok) { hh_set_error("%s", a.err.c_str()); return HH_E_NCCL; }
  HH_CUDA_TRY(cudaSetDevice(device));
  ncclUniqueId id;
  memcpy(&id, id128, 128);
  ncclComm_t c = nullptr;
  HH_NCCL_TRY(a.CommInitRank(&c, nranks, id, rank));
  Comm* cm = new Comm();
  cm->comm = c;
  cm->rank = rank;
  cm->nranks = nranks;
  *out = cm;
  return HH_OK;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (c->comm && nccl().ok) nccl().CommDestroy((ncclComm_t)c->comm);
  delete c;
}

hh_status slab_halo(const SlabCtx& X, VArg v, cudaStream_t s) {
  if (X.B > 1) {
    const int64_t cnt = (int64_t)X.G * X.plane;
    const unsigned gx = (unsigned)std::min<int64_t>(1024, (cnt + 255) / 256);
    k_halo_local<<<dim3(gx, X.B), 256, 0, s>>>(v, X.slab, X.G, X.plane, X.B);
    HH_CUDA_TRY(cudaGetLastError());
  }
  if (X.comm && X.comm->nranks > 1) {
    // the vector pointer may depend on the device-side Arnoldi index (V_j): stage the
    // boundary planes through fixed buffers so the NCCL calls are graph-capturable
    NcclApi& a = nccl();
    ncclComm_t c = (ncclComm_t)X.comm->comm;
    const int r = X.comm->rank, R = X.comm->nranks;
    const int lo = r > 0, hi = r < R - 1;
    const int64_t cnt = (int64_t)X.G * X.plane;
    const unsigned gx = (unsigned)std::min<int64_t>(1024, (cnt + 255) / 256);
    k_halo_stage<<<gx, 256, 0, s>>>(v, X.slab, X.G, X.plane, X.B, X.hsend, X.hrecv, lo, hi, 0);
    HH_CUDA_TRY(cudaGetLastError());
    const size_t nd = (size_t)cnt * 2;   // doubles
    HH_NCCL_TRY(a.GroupStart());
    if (lo) {
      HH_NCCL_TRY(a.Send((double*)X.hsend, nd, ncclFloat64, r - 1, c, s));
      HH_NCCL_TRY(a.Recv((double*)X.hrecv, nd, ncclFloat64, r - 1, c, s));
    }
    if (hi) {
      HH_NCCL_TRY(a.Send((double*)(X.hsend + cnt), nd, ncclFloat64, r + 1, c, s));
      HH_NCCL_TRY(a.Recv((double*)(X.hrecv + cnt), nd, ncclFloat64, r + 1, c, s));
    }
    HH_NCCL_TRY(a.GroupEnd());
    k_halo_stage<<<gx, 256, 0, s>>>(v, X.slab, X.G, X.plane, X.B, X.hsend, X.hrecv, lo, hi, 1);
    HH_CUDA_TRY(cudaGetLastError());
  }
  return HH_OK;
}

hh_status slab_coarse_allgather(const SlabCtx& X, VArg rc, cudaStream_t s) {
  if (X.B > 1) {
    const int64_t cnt = (int64_t)(X.maxloc / 2 + 1) * X.cplane;
    const unsigned gx = (unsigned)std::min<int64_t>(1024, (cnt + 255) / 256);
    k_cgather_local<<<dim3(gx, X.B), 256, 0, s>>>(rc, X.slab, X.cplane, X.nc1, X.B);
    HH_CUDA_TRY(cudaGetLastError());
  }
  if (X.comm && X.comm->nranks > 1) {
    NcclApi& a = nccl();
    ncclComm_t c = (ncclComm_t)X.comm->comm;
    double* base = (double*)rc.p;   // entry 0 (flat coarse vector, B == 1 with NCCL)
    HH_NCCL_TRY(a.GroupStart());
    for (int q = 0; q < X.comm->nranks; ++q) {
      const int Z0 = X.all_z[q] / 2, Z1 = std::min(X.nc1, (X.all_z[q + 1] + 1) / 2);
      const size_t off = (size_t)Z0 * X.cplane * 2, cnt = (size_t)(Z1 - Z0) * X.cplane * 2;
      HH_NCCL_TRY(a.Broadcast(base + off, base + off, cnt, ncclFloat64, q, c, s));
    }
    HH_NCCL_TRY(a.GroupEnd());
  }
  return HH_OK;
}

hh_status slab_allreduce(const SlabCtx& X, double* buf, size_t count, cudaStream_t s) {
  if (X.comm) {   // also for a single rank: exercises the NCCL path (a copy)
    NcclApi& a = nccl();
    HH_NCCL_TRY(a.AllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)X.comm->comm, s));
  }
  return HH_OK;
}

hh_status slab_user_copy(const SlabCtx& X, VArg ent, void* user, int to_user, cudaStream_t s) {
  int64_t mx = 0;
  for (const int2& z : X.h_slab) mx = std::max<int64_t>(mx, (int64_t)(z.y - z.x) * X.plane);
  const unsigned gx = (unsigned)std::min<int64_t>(2048, (mx + 255) / 256);
  k_user_copy<<<dim3(std::max(1u, gx), X.B), 256, 0, s>>>(ent, (cplx*)user, X.slab, X.G, X.plane, to_user);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

// ------------------------------------------------------------------ distributed coarse solve transport
hh_status comm_group(bool start) {
  NcclApi& a = nccl();
  if (!a.ok) { hh_set_error("%s", a.err.c_str()); return HH_E_NCCL; }
  HH_NCCL_TRY(start ? a.GroupStart() : a.GroupEnd());
  return HH_OK;
}
hh_status comm_send(Comm* c, const void* buf, size_t bytes, int peer, cudaStream_t s) {
  HH_NCCL_TRY(nccl().Send(buf, bytes / 8, ncclFloat64, peer, (ncclComm_t)c->comm, s));
  return HH_OK;
}
hh_status comm_recv(Comm* c, void* buf, size_t bytes, int peer, cudaStream_t s) {
  HH_NCCL_TRY(nccl().Recv(buf, bytes / 8, ncclFloat64, peer, (ncclComm_t)c->comm, s));
  return HH_OK;
}
hh_status comm_bcast(Comm* c, void* buf, size_t bytes, int root, cudaStream_t s) {
  HH_NCCL_TRY(nccl().Broadcast(buf, buf, bytes / 8, ncclFloat64, root, (ncclComm_t)c->comm, s));
  return HH_OK;
}
