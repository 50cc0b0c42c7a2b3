// Slab decomposition: partition and transport (comm.cu).
#pragma once
#include <vector>
#include "hh_internal.cuh"

struct Comm {            // one NCCL communicator (one slab per process)
  void* comm = nullptr;  // ncclComm_t
  int rank = 0, nranks = 1;
};

// Everything the exchange steps of one slab-decomposed solve need.
struct SlabCtx {
  int B = 1;                    // slabs held by this process (entries of the batch)
  const int2* slab = nullptr;   // device [B] (z0, z1)
  std::vector<int2> h_slab;     // host copy
  std::vector<int> all_z;       // global plane bounds of all ranks' slab ranges (nranks + 1)
  int G = 0, maxloc = 0, nc1 = 0;
  int64_t plane = 0, cplane = 0;
  Comm* comm = nullptr;         // NULL: in-process slabs only
  cplx* hsend = nullptr;        // NCCL halo staging, [2][G * plane] each
  cplx* hrecv = nullptr;
};

// Global slab bounds: S slabs of the planes 0..n, even boundaries (coarse planes
// split the same way); slab k owns [z[k], z[k+1]).
std::vector<int> slab_bounds(int n, int S);

hh_status comm_unique_id(void* out128);
hh_status comm_create(const void* id128, int rank, int nranks, int device, Comm** out);
void comm_destroy(Comm* c);

// ghost planes of fine vector v (ghosted entry layout, Level.stride)
hh_status slab_halo(const SlabCtx& X, VArg v, cudaStream_t s);
// owned coarse planes of r_c -> all slabs (full coarse vectors per entry)
hh_status slab_coarse_allgather(const SlabCtx& X, VArg rc, cudaStream_t s);
// in-place sum over the processes of `count` doubles (no-op without a communicator)
hh_status slab_allreduce(const SlabCtx& X, double* buf, size_t count, cudaStream_t s);
// user vector (concatenated owned parts of this process' slabs) <-> entry owned views
hh_status slab_user_copy(const SlabCtx& X, VArg ent, void* user, int to_user, cudaStream_t s);
