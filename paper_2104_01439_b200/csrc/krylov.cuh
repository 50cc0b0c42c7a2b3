// Batched FGMRES state and kernel launchers (krylov.cu).
#pragma once
#include "hh_internal.cuh"

enum { HHK_RUN = 0, HHK_CONVERGED = 1, HHK_MAXIT = 2, HHK_BREAKDOWN = 3, HHK_NAN = 4, HHK_FIXED = 5,
       HHK_NDFAIL = 6 /* the coarse solve's dataflow schedule timed out (nd_solve) */ };

struct KState {              // per-sample device arrays, [B] each (hist: [B][hist_len])
  double* bnorm = nullptr;   // ||b||
  double* res = nullptr;     // |g_{j+1}| (least-squares residual)
  double* rtrue = nullptr;   // ||b - A_0 x|| at exit
  int* status = nullptr;     // HHK_*
  int* its = nullptr;        // preconditioner applications so far
  int* jend = nullptr;       // Arnoldi steps of the current cycle
  int* jlast = nullptr;      // Arnoldi steps of the last finished cycle (orthogonality diagnostic)
  double* hist = nullptr;    // |g_{j+1}| / ||b|| per iteration
};

// Fine vectors of entry b are ghosted slabs of Nst nodes (Level.stride); the
// Krylov kernels work on the OWNED view: offset G * plane, length
// (z1 - z0) * plane with (z0, z1) = slab[b] (the whole grid without slabs).
// slabred = 1: the entries are slabs of ONE problem (and possibly one slab of a
// multi-process problem): every reduction is left as a per-entry partial in
// red*, summed over the entries (and across processes by the transport) and
// finished by the *_fin kernels, so every entry holds identical Krylov state.
struct KArgs {
  int64_t Nst = 0;                      // entry stride of a fine vector
  int n = 0, G = 0;
  int64_t plane = 0;
  const int2* slab = nullptr;
  cplx* V = nullptr; int64_t Vbs = 0;   // [B][m+1][Nst]
  cplx* Z = nullptr; int64_t Zbs = 0;   // [B][m][Nst]
  cplx* w = nullptr;                    // [B][Nst]
  cplx* H = nullptr; int64_t HB = 0; int ldh = 0;   // [B][m][ldh] column-major
  double* vscale = nullptr; double* cs = nullptr; cplx* sn = nullptr; cplx* g = nullptr;
  cplx* y = nullptr; int ldv = 0;       // [B][ldv]
  cplx* cpart = nullptr; int ldp = 0;   // [B][nblk][ldp]
  double* dpart = nullptr;              // [B][nblk]
  unsigned* counter = nullptr;          // [B]
  unsigned* gcounter = nullptr; int ldg = 0;   // [B][ldg] k_mdot group counters (ldg >= ceil(nblk / 32))
  const int* jdev = nullptr;
  int nblk = 1;
  double rtol = 1e-6;
  int max_iters = 500, fixed_iters = 0, hist_len = 0;
  KState ks;
  int slabred = 0;
  cplx* red = nullptr; int ldr = 0;     // [B][ldr] multi-dot partials (slabred)
  double* red2 = nullptr;               // [B] norm partials (slabred)
  // re-orthogonalisation (hh_fgmres_opts.reorth, reading C11): 0 none (single-pass
  // CGS), 1 selective (DGKS: second CGS pass when ||w'|| < ||w|| / sqrt 2), 2 always
  int reorth = 0;
  double* wnorm2 = nullptr;             // [B] ||w||^2 before the first pass (reorth = 1)
  int* reo = nullptr;                   // [B] 1: the second pass runs for this sample / step
};

// pass 1: h = V_j^H w, w' = w - V_j h (-> V[j+1]); pass 2 (reorth): the second
// CGS pass on V[j+1] for the samples whose pass 1 asked for it (reo[b] = 1)
hh_status krylov_mdot(const KArgs& A, int B, cudaStream_t s, int pass = 1);
hh_status krylov_update(const KArgs& A, int B, cudaStream_t s, int pass = 1);
hh_status krylov_advance(int* jdev, int v, cudaStream_t s);    // v < 0: ++j, else j = v
hh_status krylov_cycle_end(const KArgs& A, int B, VArg x, cudaStream_t s);
hh_status krylov_norm(const KArgs& A, int B, VArg r, int mode, cudaStream_t s);
// slabred: finish a reduction after the partials were combined across processes
hh_status krylov_mdot_fin(const KArgs& A, int B, cudaStream_t s, int pass = 1);
hh_status krylov_update_fin(const KArgs& A, int B, cudaStream_t s, int pass = 1);
// max over pairs (a, c) of the last cycle's basis v_0..v_jlast of |<v_a, v_c> - delta_ac|
// for entry b (blocks; diagnostic of the Arnoldi orthogonality)
hh_status krylov_orth_loss(const KArgs& A, int b, double* loss, int* nvec, cudaStream_t s);
hh_status krylov_norm_fin(const KArgs& A, int B, int mode, cudaStream_t s);
