/*
 * hh.h — C ABI of the B200 hot path of arXiv 2104.01439 ("PAPER"):
 * FGMRES on the Q1 finite-element Helmholtz system A_0, right-preconditioned
 * by one two-grid V(nu,nu) cycle on the complex-shifted operator A_eps.
 *
 *   A(k, eps) = K - M(k, eps) - i B(k)                (Eq. sys_matrix)
 *   A_0 = A(k, 0), A_eps = A(k, eps), eps_e = beta * k_e^sigma
 *   V-cycle: Alg. 1, L = 2, damped Jacobi, I^T / I
 *   transfers, exact coarse solve factored once
 *   FGMRES: right-preconditioned, flexible
 *
 * Conventions (all entry points):
 *  - Every call returns hh_status; HH_OK = 0.  No C++ exception crosses the
 *    ABI.  On a non-OK status hh_last_error() returns a thread-local message.
 *  - Vectors are caller-owned DEVICE pointers to complex128 stored as
 *    interleaved (re, im) doubles — the layout of torch.complex128 — of
 *    length (n+1)^dim (fine) or (n/2+1)^dim (coarse), nodes ordered
 *    lexicographically with x fastest: node (i, j[, l]) -> i + (n+1) j [+ (n+1)^2 l].
 *    They must be 16-byte aligned.  Host pointers are accepted only where
 *    stated (hh_problem_desc.k_elem*, hh_fgmres_solve_host).
 *  - The library owns everything else (coefficients, coarse factor, Krylov
 *    bases, scratch).  It allocates in hh_setup_problem / hh_sweep and
 *    frees in hh_destroy_problem; hot calls (apply_op, vcycle,
 *    fgmres_solve) never allocate.
 *  - One handle per thread/stream; handles are not thread-safe.  Calls
 *    marked "async" are enqueued on the handle's stream and return without
 *    synchronising; calls marked "blocks" synchronise that stream.
 *  - Non-convergence is a RESULT (report.converged = 0), not an error.
 */
#ifndef HH_H_
#define HH_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HH_OK = 0,
  HH_E_ARG = 1,        /* NULL pointer / invalid enum                                   */
  HH_E_CONFIG = 2,     /* dim not in {2,3}, n odd or < 4, omega not in (0,1], nu < 1 ... */
  HH_E_DIM = 3,        /* size mismatch                                                 */
  HH_E_CUDA = 4,       /* CUDA runtime error (message has the CUDA error string)        */
  HH_E_NCCL = 5,       /* reserved: NCCL error (slab decomposition)                     */
  HH_E_OOM = 6,        /* device allocation failed                                      */
  HH_E_SINGULAR = 7,   /* zero Jacobi diagonal or zero coarse pivot (message has k, eps, h) */
  HH_E_BREAKDOWN = 8,  /* Arnoldi breakdown with a residual above tolerance             */
  HH_E_DIVERGED = 9,   /* NaN/Inf in the Krylov recurrence                              */
  HH_E_STATE = 10      /* call not valid in the handle's state                          */
} hh_status;

typedef struct hh_problem hh_problem;   /* opaque */

/* operator selector for hh_apply_op */
enum { HH_OP_A0 = 0, HH_OP_AEPS = 1, HH_OP_AEPS_COARSE = 2 };

/* coarse direct solver (Alg. 1 line 3; factored once per setup,
 * PAPER.md:511-512):
 *  HH_COARSE_ND: nested-dissection LDL^T-type factor (no pivoting,
 *    reading C18); with a slab decomposition every rank holds the whole factor
 *    and solves redundantly (SURVEY.md 8(e) "first version");
 *  HH_COARSE_ND_DIST (slab decompositions only): distributed exact solve --
 *    slab-aligned nested dissection whose top separators are the P-1 coarse
 *    interface planes at the slab boundaries, eliminated middle-first over the
 *    chain of slabs (block cyclic reduction of the block-tridiagonal interface
 *    Schur complement); rank r factors and solves only its slab interior and the
 *    interface plane it owns, Schur complements / update vectors move to the
 *    parent's owner and the interface solutions are broadcast (NCCL, or device
 *    copies between in-process slabs).  Needs >= 2 coarse planes per slab.
 *    (The paper's own distributed step is parallel MUMPS LU, PAPER.md:511,
 *    1463-1466.)
 *  HH_COARSE_FD (constant k only): the same exact solve by fast diagonalisation.
 *    For constant k the Q1 coarse operator is the Kronecker sum
 *    A = sum_axes M1 x .. x (K1 - ik E) x .. x M1 - (k^2 + i eps) M1 x .. x M1
 *    of the 1D stiffness K1, mass M1 and boundary selector E, so
 *    A^{-1} = (V x .. x V) diag(1/(lam_i + lam_j (+ lam_l) - k^2 - i eps)) (V^T x .. x V^T)
 *    with S0 V = M1 V Lambda (V^T M1 V = I): the eigenpairs come from the DCT-I
 *    basis plus a rank-one secular equation per parity (validated), the solve is
 *    2 d complex GEMMs per folded parity block on the FP64 tensor cores.  The
 *    product is the exact coarse solution (parity with the oracle's LU <= 1e-13).
 *  HH_COARSE_AUTO: FD for constant k when the dense transforms beat the factor
 *    (2D nc <= 512, 3D nc <= 256, k h_c <= 2.5) and its validation passes, the
 *    ND factor otherwise (heterogeneous k, slab-distributed factor, fallback).  */
enum { HH_COARSE_AUTO = 0, HH_COARSE_ND = 1, HH_COARSE_ND_DIST = 2, HH_COARSE_FD = 3 };

typedef struct {
  int32_t dim;                  /* 2 | 3                                                    */
  int32_t n_cells;              /* fine cells per side, even, >= 4; Omega=(0,1)^dim, h=1/n   */
  double  k_const;              /* wavenumber, used iff k_elem == NULL                      */
  const double* k_elem;         /* optional per-fine-element k_e, n^dim, x fastest (HOST)    */
  const double* k_elem_coarse;  /* required iff k_elem != NULL: (n/2)^dim (HOST)             */
  double  beta, sigma;          /* eps_e = beta * k_e^sigma; beta = 0 gives eps = 0          */
  int32_t nu_pre, nu_post;      /* Jacobi steps (BASELINE: 2, 2), 1..4                       */
  double  omega;                /* Jacobi damping (BASELINE: 0.6), in (0, 1]                 */
  int32_t coarse_solver;        /* HH_COARSE_*                                              */
  int32_t device;               /* CUDA device ordinal                                      */
  void*   stream;               /* cudaStream_t for every async call on this handle (NULL = legacy default) */
  int32_t max_restart;          /* Krylov workspace: largest FGMRES restart length (m) this handle will run */
  /* Slab decomposition of ONE solve (north_star "slab decomposition,
   * with NCCL halo exchange ... and allreduce for Arnoldi inner products").  The
   * planes 0..n of the slowest axis (y in 2D, z in 3D) are cut into S slabs with
   * even boundaries (hh_slab_bounds); the coarse solve is replicated.
   *  - nslabs_local = S > 1, nccl_id = NULL: all S slabs in this process (the
   *    exchanges are device copies; same arithmetic as S processes).
   *  - nccl_id != NULL: slab `rank` of S = nranks processes (one per GPU), NCCL
   *    communicator created from the id (collective: every rank calls setup).
   * User vectors of a slab handle hold the handle's OWNED planes only
   * (hh_local_layout); with S = 1 that is the whole grid.                    */
  int32_t nslabs_local;         /* 0 or 1: no in-process slabs                              */
  int32_t rank, nranks;         /* NCCL process group (used iff nccl_id != NULL)            */
  const void* nccl_id;          /* 128-byte ncclUniqueId from hh_nccl_unique_id(), or NULL  */
  /* Shift exponent: 0 = fixed sigma; p = 1..3 = the fitted map sigma_p(k_e, l)
   * of PAPER.md:437-443 with Table 1 row p, l = log2(n_cells)
   * of the FINE mesh, evaluated per element on both levels (eps = beta k^sigma_p,
   * PAPER.md:532-533).                                                       */
  int32_t shift_map;
} hh_problem_desc;

typedef struct {
  int32_t restart;              /* m (<= desc.max_restart)                                  */
  int32_t max_iters;            /* total preconditioner applications cap (BASELINE reading: 500) */
  int32_t fixed_iters;          /* > 0: run exactly this many Arnoldi steps (parity at threshold) */
  double  rtol;                 /* stop when |g_{j+1}| <= rtol * ||b||                      */
  int32_t check_every;          /* host reads the device convergence flag every this many steps (>=1) */
  /* Orthogonalisation of the Arnoldi step (PAPER.md:357-359 is silent; SURVEY 8(c)
   * C11): 0 = single-pass classical Gram-Schmidt (default: one
   * batched multi-dot pass + one update pass); 1 = selective re-orthogonalisation
   * (DGKS): a second CGS pass whenever ||w'|| < ||w|| / sqrt(2); 2 = always two
   * passes (CGS2).  Anything else: HH_E_CONFIG.                                  */
  int32_t reorth;
} hh_fgmres_opts;

typedef struct {
  int32_t iterations;           /* preconditioner applications                              */
  int32_t restarts;
  int32_t converged;
  double  rel_res_lsq;          /* |g_{j+1}| / ||b|| at exit                               */
  double  rel_res_true;         /* ||b - A_0 x|| / ||b|| recomputed at exit */
  double  rho;                  /* (rel_res_true)^(1/iterations)             */
  double  setup_s;              /* handle setup incl. coarse factorisation (s)              */
  double  solve_s;              /* this solve (s, device events)                            */
} hh_fgmres_report;

typedef struct {
  int64_t id;
  int32_t n_cells;              /* 2D, constant k                                          */
  double  k, beta, sigma;
} hh_sample;

typedef struct {
  int64_t id;
  int32_t status, iterations, converged;
  double  rel_res_true, rho, setup_s, solve_s;
} hh_sample_result;

/* Build a problem: coefficients, coarse operator A_eps^{(1)} (rediscretised on
 * the 2h mesh) and its factorisation, Krylov workspace.  blocks. */
hh_status hh_setup_problem(const hh_problem_desc* d, hh_problem** out);

/* Node counts: fine = this handle's owned nodes (the user-vector length; the
 * whole grid (n+1)^dim without slabs), coarse = (n/2+1)^dim (replicated).      */
hh_status hh_layout(const hh_problem* p, int64_t* n_fine_nodes, int64_t* n_coarse_nodes);

/* Owned part of the fine grid: n_local_nodes = n_planes * (n+1)^(dim-1) nodes of
 * the global planes [first_plane, first_plane + n_planes), x fastest.          */
hh_status hh_local_layout(const hh_problem* p, int64_t* n_local_nodes, int64_t* first_plane,
                          int64_t* n_planes);

/* Slab bounds used by the slab decomposition: z[0..nslabs], slab k owns the
 * planes [z[k], z[k+1]) (host only, no GPU needed).                            */
hh_status hh_slab_bounds(int32_t n_cells, int32_t nslabs, int32_t* z);

/* A fresh ncclUniqueId (128 bytes) for hh_problem_desc.nccl_id; call on one rank
 * and broadcast (e.g. with torch.distributed).  NCCL is loaded at run time;
 * HH_E_NCCL if it cannot be loaded.                                            */
hh_status hh_nccl_unique_id(void* id128);

/* y = A x with A = A_0 | A_eps (fine, matrix-free) | A_eps^{(1)} (coarse).
 * x, y: device complex128, distinct; fine: owned-node vectors (hh_layout),
 * coarse: full coarse vectors.  async. (PAPER.md:387-396 semi matrix-free) */
hh_status hh_apply_op(hh_problem* p, int32_t op, const void* x, void* y);

/* z = P_eps^{-1} f: one V(nu_pre, nu_post) cycle from a zero initial guess
 * (Alg. 1).  f, z: device complex128 fine vectors. async. */
hh_status hh_vcycle(hh_problem* p, const void* f, void* z);

/* Coarse direct solve e = (A_eps^{(1)})^{-1} r (coarse device vectors). async. */
hh_status hh_coarse_solve(hh_problem* p, const void* r, void* e);

/* FGMRES(m) on A_0 x = b with right preconditioner one V-cycle
 * (PAPER.md:357-360).  b: device; x: device, in: the initial guess x0 (the
 * paper's u^(0); the BASELINE configs use x0 = 0, so pass zeros),
 * out: solution.  r_0 = b - A_0 x0; the stopping threshold stays rtol ||b||
 * and restarts recompute r = b - A_0 x (reading C14).  res_hist: optional HOST
 * array of max_iters+1 doubles receiving |g_{j+1}|/||b|| per iteration (entry 0
 * = 1).  Errors: HH_E_CONFIG (restart not in 1..max_restart,
 * max_iters/fixed_iters out of range, reorth not in 0..2); HH_E_CUDA also when
 * the coarse solve's dataflow schedule timed out (never a silent wrong
 * result; the schedule is then disabled for the handle's grid).  blocks. */
hh_status hh_fgmres_solve(hh_problem* p, const void* b, void* x, const hh_fgmres_opts* o,
                          hh_fgmres_report* r, double* res_hist);

/* Same, with HOST b and x (complex128; x in: x0, out: solution): the
 * host<->device copies are part of the call (end-to-end path).  blocks. */
hh_status hh_fgmres_solve_host(hh_problem* p, const void* b_host, void* x_host,
                               const hh_fgmres_opts* o, hh_fgmres_report* r);

/* Orthogonality of the Arnoldi basis of the LAST cycle of the last solve on
 * this handle (diagnostic; SURVEY 8(c) "FGMRES" pin):
 * max_loss = max over a, c <= J of |<v_a, v_c> - delta_ac| for the normalised
 * basis v_0..v_J (J = Arnoldi steps of that cycle; a zero last vector after a
 * breakdown is excluded), nvec = J + 1.  HH_E_STATE for slab handles.  blocks. */
hh_status hh_arnoldi_orthogonality(hh_problem* p, double* max_loss, int32_t* nvec);

typedef struct {
  int64_t id;
  int32_t n_cells;              /* 2D, constant k                                          */
  double  k, beta;              /* eps = beta k^sigma, sigma searched                       */
} hh_search_sample;

typedef struct {
  int64_t id;
  int32_t status, evaluations, iterations_total;
  double  sigma_hat;            /* midpoint of the final bracket (width <= tol)             */
  double  sigma_best, rho_best; /* best evaluated point and its rho                         */
} hh_search_result;

/* Sweep: for each 2D constant-k sample, set up, factor and solve with a unit
 * point source at the centre node (BASELINE configs[1]); common carries dim,
 * nu, omega, device, stream and coarse_solver (HH_COARSE_AUTO: fast
 * diagonalisation per batch where it applies, ND factor otherwise or after a
 * failed FD validation; HH_COARSE_ND / HH_COARSE_FD force one; ND_DIST is
 * rejected).  Samples are grouped by grid, ordered by shift strength and run in
 * lockstep batches on several engine streams; results do not depend on the
 * batching.  s, out: HOST arrays of n entries.  blocks. */
hh_status hh_sweep(const hh_problem_desc* common, const hh_fgmres_opts* o,
                   const hh_sample* s, int32_t n, hh_sample_result* out);

/* Near-optimal shift search (Sec. 5 steps 1-6, step 5):
 * for each sample, golden-section search of sigma in [sigma_lo, sigma_hi] (paper:
 * [1, 2], tol 1e-2) minimising rho(sigma) = (r_end/r_0)^(1/end) of the FGMRES
 * solve of A_0 u = f (x0 = 0, budget o: paper rtol 1e-8, max_iters 50)
 * preconditioned by the V-cycle on A(k, beta k^sigma).  rhs[i]: HOST complex128
 * right-hand side of sample i ((n+1)^2 nodes; paper: components U[-1,1]), reused
 * for every sigma.  Tie f(c) == f(d) keeps [c, b]; a failed solve scores rho = 1.
 * Every round of evaluations is one batched sweep.  s, rhs, out: HOST.  blocks. */
hh_status hh_shift_search(const hh_problem_desc* common, const hh_fgmres_opts* o,
                          const hh_search_sample* s, int32_t n, const void* const* rhs,
                          double sigma_lo, double sigma_hi, double tol, hh_search_result* out);

/* Local Fourier analysis of the two-grid method (Sec. 3,
 * symbols PAPER.md:273-334; NEXT f4 alternative in SURVEY.md 8(f)): for the 2D Q1
 * operator with lambda = k^2 + i beta k^sigma (readings C1, C2), the 4 x 4 symbol
 *   T(theta) = S^nu2 (I - P L_2h^{-1} R L_h) S^nu1        (R = P^T / 4)
 * on the harmonics of theta, and
 *   rho_loc = max over the m x m grid theta_i = -pi/2 + pi (i + 1) / m of
 *             T^low = (-pi/2, pi/2]^2, theta != 0, of the spectral radius of T
 * (the sup over the continuum is read as this grid maximum).
 * Eigenvalues: T = D - a b^T (diagonal minus rank one) has the characteristic
 * polynomial prod(x - d_i) + sum_i a_i b_i prod_{j!=i}(x - d_j); its four roots
 * are found by Aberth iterations in fp64 (root accuracy ~1e-8 near double roots).
 * q: HOST array of n queries; rho_out: HOST array of n doubles.  device: CUDA
 * ordinal; the call blocks.  HH_E_ARG: NULL pointer; HH_E_CONFIG: m < 2 or
 * > 4096, nu1/nu2 < 0, h <= 0, omega not in (0, 1]. */
typedef struct {
  double  k, h, beta, sigma, omega;
  int32_t nu1, nu2, m;
  int32_t pad;
} hh_lfa_query;
hh_status hh_lfa_rho(const hh_lfa_query* q, int32_t n, int32_t device, double* rho_out);

/* sigma_c = the smallest sigma in [sigma_lo, sigma_hi] with rho_loc(sigma) < 1
 * (I_conv = [sigma_c, 2], reading G2): bisection to width tol
 * assuming rho_loc decreases in sigma (a stronger shift damps more), every round
 * one batched rho_loc evaluation of all queries (q[i].sigma ignored).
 * sigma_c_out[i] = sigma_lo if rho_loc(sigma_lo) < 1, NaN if rho_loc(sigma_hi) >= 1,
 * else the upper end of the final bracket.  HOST arrays; blocks. */
hh_status hh_lfa_sigma_c(const hh_lfa_query* q, int32_t n, int32_t device, double sigma_lo,
                         double sigma_hi, double tol, double* sigma_c_out);

/* LFA instrumentation since the last reset: st4 = [theta points evaluated,
 * Aberth iterations, device ms of the rho_loc kernels (CUDA events), kernel
 * launches]; reset != 0 zeroes them after reading.  st4 may be NULL. */
hh_status hh_lfa_stats(int32_t reset, double* st4);

hh_status hh_destroy_problem(hh_problem* p);

/* Phase instrumentation for the bench roofline (device events around each
 * phase of sampled FGMRES iterations; enabling it adds host syncs).
 * st24 (24 doubles, caller-owned HOST array) = [ms x4, compulsory HBM bytes x4,
 * phase launches x4, compulsory HBM bytes of EVERY iteration x4, SURVEY 8(d)
 * model bytes x4, model bytes of EVERY iteration x4] (ms, bytes, launches,
 * model over the timed, i.e. sampled, iterations) for the phases
 * [pre-smooth+restrict, coarse solve, prolong+post-smooth+A_0, Krylov
 * (multi-dot + update)], accumulated since the last reset.  "Compulsory" = each
 * fused kernel reads its inputs and writes its outputs once; "model" = every
 * Jacobi step / transfer / apply as its own pass. */
hh_status hh_reset_timers(hh_problem* p, int32_t enable);
hh_status hh_read_timers(hh_problem* p, double* st24, int64_t* launches);

/* Sweep-wide phase instrumentation (same st24 layout as hh_read_timers) and
 * kernel-launch count since the last reset; reset_enable >= 0 resets and sets
 * timing on (1) / off (0); -1 only reads. */
hh_status hh_sweep_timers(int32_t reset_enable, double* st24, int64_t* launches);

/* The coarse solver a handle actually uses (HH_COARSE_ND / _ND_DIST / _FD; AUTO
 * resolved, including FD's fallback to ND when its eigen-decomposition fails
 * validation).  kind: out.                                                     */
hh_status hh_coarse_kind(const hh_problem* p, int32_t* kind);

/* Coarse-solve flops since the last timer reset (hh_reset_timers / hh_sweep_timers):
 * flops2 = [flops of the timed (sampled) iterations, flops of every iteration]
 * (real flops of the fast-diagonalisation GEMMs, 8 per complex multiply-add;
 * 0 for the ND factor, whose roofline is bytes).  p = NULL: the sweep's.       */
hh_status hh_coarse_flops(hh_problem* p, double* flops2);

/* FP64 FMA throughput of the device (microbenchmark: independent DFMA chains on
 * every SM, best of 5 timed launches, 2 flops per DFMA): the measured peak the
 * coarse factorisation's TFLOP/s are quoted against.
 * tflops: out; sm_mhz: out (nullable), the device's nominal SM clock.  blocks. */
hh_status hh_fp64_peak(int32_t device, double* tflops, double* sm_mhz);

/* FP64 tensor-core throughput (microbenchmark: independent mma.sync m8n8k4 f64
 * accumulators on every SM, best of 5, 512 flops per MMA): the denominator of
 * the fast-diagonalisation coarse solve's TFLOP/s (its GEMMs run on this
 * instruction).  tflops: out.  Blocks.                                        */
hh_status hh_fp64_mma_peak(int32_t device, double* tflops);

const char* hh_last_error(void);
const char* hh_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HH_H_ */
