// Coarse-grid direct solver for A_eps^{(1)} (Alg. 1 line 3, PAPER.md:374;
// factor once, reuse every V-cycle: PAPER.md:511-512).
//
// B200 design (differs from the paper's MUMPS LU):
//  * geometric nested dissection of the structured (m)^d coarse node grid:
//    recursive bisection of boxes by a separator line/plane; leaves <= 64 nodes.
//    Front(t) = sep(t) (eliminated at t) + halo(t) (1-ring of box(t), clipped).
//  * multifrontal elimination WITHOUT pivoting (reading C18: the Hermitian part
//    of i*A_eps is eps*M + k*B, positive definite for eps > 0, so every
//    principal submatrix is non-singular); all fronts of one tree level of all
//    B samples of a batch in one launch.  Each front is "swept" on its
//    separator block by partial Gauss-Jordan (block size 16, 32 on large fronts): afterwards the
//    dense front holds
//        [ X = F_ss^{-1}      H = F_ss^{-1} F_su ]
//        [ -H^T               S = F_uu - F_us X F_su ]
//    and S is extend-added into the parent front.
//  * solve = two sweeps of batched GEMVs over the stored blocks (explicit
//    inverses, no triangular recurrences):
//        forward (leaves -> root):  z_s = r[sep] + sum of descendant contributions,
//                                   contribution_t = -H^T z_s  (gathered, no atomics)
//        backward (root -> leaves): x[sep] = X z_s - H x[halo]
//    Bytes streamed per solve ~ 16 * sum_t (s_t f_t + u_t s_t), the same as a
//    triangular LDL^T solve; every launch is fully parallel.
// The tree (NDPlan) depends only on (dim, m) and is shared by all samples.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <cooperative_groups.h>
#include "hh_internal.cuh"
#include "krylov.cuh"
namespace cg = cooperative_groups;

namespace {
constexpr int PIV_CHUNK = 256;   // rows / columns per k_nd_piv CTA
constexpr int LEAF = 64;    // max nodes of a leaf box
#ifndef ND_PIV_REG
#define ND_PIV_REG 0   // 1: 16-pivot row scaling with the column in registers (120 registers; sweep 0.369 -> 0.379 s)
#endif
#ifndef ND_RB
#define ND_RB 2
#endif

struct FrontMeta {          // device-visible per-front data
  int s, u, f, level;
  int64_t Foff;             // offset (complex entries) of the f x f front
  int64_t sepOff, haloOff;  // into sep / halo index arrays
  int64_t posOff, outOff;   // into the solve work vector: w (f entries) / update vector (u entries)
  int64_t eaOff;            // into extend-add map (u entries)
  int parent;
  int pad;
};

// lean storage (large 3D trees): a level is factored in chunks of fronts that
// fit a reusable workspace W; afterwards only the rows [X | H] (s x f) of every
// front are kept (the forward solve reads H transposed), the Schur complement S
// goes packed (lower triangle) into a per-level-parity buffer for the parent's
// extend-add, and W is reused by the next chunk.
struct Chunk {
  int level, t0, t1;
  int64_t Wcount;                    // workspace entries of the chunk
  int64_t asmBegin, asmCount;
  int ea_count[2];
  int64_t ea_list_off[2];            // children (by slot) of the chunk's fronts, in eaListC
};

struct LevelInfo {
  int begin, count;         // fronts [begin, begin+count)
  int max_s, max_u, max_f;
  int64_t asmBegin, asmCount;        // assembly entries
  int64_t Fbegin, Fcount;            // F entries of the level
  int ea_count[2];                   // children per slot
  int64_t ea_list_off[2];            // offsets into eaList
};
}  // namespace

// Solve schedule: levels <= sub_cut run as one-CTA subtree walks, levels
// (sub_cut, split] as per-level kernels, levels > split inside one cluster kernel.
// wide backward levels with fronts of order > this (HH_ND_BWDK_F) use the K-split rows
static int bwdk_f() {
  static const int v = getenv("HH_ND_BWDK_F") ? atoi(getenv("HH_ND_BWDK_F")) : 1024;
  return v;
}

struct SolveCfg { int sub_cut, split, flow = 0; };

struct NDPlan {
  int dim = 2, m = 0;            // coarse grid nodes per side
  int64_t N = 0;                 // coarse nodes
  int S = 9;                     // stencil entries per node
  std::vector<FrontMeta> fronts; // host copy
  std::vector<LevelInfo> levels;
  FrontMeta* d_fronts = nullptr;
  int* d_sep = nullptr;
  int* d_halo = nullptr;
  int4* d_asm = nullptr;         // (front, a, b, stencil index)
  int* d_eamap = nullptr;        // child halo pos -> parent front pos
  int* d_eaList = nullptr;       // child front ids grouped by (level, slot)
  int2* d_gmap = nullptr;        // per front position: update-vector entries of child 0 / 1 (-1: none)
  int64_t* d_Coff = nullptr;     // per front offset into the pivot column buffer (level-local)
  int64_t F_entries = 0, w_entries = 0, out_entries = 0, C_entries = 0;
  int64_t stream_bytes = 0;
  // bottom-subtree decompositions, one per candidate cut level L (fronts of level <= L)
  std::vector<int> sub_cnt;          // number of subtrees for cut L
  std::vector<int64_t> sub_off;      // offset of cut L's ptr array in d_sub_ptr
  std::vector<int64_t> list_off;     // offset of cut L's front list in d_sub_list
  std::vector<double> sub_cost_us;   // estimated cost of the slowest subtree (one CTA)
  std::vector<int> sub_maxf;
  int* d_sub_ptr = nullptr;
  int* d_sub_list = nullptr;
  // per-level entry ranges + entry -> front maps (cluster solve)
  std::vector<double> level_bytes;   // factor bytes streamed per level per sample
  int* d_sep_front = nullptr;
  int* d_halo_front = nullptr;
  int* d_pos_front = nullptr;
  int64_t* d_lvr = nullptr;          // [nlev][6]: sep begin/end, halo begin/end, position begin/end
  // dataflow solve
  int2* d_child = nullptr;           // per front: children (-1: none)
  int* d_lvbeg = nullptr;            // per level: first front
  std::mutex cut_mu;
  std::vector<std::pair<int, SolveCfg>> cfg_cache;   // (B, schedule) chosen by nd_autotune
  bool flow_disabled = false;                          // a dataflow solve failed (nd_flow_disable)
  // lean storage
  bool lean = false;
  std::vector<Chunk> chunks;
  FrontMeta* d_fronts_w = nullptr;   // Foff = chunk-relative workspace offset
  int64_t* d_Coff_w = nullptr;       // chunk-local pivot column buffer offsets
  int64_t* d_Soff = nullptr;         // packed S offset (in the level-parity buffer)
  int64_t* d_Poff = nullptr;         // forward partial-sum offset (level-local)
  int* d_eaListC = nullptr;
  int64_t Wmax = 0, Cw = 0, Smax[2] = {0, 0}, Pmax = 0;
  // K-split backward of long rows (3D): per front ceil(f / KC) x s partial sums
  int64_t Kmax = 0;
  int64_t* d_Koff = nullptr;
  // distributed (slab-aligned) plan: the view of rank `rank` of a P-rank tree
  // (nd_plan_create_dist).  Fronts are ordered by (level, owner), so `levels`
  // holds this rank's contiguous range of every level; the storage offsets
  // (Foff, Poff) cover its own fronts only, the work layout and the packed-S
  // offsets are global (identical on every rank: exchanged blocks land at the
  // same place on both sides).
  int P = 1, rank = 0;
  std::vector<int> owner;                 // per front
  std::vector<std::vector<int>> xcross;   // per level: fronts whose parent has another owner
  std::vector<std::vector<int>> xtop;     // per level: fronts spanning several ranks (interface planes)
  std::vector<int64_t> Soff_h;            // packed-S offsets (host copy)
  int64_t top_sep_max = 0;                // largest sum of top-front separators of one level
};

// ============================================================ device kernels
namespace {

__global__ void k_nd_zero(cplx* __restrict__ F, int64_t FE, int64_t begin, int64_t count) {
  cplx* p = F + (int64_t)blockIdx.y * FE + begin;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = cmake(0, 0);
}

__global__ void k_nd_assemble(const int4* __restrict__ e, int64_t cnt,
                              const FrontMeta* __restrict__ fr, const cplx* __restrict__ st,
                              int64_t stS, cplx* __restrict__ F, int64_t FE) {
  const int b = blockIdx.y;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  const int4 v = e[i];
  const FrontMeta m = fr[v.x];
  F[(int64_t)b * FE + m.Foff + (int64_t)v.y * m.f + v.z] = st[(int64_t)b * stS + v.w];
}

// extend-add of the child update matrices S_c into the parents (one child per parent per launch)
__global__ void k_nd_extend_add(const int* __restrict__ list, const FrontMeta* __restrict__ fr,
                                const int* __restrict__ eamap, cplx* __restrict__ Fall,
                                int64_t FE) {
  cplx* F = Fall + (int64_t)blockIdx.z * FE;
  const int c = list[blockIdx.x];
  const FrontMeta mc = fr[c];
  const FrontMeta mp = fr[mc.parent];
  const int* map = eamap + mc.eaOff;
  for (int a = blockIdx.y; a < mc.u; a += gridDim.y) {
    const cplx* src = F + mc.Foff + (int64_t)(mc.s + a) * mc.f + mc.s;
    cplx* dst = F + mp.Foff + (int64_t)map[a] * mp.f;
    for (int b = threadIdx.x; b < mc.u; b += blockDim.x) {
      const cplx v = src[b];
      cplx& d = dst[map[b]];
      d.x += v.x;
      d.y += v.y;
    }
  }
}

// pivot step: P = F[K,K]^{-1}; save column block C = F[:,K]; rows K <- P F[K,:], F[K,K] <- P
// NBT = pivot block (16, or 32 on large fronts: half the passes over the front)
template <int NBT>
__global__ void __launch_bounds__(256) k_nd_piv(const FrontMeta* __restrict__ fr, int begin,
                                                int kb, cplx* __restrict__ Fall, int64_t FE,
                                                cplx* __restrict__ Call, int64_t CE,
                                                const int64_t* __restrict__ Coff,
                                                int* __restrict__ flag) {
  const int t = begin + blockIdx.x;
  const int b = blockIdx.y;
  const FrontMeta m = fr[t];
  if (kb >= m.s) return;
  const int nb = min(NBT, m.s - kb);
  const int f = m.f;
  // chunk blockIdx.z of PIV_CHUNK rows (column-block save) / columns (row scaling)
  const int c0 = blockIdx.z * PIV_CHUNK, c1 = min(f, c0 + PIV_CHUNK);
  if (c0 >= f) return;
  cplx* A = Fall + (int64_t)b * FE + m.Foff;
  cplx* C = Call + (int64_t)b * CE + Coff[blockIdx.x];
  cplx* Pg = C + (int64_t)f * NBT;   // P for k_nd_upd (the pivot block itself is rewritten there)
  // shared memory (dynamic): P [NBT][NBT + 1], rp, cp [NBT], and for NBT > 16 colS [NBT][32]
  extern __shared__ double4 smem_raw[];
  cplx (*P)[NBT + 1] = reinterpret_cast<cplx (*)[NBT + 1]>(smem_raw);
  cplx* rp = reinterpret_cast<cplx*>(smem_raw) + NBT * (NBT + 1);
  cplx* cp = rp + NBT;
  for (int e = threadIdx.x; e < NBT * NBT; e += 256) {
    const int ti = e / NBT, tj = e % NBT;
    if (ti < nb && tj < nb) P[ti][tj] = A[(int64_t)(kb + ti) * f + kb + tj];
  }
  // save this chunk's rows of the column block (rows outside K only are used later)
  for (int i = c0 + threadIdx.x / NBT; i < c1; i += 256 / NBT) {
    const int k = threadIdx.x % NBT;
    if (k < nb) C[(int64_t)i * NBT + k] = A[(int64_t)i * f + kb + k];
  }
  __syncthreads();
  // in-place Gauss-Jordan inversion of the nb x nb pivot block (sweep operator):
  // row p scaled by 1/P[p][p], column p -> -P[i][p]/P[p][p], the rest
  // P[i][j] -= P[i][p] * (scaled row p)[j], P[p][p] -> 1/P[p][p]
  for (int p = 0; p < nb; ++p) {
    const cplx piv = P[p][p];
    if (cabs2(piv) == 0.0 && threadIdx.x == 0) atomicExch(flag + b, 1);
    const cplx pinv = cinv(piv);
    if (threadIdx.x < nb) {
      const int q = threadIdx.x;
      rp[q] = q == p ? pinv : cmul(P[p][q], pinv);
      cp[q] = P[q][p];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < NBT * NBT; e += 256) {
      const int i = e / NBT, j = e % NBT;
      if (i >= nb || j >= nb) continue;
      if (i == p) {
        P[p][j] = rp[j];
      } else if (j == p) {
        const cplx v = cmul(cp[i], pinv);
        P[i][p] = cmake(-v.x, -v.y);
      } else {
        cplx v = P[i][j];
        cfms(v, cp[i], rp[j]);
        P[i][j] = v;
      }
    }
    __syncthreads();
  }
  if (blockIdx.z == 0)
    for (int e = threadIdx.x; e < NBT * NBT; e += 256) {
      const int ti = e / NBT, tj = e % NBT;
      Pg[e] = (ti < nb && tj < nb) ? P[ti][tj] : cmake(0, 0);
    }
  // rows K of this chunk's columns: R[k][j] = sum_l P[k][l] A[kb+l][j] for j not in K
  // (F[K,K] = P is written by k_nd_upd: the pivot block is read by every chunk here)
  if constexpr (NBT == 16 && ND_PIV_REG) {
    for (int j = c0 + threadIdx.x; j < c1; j += blockDim.x) {
      if (j >= kb && j < kb + nb) continue;
      cplx col[NBT];
#pragma unroll
      for (int l = 0; l < NBT; ++l) col[l] = (l < nb) ? A[(int64_t)(kb + l) * f + j] : cmake(0, 0);
#pragma unroll
      for (int k = 0; k < NBT; ++k) {
        if (k >= nb) break;
        cplx acc = cmake(0, 0);
#pragma unroll
        for (int l = 0; l < NBT; ++l)
          if (l < nb) cfma(acc, P[k][l], col[l]);
        A[(int64_t)(kb + k) * f + j] = acc;
      }
    }
  } else {   // 32 columns at a time through shared memory (32 column values per thread would spill)
    cplx (*colS)[32] = reinterpret_cast<cplx (*)[32]>(cp + NBT);
    for (int js = c0; js < c1; js += 32) {
      for (int e = threadIdx.x; e < NBT * 32; e += 256) {
        const int l = e / 32, jj = e % 32;
        colS[l][jj] = (l < nb && js + jj < c1) ? A[(int64_t)(kb + l) * f + js + jj] : cmake(0, 0);
      }
      __syncthreads();
      for (int e = threadIdx.x; e < NBT * 32; e += 256) {
        const int k = e / 32, jj = e % 32, j = js + jj;
        if (k >= nb || j >= c1 || (j >= kb && j < kb + nb)) continue;
        cplx acc = cmake(0, 0);
        for (int l = 0; l < nb; ++l) cfma(acc, P[k][l], colS[l][jj]);
        A[(int64_t)(kb + k) * f + j] = acc;
      }
      __syncthreads();
    }
  }
}

// rank-nb update of all rows outside K:
//   F[i][j] <- (j in K ? 0 : F[i][j]) - sum_k C[i][k] * F[kb+k][j]
constexpr int UT = 32;   // update tile columns (UR x UT outputs per CTA, 256 threads)
constexpr int NB_MAX = 32;   // C-buffer layout allows pivot blocks up to this size (64 needs NB_MAX = 64; measured slower, also with DMMA)
// update tile rows UR (UR / 8 rows per thread): 64 for fronts of order >= 1024
// (more multiply-adds per shared-memory read; 3 CTAs per SM), 32 below (more CTAs
// for the many small fronts)
template <int UR, int NBT>
__global__ void __launch_bounds__(256, UR == 64 ? (NBT == 64 ? 2 : 3) : 5) k_nd_upd(const FrontMeta* __restrict__ fr, int begin,
                                                int kb, int tiles, cplx* __restrict__ Fall,
                                                int64_t FE, const cplx* __restrict__ Call,
                                                int64_t CE, const int64_t* __restrict__ Coff) {
  const int t = begin + blockIdx.y;
  const int b = blockIdx.z;
  const FrontMeta m = fr[t];
  if (kb >= m.s) return;
  const int f = m.f;
  const int i0 = (blockIdx.x / tiles) * UR, j0 = (blockIdx.x % tiles) * UT;   // tiles = column tiles
  if (i0 >= f || j0 >= f) return;
  const int nb = min(NBT, m.s - kb);
  cplx* A = Fall + (int64_t)b * FE + m.Foff;
  const cplx* C = Call + (int64_t)b * CE + Coff[blockIdx.y];
  const cplx* Pg = C + (int64_t)f * NBT;
  // unpadded: C is read as warp broadcasts, R rows and both fills are contiguous
  extern __shared__ double4 smem_raw[];   // Cs [UR][NBT], Rs [NBT][UT]
  cplx (*Cs)[NBT] = reinterpret_cast<cplx (*)[NBT]>(smem_raw);
  cplx (*Rs)[UT] = reinterpret_cast<cplx (*)[UT]>(reinterpret_cast<cplx*>(smem_raw) + UR * NBT);
  for (int idx = threadIdx.x; idx < UR * NBT; idx += 256) {
    const int i = idx / NBT, k = idx % NBT;
    Cs[i][k] = (i0 + i < f && k < nb) ? C[(int64_t)(i0 + i) * NBT + k] : cmake(0, 0);
  }
  for (int idx = threadIdx.x; idx < NBT * UT; idx += 256) {
    const int k = idx / UT, j = idx % UT;
    const int jj = j0 + j;
    cplx r = cmake(0, 0);
    if (k < nb && jj < f) r = (jj >= kb && jj < kb + nb) ? Pg[k * NBT + (jj - kb)] : A[(int64_t)(kb + k) * f + jj];
    Rs[k][j] = r;
  }
  __syncthreads();
  const int tx = threadIdx.x % UT, ty = threadIdx.x / UT;   // 32 x 8
  const int j = j0 + tx;
  if (j >= f) return;
  const bool jK = (j >= kb && j < kb + nb);
  // the thread's UR/8 rows at once, k outermost: every R value read from shared
  // memory feeds UR/8 multiply-adds (the C values are warp broadcasts), so the
  // update is FP64-bound instead of shared-memory bound; per output the k order
  // (and so the rounding) is unchanged
  constexpr int RPT = UR / 8;
  cplx acc[RPT];
  bool upd[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = i0 + ty + 8 * r;
    upd[r] = i < f && !(i >= kb && i < kb + nb);
    acc[r] = (upd[r] && !jK) ? A[(int64_t)i * f + j] : cmake(0, 0);
  }
#pragma unroll
  for (int k = 0; k < NBT; ++k) {
    const cplx rv = Rs[k][tx];
#pragma unroll
    for (int r = 0; r < RPT; ++r) cfms(acc[r], Cs[ty + 8 * r][k], rv);
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = i0 + ty + 8 * r;
    if (i >= f) continue;
    if (upd[r]) A[(int64_t)i * f + j] = acc[r];
    else if (jK) A[(int64_t)i * f + j] = Pg[(i - kb) * NBT + (j - kb)];   // rows K: F[K,K] = P
  }
}

// The same rank-nb update on the FP64 tensor path (mma.sync m8n8k4 f64, DMMA):
// the CTA's 64 x 32 complex tile is split over 8 warps as 16 x 16 complex warp
// tiles, i.e. 2 x 2 blocks of 8 x 8 real and imaginary accumulators; per k step
// of 4 the complex product takes four real MMAs (Re -= Cr Rr - Ci Ri, Im -= Cr Ri +
// Ci Rr).  Same inputs / outputs / special cases as k_nd_upd<64, NBT>; only the
// summation order inside the MMA differs.  (Measured on this B200: DMMA 37.2
// TFLOP/s, DFMA chains 36.3: the win is fewer issued instructions and
// shared-memory reads per multiply-add, not a higher peak.)
constexpr int MU_C = 32;
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// UR = 64: 4 x 2 warps of 16 x 16 complex; UR = 32: 2 x 4 warps of 16 x 8 complex
template <int UR, int NBT>
__global__ void __launch_bounds__(256, UR == 64 ? 3 : 4) k_nd_upd_mma(const FrontMeta* __restrict__ fr, int begin, int kb, int tiles,
                                                     cplx* __restrict__ Fall, int64_t FE, const cplx* __restrict__ Call,
                                                     int64_t CE, const int64_t* __restrict__ Coff) {
  const int t = begin + blockIdx.y;
  const int b = blockIdx.z;
  const FrontMeta m = fr[t];
  if (kb >= m.s) return;
  const int f = m.f;
  constexpr int MU_R = UR, WC = 8 / (UR / 16), CBN = MU_C / WC / 8;   // warp grid, 8-col blocks per warp
  const int i0 = (blockIdx.x / tiles) * MU_R, j0 = (blockIdx.x % tiles) * MU_C;
  if (i0 >= f || j0 >= f) return;
  const int nb = min(NBT, m.s - kb);
  cplx* A = Fall + (int64_t)b * FE + m.Foff;
  const cplx* C = Call + (int64_t)b * CE + Coff[blockIdx.y];
  const cplx* Pg = C + (int64_t)f * NBT;
  constexpr int CSX = NBT + 1, RSX = MU_C + 1;   // padded strides
  extern __shared__ double4 smem_raw[];
  cplx* Cs = reinterpret_cast<cplx*>(smem_raw);   // [MU_R][CSX]
  cplx* Rs = Cs + MU_R * CSX;                     // [NBT][RSX]
  for (int idx = threadIdx.x; idx < MU_R * NBT; idx += 256) {
    const int i = idx / NBT, k = idx % NBT;
    Cs[i * CSX + k] = (i0 + i < f && k < nb) ? C[(int64_t)(i0 + i) * NBT + k] : cmake(0, 0);
  }
  for (int idx = threadIdx.x; idx < NBT * MU_C; idx += 256) {
    const int k = idx / MU_C, j = idx % MU_C;
    const int jj = j0 + j;
    cplx r = cmake(0, 0);
    if (k < nb && jj < f) r = (jj >= kb && jj < kb + nb) ? Pg[k * NBT + (jj - kb)] : A[(int64_t)(kb + k) * f + jj];
    Rs[k * RSX + j] = r;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = warp / WC, wc = warp % WC, g = lane >> 2, q = lane & 3;
  const int wcol = wc * (MU_C / WC);
  double re[2][CBN][2], im[2][CBN][2];
#pragma unroll
  for (int rb = 0; rb < 2; ++rb) {
    const int i = i0 + wr * 16 + rb * 8 + g;
    const bool upd = i < f && !(i >= kb && i < kb + nb);
#pragma unroll
    for (int cb = 0; cb < CBN; ++cb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = j0 + wcol + cb * 8 + 2 * q + e;
        const bool jK = j >= kb && j < kb + nb;
        cplx v = cmake(0, 0);
        if (upd && j < f && !jK) v = A[(int64_t)i * f + j];
        re[rb][cb][e] = v.x;
        im[rb][cb][e] = v.y;
      }
  }
#pragma unroll
  for (int ks = 0; ks < NBT / 4; ++ks) {
    const int k = ks * 4 + q;
    cplx av[2], bv[CBN];
#pragma unroll
    for (int rb = 0; rb < 2; ++rb) av[rb] = Cs[(wr * 16 + rb * 8 + g) * CSX + k];
#pragma unroll
    for (int cb = 0; cb < CBN; ++cb) bv[cb] = Rs[k * RSX + wcol + cb * 8 + g];
#pragma unroll
    for (int rb = 0; rb < 2; ++rb)
#pragma unroll
      for (int cb = 0; cb < CBN; ++cb) {
        dmma884(re[rb][cb][0], re[rb][cb][1], -av[rb].x, bv[cb].x);   // Re -= Cr Rr
        dmma884(re[rb][cb][0], re[rb][cb][1], av[rb].y, bv[cb].y);    // Re += Ci Ri
        dmma884(im[rb][cb][0], im[rb][cb][1], -av[rb].x, bv[cb].y);   // Im -= Cr Ri
        dmma884(im[rb][cb][0], im[rb][cb][1], -av[rb].y, bv[cb].x);   // Im -= Ci Rr
      }
  }
#pragma unroll
  for (int rb = 0; rb < 2; ++rb) {
    const int i = i0 + wr * 16 + rb * 8 + g;
    if (i >= f) continue;
    const bool upd = !(i >= kb && i < kb + nb);
#pragma unroll
    for (int cb = 0; cb < CBN; ++cb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = j0 + wcol + cb * 8 + 2 * q + e;
        if (j >= f) continue;
        const bool jK = j >= kb && j < kb + nb;
        if (upd) A[(int64_t)i * f + j] = cmake(re[rb][cb][e], im[rb][cb][e]);
        else if (jK) A[(int64_t)i * f + j] = Pg[(i - kb) * NBT + (j - kb)];   // rows K: F[K,K] = P
      }
  }
}
template <int UR, int NBT>
constexpr size_t upd_mma_smem() { return (size_t)(UR * (NBT + 1) + NBT * (MU_C + 1)) * sizeof(cplx); }

// ------------------------------------------------------------ lean storage kernels
// extend-add of packed child Schur complements into the parents' workspace
__global__ void k_nd_ea_packed(const int* __restrict__ list, const FrontMeta* __restrict__ frw,
                               const int64_t* __restrict__ Soff, const cplx* __restrict__ Sprev,
                               const int* __restrict__ eamap, cplx* __restrict__ W) {
  const int c = list[blockIdx.x];
  const FrontMeta mc = frw[c];
  const FrontMeta mp = frw[mc.parent];
  const int* map = eamap + mc.eaOff;
  const cplx* S = Sprev + Soff[c];
  for (int a = blockIdx.y; a < mc.u; a += gridDim.y) {
    cplx* dst = W + mp.Foff + (int64_t)map[a] * mp.f;
    for (int b = threadIdx.x; b < mc.u; b += blockDim.x) {
      const int hi = max(a, b), lo = min(a, b);
      const cplx v = S[(int64_t)hi * (hi + 1) / 2 + lo];
      cplx& d = dst[map[b]];
      d.x += v.x;
      d.y += v.y;
    }
  }
}

// copy out of a factored chunk: rows [X | H] -> the solve factor, S -> packed store
__global__ void k_nd_copyout(const FrontMeta* __restrict__ frw, const FrontMeta* __restrict__ frx,
                             const int64_t* __restrict__ Soff, int t0, const cplx* __restrict__ W,
                             cplx* __restrict__ XH, cplx* __restrict__ Scur) {
  const int t = t0 + blockIdx.x;
  const FrontMeta mw = frw[t];
  const int s = mw.s, u = mw.u, f = mw.f;
  const cplx* src = W + mw.Foff;
  cplx* dst = XH + frx[t].Foff;
  const int64_t n1 = (int64_t)s * f;
  for (int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; i < n1; i += (int64_t)gridDim.y * blockDim.x)
    dst[i] = src[i];
  if (u == 0) return;
  cplx* S = Scur + Soff[t];
  const int64_t n2 = (int64_t)u * (u + 1) / 2;
  for (int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.y * blockDim.x) {
    // i = a (a + 1) / 2 + b, b <= a
    int a = (int)((sqrt(8.0 * (double)i + 1.0) - 1.0) * 0.5);
    while ((int64_t)(a + 1) * (a + 2) / 2 <= i) ++a;
    while ((int64_t)a * (a + 1) / 2 > i) --a;
    const int b = (int)(i - (int64_t)a * (a + 1) / 2);
    S[i] = src[(int64_t)(s + a) * f + s + b];
  }
}

// ------------------------------------------------------------------ solve
// Multifrontal solve with the stored blocks.  Front t owns the work vector
// w_t (f entries: separator part z_s, halo part) and an update vector upd_t
// (u entries) for its parent:
//   forward  (leaves -> root):  w_t = [r[sep]; 0] + extend-add of upd_c of its (<= 2)
//                               children;  upd_t = w_t[halo] - H^T z_s
//   backward (root -> leaves):  x[sep] = X z_s - H x[halo]
// The gather of w_t reads at most two child entries per position (gmap), so
// every stage is one short dependent chain instead of a walk over all
// descendant contributions.
constexpr int VMAX = 4096;   // front vectors up to this length are staged in shared memory
int nd_vmax() {              // HH_ND_VMAX lowers it (tests of the global-memory path on small grids)
  static const int v = getenv("HH_ND_VMAX") ? std::min(VMAX, atoi(getenv("HH_ND_VMAX"))) : VMAX;
  return v;
}

__device__ __forceinline__ cplx warp_sum(cplx v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// lane-strided dot of a front row with v: 4 independent (predicated) loads in
// flight per lane for every 128 entries -- no serial tail loop, so short rows
// (the 36..100-entry rows of the leaves) cost one load round trip
__device__ __forceinline__ cplx row_dot(const cplx* __restrict__ row, const cplx* v, int len, int lane) {
  cplx a0 = cmake(0, 0), a1 = cmake(0, 0), a2 = cmake(0, 0), a3 = cmake(0, 0);
  for (int c = lane; c < len; c += 128) {
    const bool p1 = c + 32 < len, p2 = c + 64 < len, p3 = c + 96 < len;
    const cplx r0 = __ldg(&row[c]);
    const cplx r1 = p1 ? __ldg(&row[c + 32]) : cmake(0, 0);
    const cplx r2 = p2 ? __ldg(&row[c + 64]) : cmake(0, 0);
    const cplx r3 = p3 ? __ldg(&row[c + 96]) : cmake(0, 0);
    cfma(a0, r0, v[c]);
    if (p1) cfma(a1, r1, v[c + 32]);
    if (p2) cfma(a2, r2, v[c + 64]);
    if (p3) cfma(a3, r3, v[c + 96]);
  }
  return warp_sum(cadd(cadd(a0, a1), cadd(a2, a3)));
}

// dot of one row with v by a group of G lanes (G = 32, 16, 8, 4), 4 predicated
// loads in flight per lane; the group sum is left in every lane of the group
template <int G, int DEPTH = 4>
__device__ __forceinline__ cplx row_dot_g(const cplx* __restrict__ row, const cplx* v, int len, int sub) {
  cplx a0 = cmake(0, 0), a1 = cmake(0, 0);
  for (int c = sub; c < len; c += DEPTH * G) {
    cplx r[DEPTH];
#pragma unroll
    for (int t = 0; t < DEPTH; ++t) r[t] = (c + G * t < len) ? __ldg(&row[c + G * t]) : cmake(0, 0);
#pragma unroll
    for (int t = 0; t < DEPTH; ++t)
      if (c + G * t < len) cfma(t & 1 ? a1 : a0, r[t], v[c + G * t]);
  }
  cplx a = cadd(a0, a1);
#pragma unroll
  for (int o = G / 2; o; o >>= 1) {
    a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
    a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
  }
  return a;
}

// lanes per row for rows of length len (4 loads per lane at most, 16 B each)
__host__ __device__ inline int wide_group(int len) { return len > 64 ? 32 : (len > 32 ? 16 : (len > 16 ? 8 : 4)); }

struct SolveArgs {
  const FrontMeta* fr;
  const int* st;
  const int* sep;
  const int* halo;
  const int2* gmap;
  const cplx* F; int64_t FE;
  cplx* work; int64_t WE, updE;   // work[b] = [w (w_entries) | upd (out_entries)]
  VArg rhs, x;
  int vmax;                        // fronts with f <= vmax stage their vectors in shared memory
  int prefetch;                    // L2 bulk prefetch of the factor rows before the PDL wait
  int* fail;                       // dataflow failure flag when st == nullptr (see nd_solve)
};

// Programmatic dependent launch: a level kernel may start while its predecessor
// drains; before griddepcontrol.wait it touches only the (immutable) factor,
// which it prefetches into L2 with bulk prefetches, so the factor stream of
// level L+1 overlaps the tail of level L.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p, int bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// prefetch the rows r0, r0 + step, ... (< nrows, at most 8 per warp) of length len starting at
// row0; one bulk prefetch per <= 32 KB piece
__device__ __forceinline__ void prefetch_rows(const cplx* row0, int64_t ld, int len, int nrows, int r0,
                                              int step, int lane) {
  if (len <= 0) return;
  const int r = r0 + lane * step;
  if (lane < 8 && r < nrows) {
    const char* p = reinterpret_cast<const char*>(row0 + (int64_t)r * ld);
    for (int64_t left = (int64_t)len * (int64_t)sizeof(cplx); left > 0; left -= 32768, p += 32768)
      prefetch_l2(p, (int)(left < 32768 ? left : 32768));
  }
}

__device__ __forceinline__ cplx* w_of(const SolveArgs& A, int b) { return A.work + (int64_t)b * A.WE; }
__device__ __forceinline__ cplx* upd_of(const SolveArgs& A, int b) { return A.work + (int64_t)b * A.WE + A.updE; }

// w_t[p] for p = p0, p0 + stride, ... -> dst (smem, may be NULL) and wg (global, sep part or all)
__device__ __forceinline__ void front_gather(const SolveArgs& A, const FrontMeta& m, int b, cplx* dst,
                                             cplx* wg, int wg_len, int p0, int stride) {
  const cplx* r = A.rhs.at(b);
  const cplx* upd = upd_of(A, b);
  const int2* gm = A.gmap + m.posOff;
  const int* sp = A.sep + m.sepOff;
  for (int p = p0; p < m.f; p += stride) {
    const int2 g = __ldg(&gm[p]);
    cplx v = p < m.s ? __ldg(&r[__ldg(&sp[p])]) : cmake(0, 0);
    if (g.x >= 0) v = cadd(v, upd[g.x]);
    if (g.y >= 0) v = cadd(v, upd[g.y]);
    if (dst) dst[p] = v;
    if (wg && p < wg_len) wg[p] = v;
  }
}

// Rows of one front, DIR 0 (forward): upd[r] = w[s + r] + (-H^T row r) . z_s
// (rows s + r of F, length s); DIR 1 (backward): x[sep[r]] = F[r][0:f] . v.
// Warp slots gw, gw + nw, ... each take 32 / G consecutive rows at once (G
// lanes per row, G from the row length), so the short rows of the low levels
// keep every lane loading instead of walking one row per warp round trip.
template <int DIR, int G>
__device__ __forceinline__ void front_rows_g(const SolveArgs& A, const FrontMeta& m, int bs, const cplx* v,
                                             int gw, int nw, int lane) {
  constexpr int RPW = 32 / G;   // row groups per warp
  constexpr int RB = ND_RB;     // rows per group and pass: their loads are in flight together
  constexpr int DEPTH = 4;
  const int rows = DIR == 0 ? m.u : m.s, len = DIR == 0 ? m.s : m.f;
  const cplx* F = A.F + (int64_t)bs * A.FE + m.Foff;
  const cplx* row0 = DIR == 0 ? F + (int64_t)m.s * m.f : F;
  const int grp = lane / G, sub = lane % G;
  for (int base = gw * RPW * RB; base < rows; base += nw * RPW * RB) {
    cplx a0[RB], a1[RB];
#pragma unroll
    for (int k = 0; k < RB; ++k) a0[k] = a1[k] = cmake(0, 0);
    for (int c = sub; c < len; c += DEPTH * G) {
      cplx x[RB][DEPTH];
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const int r = base + grp + k * RPW;
        const cplx* row = row0 + (int64_t)(r < rows ? r : 0) * m.f;
#pragma unroll
        for (int t = 0; t < DEPTH; ++t)
          x[k][t] = (r < rows && c + G * t < len) ? __ldg(&row[c + G * t]) : cmake(0, 0);
      }
#pragma unroll
      for (int t = 0; t < DEPTH; ++t) {
        if (c + G * t >= len) break;
        const cplx vt = v[c + G * t];
#pragma unroll
        for (int k = 0; k < RB; ++k) cfma(t & 1 ? a1[k] : a0[k], x[k][t], vt);
      }
    }
#pragma unroll
    for (int k = 0; k < RB; ++k) {
      cplx a = cadd(a0[k], a1[k]);
#pragma unroll
      for (int o = G / 2; o; o >>= 1) {
        a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
        a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
      }
      const int r = base + grp + k * RPW;
      if (r < rows && sub == 0) {
        if (DIR == 0) upd_of(A, bs)[m.outOff + r] = cadd(a, v[m.s + r]);
        else A.x.at(bs)[A.sep[m.sepOff + r]] = a;
      }
    }
  }
}
template <int DIR>
__device__ __forceinline__ void front_rows(const SolveArgs& A, const FrontMeta& m, int bs, const cplx* v,
                                           int gw, int nw, int lane) {
  switch (wide_group(DIR == 0 ? m.s : m.f)) {
    case 32: front_rows_g<DIR, 32>(A, m, bs, v, gw, nw, lane); break;
    case 16: front_rows_g<DIR, 16>(A, m, bs, v, gw, nw, lane); break;
    case 8: front_rows_g<DIR, 8>(A, m, bs, v, gw, nw, lane); break;
    default: front_rows_g<DIR, 4>(A, m, bs, v, gw, nw, lane); break;
  }
}
__device__ __forceinline__ void front_fwd_rows(const SolveArgs& A, const FrontMeta& m, int bs, const cplx* w,
                                               int gw, int nw, int lane) {
  front_rows<0>(A, m, bs, w, gw, nw, lane);
}
__device__ __forceinline__ void front_bwd_rows(const SolveArgs& A, const FrontMeta& m, int bs, const cplx* v,
                                               int gw, int nw, int lane) {
  front_rows<1>(A, m, bs, v, gw, nw, lane);
}

__device__ __forceinline__ void stage_bwd(const SolveArgs& A, const FrontMeta& m, int bs, cplx* v) {
  const cplx* zs = w_of(A, bs) + m.posOff;
  const cplx* x = A.x.at(bs);
  for (int c = threadIdx.x; c < m.f; c += blockDim.x) {
    if (c < m.s) v[c] = zs[c];
    else {
      const cplx t = x[__ldg(&A.halo[m.haloOff + c - m.s])];
      v[c] = cmake(-t.x, -t.y);
    }
  }
}

// large fronts only (f > VMAX): gather w_t to global (separate pass)
__global__ void k_nd_gather(SolveArgs A, int begin) {
  const int b = blockIdx.z;
  pdl_trigger();
  pdl_wait();
  if (A.st && A.st[b]) return;
  const FrontMeta m = A.fr[begin + blockIdx.x];
  front_gather(A, m, b, nullptr, w_of(A, b) + m.posOff, m.f, threadIdx.x + blockIdx.y * blockDim.x,
               blockDim.x * gridDim.y);
}

constexpr int LT = 128;   // threads of the per-level solve kernels (4 warps)

// one tree level, forward: gather w_t into smem, write z_s, update-vector rows
__global__ void __launch_bounds__(LT) k_nd_fwd(SolveArgs A, int begin) {
  extern __shared__ double4 smem_raw[];
  cplx* wsh = reinterpret_cast<cplx*>(smem_raw);
  const int b = blockIdx.z;
  const FrontMeta m = A.fr[begin + blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();
  if (A.prefetch && !(A.st && *(volatile const int*)&A.st[b]))   // (possibly stale) status: prefetch hint only
    prefetch_rows(A.F + (int64_t)b * A.FE + m.Foff + (int64_t)m.s * m.f, m.f, m.s, m.u,
                  blockIdx.y * (LT / 32) + warp, gridDim.y * (LT / 32), lane);
  pdl_wait();
  if (A.st && A.st[b]) return;
  const cplx* w;
  if (m.f <= A.vmax) {
    front_gather(A, m, b, wsh, blockIdx.y == 0 ? w_of(A, b) + m.posOff : nullptr, m.s, threadIdx.x,
                 blockDim.x);
    __syncthreads();
    w = wsh;
  } else {
    w = w_of(A, b) + m.posOff;   // gathered by k_nd_gather
  }
  front_fwd_rows(A, m, b, w, blockIdx.y * (LT / 32) + warp, gridDim.y * (LT / 32), lane);
}

// one tree level, backward
__global__ void __launch_bounds__(LT) k_nd_bwd(SolveArgs A, int begin) {
  extern __shared__ double4 smem_raw[];
  cplx* v = reinterpret_cast<cplx*>(smem_raw);
  const int b = blockIdx.z;
  const FrontMeta m = A.fr[begin + blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();
  if (A.prefetch && !(A.st && *(volatile const int*)&A.st[b]))
    prefetch_rows(A.F + (int64_t)b * A.FE + m.Foff, m.f, m.f, m.s, blockIdx.y * (LT / 32) + warp,
                  gridDim.y * (LT / 32), lane);
  pdl_wait();
  if (A.st && A.st[b]) return;
  if (m.f <= A.vmax) {
    stage_bwd(A, m, b, v);
    __syncthreads();
    front_bwd_rows(A, m, b, v, blockIdx.y * (LT / 32) + warp, gridDim.y * (LT / 32), lane);
  } else {   // huge fronts: v = [z_s ; -x[halo]] was staged in w (k_nd_bwd_stage)
    front_bwd_rows(A, m, b, w_of(A, b) + m.posOff, blockIdx.y * (LT / 32) + warp, gridDim.y * (LT / 32),
                   lane);
  }
}

// huge fronts (f > VMAX): stage -x[halo] into the halo part of w (the forward
// halo values are dead by now), so the backward rows are plain contiguous dots
__global__ void k_nd_bwd_stage(SolveArgs A, int begin) {
  const int b = blockIdx.z;
  pdl_trigger();
  pdl_wait();
  if (A.st && A.st[b]) return;
  const FrontMeta m = A.fr[begin + blockIdx.x];
  cplx* wv = w_of(A, b) + m.posOff + m.s;
  const cplx* x = A.x.at(b);
  for (int c = threadIdx.x + blockIdx.y * blockDim.x; c < m.u; c += blockDim.x * gridDim.y) {
    const cplx t = x[__ldg(&A.halo[m.haloOff + c])];
    wv[c] = cmake(-t.x, -t.y);
  }
}

// Wide levels (many rows per front): the front vector is gathered / staged once
// into global w (k_nd_gather / k_nd_bwd_stage), and the rows are spread over
// many CTAs (WIDE_RPC rows each) that copy only what they need (z_s forward,
// [z_s ; -x[halo]] backward) from L2 into shared memory -- instead of every CTA
// re-gathering the whole front, which capped the CTAs per front.
constexpr int WIDE_RPC = 8;   // rows per CTA for rows longer than 64 entries

template <int DIR, int G, int DEPTH = 4>
__device__ __forceinline__ void wide_rows(const SolveArgs& A, const FrontMeta& m, int b, const cplx* row0,
                                          const cplx* v, const cplx* wg, int len, int r0, int r1, int warp,
                                          int lane) {
  constexpr int RPW = 32 / G;                 // rows per warp pass
  const int grp = lane / G, sub = lane % G;
  for (int rb = r0 + warp * RPW; rb < r1; rb += (LT / 32) * RPW) {
    const int r = rb + grp;
    const bool ok = r < r1;
    const cplx acc = row_dot_g<G, DEPTH>(row0 + (int64_t)(ok ? r : r0) * m.f, v, ok ? len : 0, sub);
    if (ok && sub == 0) {
      if (DIR == 0) upd_of(A, b)[m.outOff + r] = cadd(acc, wg[m.s + r]);
      else A.x.at(b)[A.sep[m.sepOff + r]] = acc;
    }
  }
}

// rows per CTA of the wide kernels: 8 warp passes of 32 / G rows
__host__ __device__ inline int wide_rpc(int len) { return WIDE_RPC * (32 / wide_group(len)); }

template <int DIR>
__global__ void __launch_bounds__(LT) k_nd_rows_wide(SolveArgs A, int begin, int cap) {
  extern __shared__ double4 smem_raw[];
  cplx* vs = reinterpret_cast<cplx*>(smem_raw);
  const int b = blockIdx.z;
  const FrontMeta m = A.fr[begin + blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rows = DIR == 0 ? m.u : m.s;
  const int len = DIR == 0 ? m.s : m.f;
  const int rpc = wide_rpc(len);
  const int r0 = blockIdx.y * rpc;
  if (r0 >= rows) return;
  const int r1 = min(rows, r0 + rpc);
  const cplx* F = A.F + (int64_t)b * A.FE + m.Foff;
  const cplx* row0 = DIR == 0 ? F + (int64_t)m.s * m.f : F;
  pdl_trigger();
  if (A.prefetch && !(A.st && *(volatile const int*)&A.st[b]))
    prefetch_rows(row0, m.f, len, r1, r0 + warp, LT / 32, lane);
  pdl_wait();
  if (A.st && A.st[b]) return;
  const cplx* wg = w_of(A, b) + m.posOff;
  const cplx* v = wg;
  if (len <= cap) {                            // cap = shared-memory entries of this launch
    for (int c = threadIdx.x; c < len; c += blockDim.x) vs[c] = wg[c];
    __syncthreads();
    v = vs;
  }
  if (len > 1024) {   // long rows (3D top levels): 8 loads in flight per lane
    wide_rows<DIR, 32, 8>(A, m, b, row0, v, wg, len, r0, r1, warp, lane);
    return;
  }
  switch (wide_group(len)) {
    case 32: wide_rows<DIR, 32>(A, m, b, row0, v, wg, len, r0, r1, warp, lane); break;
    case 16: wide_rows<DIR, 16>(A, m, b, row0, v, wg, len, r0, r1, warp, lane); break;
    case 8: wide_rows<DIR, 8>(A, m, b, row0, v, wg, len, r0, r1, warp, lane); break;
    default: wide_rows<DIR, 4>(A, m, b, row0, v, wg, len, r0, r1, warp, lane); break;
  }
}

// Lean forward (no stored -H^T rows): upd[b] = w[s+b] - sum_a H[a][b] z[a] with
// H = rows [0, s) x columns [s, f) of [X | H]; CTAs take (128-column block, 256-row
// chunk) tiles, threads own one column (coalesced row reads, 8 rows in flight),
// and the row-chunk partials are summed in a fixed order by k_nd_fwdT_red.
constexpr int FT_COLS = 128, FT_ROWS = 256;
__global__ void __launch_bounds__(FT_COLS) k_nd_fwdT(SolveArgs A, int begin, const int64_t* __restrict__ Poff,
                                                     int ncb, int64_t PE) {
  __shared__ cplx zs[FT_ROWS];
  const int b = blockIdx.z;
  const int t = begin + blockIdx.y;
  const FrontMeta m = A.fr[t];
  const int cb = blockIdx.x % ncb, rc = blockIdx.x / ncb;
  const int a0 = rc * FT_ROWS;
  pdl_trigger();
  pdl_wait();
  if (A.st && A.st[b]) return;
  if (cb * FT_COLS >= m.u || a0 >= m.s) return;
  const int a1 = min(m.s, a0 + FT_ROWS);
  const cplx* w = w_of(A, b) + m.posOff;
  for (int i = threadIdx.x; i < a1 - a0; i += blockDim.x) zs[i] = w[a0 + i];
  __syncthreads();
  const int col = cb * FT_COLS + threadIdx.x;
  if (col >= m.u) return;
  const cplx* H = A.F + (int64_t)b * A.FE + m.Foff + m.s + col;   // H[a][col] at H + a * f
  cplx acc0 = cmake(0, 0), acc1 = cmake(0, 0);
  int a = a0;
  for (; a + 8 <= a1; a += 8) {
    cplx h[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) h[k] = __ldg(&H[(int64_t)(a + k) * m.f]);
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      cfma(acc0, h[k], zs[a + k - a0]);
      cfma(acc1, h[k + 1], zs[a + k + 1 - a0]);
    }
  }
  for (; a < a1; ++a) cfma(acc0, __ldg(&H[(int64_t)a * m.f]), zs[a - a0]);
  cplx* part = A.work + (int64_t)b * A.WE + PE + Poff[t];
  part[(int64_t)rc * m.u + col] = cadd(acc0, acc1);
}

__global__ void k_nd_fwdT_red(SolveArgs A, int begin, const int64_t* __restrict__ Poff, int64_t PE) {
  const int b = blockIdx.z;
  pdl_trigger();
  pdl_wait();
  if (A.st && A.st[b]) return;
  const int t = begin + blockIdx.y;
  const FrontMeta m = A.fr[t];
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= m.u) return;
  const int nrc = (m.s + FT_ROWS - 1) / FT_ROWS;
  const cplx* part = A.work + (int64_t)b * A.WE + PE + Poff[t];
  cplx sum = cmake(0, 0);
  for (int rc = 0; rc < nrc; ++rc) sum = cadd(sum, part[(int64_t)rc * m.u + col]);
  const cplx* w = w_of(A, b) + m.posOff;
  upd_of(A, b)[m.outOff + col] = csub(w[m.s + col], sum);
}

// K-split backward for long rows (3D levels with f > 1024): CTA = (32 rows,
// KC-column chunk); the chunk of v = [z_s ; -x[halo]] (staged in w) goes to shared
// memory, each warp dots 8 rows over it (8 loads in flight per lane); the chunk
// partials are summed in a fixed order by k_nd_bwdK_red.
constexpr int KC = 2048, KR = 32;
__global__ void __launch_bounds__(LT) k_nd_bwdK(SolveArgs A, int begin, int ncb, const int64_t* __restrict__ Koff,
                                                int64_t KE) {
  __shared__ cplx vs[KC];
  const int b = blockIdx.z;
  const FrontMeta m = A.fr[begin + blockIdx.y];
  const int rb = blockIdx.x / ncb, cb = blockIdx.x % ncb;
  const int r0 = rb * KR, c0 = cb * KC;
  pdl_trigger();
  pdl_wait();
  if (A.st && A.st[b]) return;
  if (r0 >= m.s || c0 >= m.f) return;
  const int r1 = min(m.s, r0 + KR), len = min(m.f - c0, KC);
  const cplx* wg = w_of(A, b) + m.posOff + c0;
  for (int c = threadIdx.x; c < len; c += blockDim.x) vs[c] = wg[c];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const cplx* F = A.F + (int64_t)b * A.FE + m.Foff + c0;
  cplx* part = A.work + (int64_t)b * A.WE + KE + Koff[begin + blockIdx.y] + (int64_t)cb * m.s;
  for (int r = r0 + warp; r < r1; r += LT / 32) {
    const cplx acc = row_dot_g<32, 8>(F + (int64_t)r * m.f, vs, len, lane);
    if (lane == 0) part[r] = acc;
  }
}

__global__ void k_nd_bwdK_red(SolveArgs A, int begin, const int64_t* __restrict__ Koff, int64_t KE) {
  const int b = blockIdx.z;
  pdl_trigger();
  pdl_wait();
  if (A.st && A.st[b]) return;
  const FrontMeta m = A.fr[begin + blockIdx.y];
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m.s) return;
  const int ncb = (m.f + KC - 1) / KC;
  const cplx* part = A.work + (int64_t)b * A.WE + KE + Koff[begin + blockIdx.y];
  cplx sum = cmake(0, 0);
  for (int cb = 0; cb < ncb; ++cb) sum = cadd(sum, part[(int64_t)cb * m.s + r]);
  A.x.at(b)[A.sep[m.sepOff + r]] = sum;
}

// ------------------------------------------------------------ cluster solve
// One thread-block cluster (CL CTAs on CL SMs) per sample walks the tree levels
// [L0, nlev): forward (gather, update rows) up to the root, then backward down
// to L0, with a cluster barrier between phases.  Operands go through L2/global
// memory; the barrier (release/acquire at cluster scope, preceded by a device
// fence) orders them.  This replaces ~3 launches per level.
__device__ __forceinline__ void cl_sync(cg::cluster_group& cl) {
  __threadfence();
  cl.sync();
}

__global__ void __launch_bounds__(256) k_nd_cluster(SolveArgs A, const int64_t* __restrict__ lvr,
                                                    int L0, int nlev, const int* __restrict__ sep_front,
                                                    const int* __restrict__ halo_front,
                                                    const int* __restrict__ pos_front) {
  cg::cluster_group cl = cg::this_cluster();
  const int CL = (int)cl.num_blocks();
  const int b = blockIdx.x / CL;
  if (A.st && A.st[b]) return;              // uniform over the cluster
  const int rank = (int)cl.block_rank();
  const int tid = rank * blockDim.x + threadIdx.x, nth = CL * blockDim.x;
  const int lane = threadIdx.x & 31, gw = tid >> 5, nw = nth >> 5;
  cplx* w = w_of(A, b);
  cplx* upd = upd_of(A, b);
  const cplx* r = A.rhs.at(b);
  cplx* x = A.x.at(b);
  const cplx* Fb = A.F + (int64_t)b * A.FE;
  for (int L = L0; L < nlev; ++L) {
    const int64_t hb = lvr[6 * L + 2], he = lvr[6 * L + 3], pb = lvr[6 * L + 4], pe = lvr[6 * L + 5];
    for (int64_t e = pb + tid; e < pe; e += nth) {        // gather w of every front of the level
      const FrontMeta m = A.fr[pos_front[e]];
      const int p = (int)(e - m.posOff);
      const int2 g = A.gmap[e];
      cplx v = p < m.s ? r[A.sep[m.sepOff + p]] : cmake(0, 0);
      if (g.x >= 0) v = cadd(v, upd[g.x]);
      if (g.y >= 0) v = cadd(v, upd[g.y]);
      w[e] = v;
    }
    cl_sync(cl);
    if (he > hb) {
      for (int64_t hrow = hb + gw; hrow < he; hrow += nw) {   // update rows
        const FrontMeta m = A.fr[halo_front[hrow]];
        const int brow = (int)(hrow - m.haloOff);
        const cplx acc = row_dot(Fb + m.Foff + (int64_t)(m.s + brow) * m.f, w + m.posOff, m.s, lane);
        if (lane == 0) upd[hrow] = cadd(acc, w[m.posOff + m.s + brow]);
      }
      cl_sync(cl);
    }
  }
  for (int L = nlev - 1; L >= L0; --L) {
    const int64_t sb = lvr[6 * L], se = lvr[6 * L + 1];
    for (int64_t e = sb + gw; e < se; e += nw) {
      const FrontMeta m = A.fr[sep_front[e]];
      const int a = (int)(e - m.sepOff);
      const cplx* row = Fb + m.Foff + (int64_t)a * m.f;
      cplx acc = row_dot(row, w + m.posOff, m.s, lane);
      cplx acc2 = cmake(0, 0);
      const int* hl = A.halo + m.haloOff;
      for (int c = lane; c < m.u; c += 32) cfms(acc2, __ldg(&row[m.s + c]), x[hl[c]]);
      acc = cadd(acc, warp_sum(acc2));
      if (lane == 0) x[A.sep[e]] = acc;
    }
    if (L > L0) cl_sync(cl);
  }
}

// ------------------------------------------------------------ dataflow solve
// The per-level kernels of levels (sub_cut, split] replaced by ONE forward and
// ONE backward kernel: a CTA (front t, sample b, row chunk c) starts as soon as
// the fronts it depends on are complete -- its children (forward) or its
// parent (backward) -- instead of waiting for a whole level and a launch.
// CTAs are numbered in dependency order (forward: levels bottom-up, backward:
// top-down), so every CTA a CTA waits for has a smaller index and was
// dispatched before it (the ordering decoupled look-back scans rely on).
// Completion: per (sample, front) counters in the work buffer, one atomic
// increment per finished CTA after a device fence; consumers poll with
// ld.acquire and read the producers' values through L2 (__ldcg).  The forward
// counters are cleared by the backward kernel and vice versa, so they are zero
// again at the start of every solve.  A wait that exceeds max_polls polls
// (~1 s by default; HH_ND_FLOW_POLLS) gives up and marks the SAMPLE failed:
// st[b] = HHK_NDFAIL (the FGMRES driver then reports an error for it, resets
// the counters and disables the schedule), or *fail when there is no status
// array (hh_vcycle / hh_coarse_solve check it before returning; the autotuner
// passes g_flow_timeout and rejects the schedule).  Later waits of the same
// sample see the mark and give up at once; other samples are not affected.
constexpr int FLOW_MAXL = 40;
struct FlowArgs {
  int L0, nl;                    // flow levels [L0, L0 + nl)
  int base[FLOW_MAXL + 1];       // CTA index ranges in launch order
  int lev[FLOW_MAXL];            // level offset of launch slot k
  int nch[FLOW_MAXL];            // CTAs per front of level offset j (this direction)
  int64_t cnt_off;               // counters: (int*)(work[b] + cnt_off) (complex entries), [2][nfronts]
  int nfr;
  unsigned max_polls;            // give up a dependency wait after this many polls
};
__device__ int g_flow_timeout = 0;

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void flow_wait(const int* c, int target, int* fail, int fail_code,
                                          unsigned max_polls) {
  if (target <= 0) return;
  if (max_polls == 0) { atomicExch(fail, fail_code); return; }   // HH_ND_FLOW_POLLS=0: fault injection (tests)
  unsigned polls = 0;
  while (ld_acquire(c) < target) {
    if (*(volatile int*)fail) break;                                     // this sample already failed
    if (++polls > max_polls) { atomicExch(fail, fail_code); break; }
    __nanosleep(64);
  }
}
// failure flag of sample b: its Krylov status, else the solve's flag
__device__ __forceinline__ int* flow_fail(const SolveArgs& A, int b, int& code) {
  if (A.st) { code = HHK_NDFAIL; return const_cast<int*>(A.st) + b; }
  code = 1;
  return A.fail ? A.fail : &g_flow_timeout;
}
__device__ __forceinline__ int* flow_cnt(const SolveArgs& A, const FlowArgs& W, int b) {
  return reinterpret_cast<int*>(A.work + (int64_t)b * A.WE + W.cnt_off);
}
// CTA index -> (level offset j, front t, sample b, chunk c)
__device__ __forceinline__ void flow_item(const FlowArgs& W, int B, int i, int& j, int& t, int& b, int& c) {
  int k = 0;
  while (k + 1 < W.nl && i >= W.base[k + 1]) ++k;
  j = W.lev[k];
  int rem = i - W.base[k];
  c = rem % W.nch[j];
  rem /= W.nch[j];
  b = rem % B;
  t = rem / B;
}

template <bool CG>
__device__ __forceinline__ cplx ld_v(const cplx* p) { return CG ? __ldcg(p) : *p; }

__global__ void __launch_bounds__(LT) k_nd_flow_fwd(SolveArgs A, FlowArgs W, const int* __restrict__ lvbeg,
                                                   const int2* __restrict__ child, int B) {
  extern __shared__ double4 smem_raw[];
  cplx* wsh = reinterpret_cast<cplx*>(smem_raw);
  int j, t, b, c;
  flow_item(W, B, blockIdx.x, j, t, b, c);
  t += lvbeg[W.L0 + j];
  const FrontMeta m = A.fr[t];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = W.nch[j];
  pdl_trigger();
  if (A.prefetch && !(A.st && *(volatile const int*)&A.st[b]))
    prefetch_rows(A.F + (int64_t)b * A.FE + m.Foff + (int64_t)m.s * m.f, m.f, m.s, m.u,
                  c * (LT / 32) + warp, nch * (LT / 32), lane);
  pdl_wait();
  if (A.st && A.st[b]) return;
  int* cnt = flow_cnt(A, W, b);
  if (threadIdx.x == 0) {
    if (c == 0) cnt[W.nfr + t] = 0;          // backward counter of t, for this solve's backward
    const int2 ch = child[t];
    for (int q = 0; q < 2; ++q) {
      const int cc = q ? ch.y : ch.x;
      if (cc < 0) continue;
      const int jc = A.fr[cc].level - W.L0;
      int code;
      int* fl = flow_fail(A, b, code);
      if (jc >= 0) flow_wait(cnt + cc, W.nch[jc], fl, code, W.max_polls);
    }
    __threadfence();
  }
  __syncthreads();
  {   // gather w_t (children's update vectors through L2)
    const cplx* r = A.rhs.at(b);
    const cplx* upd = upd_of(A, b);
    const int2* gm = A.gmap + m.posOff;
    const int* sp = A.sep + m.sepOff;
    cplx* wg = c == 0 ? w_of(A, b) + m.posOff : nullptr;
    for (int p = threadIdx.x; p < m.f; p += blockDim.x) {
      const int2 g = __ldg(&gm[p]);
      cplx v = p < m.s ? __ldg(&r[__ldg(&sp[p])]) : cmake(0, 0);
      if (g.x >= 0) v = cadd(v, __ldcg(&upd[g.x]));
      if (g.y >= 0) v = cadd(v, __ldcg(&upd[g.y]));
      wsh[p] = v;
      if (wg && p < m.s) wg[p] = v;
    }
  }
  __syncthreads();
  front_fwd_rows(A, m, b, wsh, c * (LT / 32) + warp, nch * (LT / 32), lane);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(cnt + t, 1);
  }
}

__global__ void __launch_bounds__(LT) k_nd_flow_bwd(SolveArgs A, FlowArgs W, const int* __restrict__ lvbeg,
                                                   int B) {
  extern __shared__ double4 smem_raw[];
  cplx* v = reinterpret_cast<cplx*>(smem_raw);
  int j, t, b, c;
  flow_item(W, B, blockIdx.x, j, t, b, c);
  t += lvbeg[W.L0 + j];
  const FrontMeta m = A.fr[t];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = W.nch[j];
  pdl_trigger();
  if (A.prefetch && !(A.st && *(volatile const int*)&A.st[b]))
    prefetch_rows(A.F + (int64_t)b * A.FE + m.Foff, m.f, m.f, m.s, c * (LT / 32) + warp, nch * (LT / 32), lane);
  pdl_wait();
  if (A.st && A.st[b]) return;
  int* cnt = flow_cnt(A, W, b);
  if (threadIdx.x == 0) {
    if (c == 0) cnt[t] = 0;                  // forward counter of t, for the next solve's forward
    if (m.parent >= 0) {
      const int jp = A.fr[m.parent].level - W.L0;
      int code;
      int* fl = flow_fail(A, b, code);
      if (jp < W.nl) flow_wait(cnt + W.nfr + m.parent, W.nch[jp], fl, code, W.max_polls);
    }
    __threadfence();
  }
  __syncthreads();
  {   // v = [z_s ; -x[halo]]  (halo values written by ancestors: through L2)
    const cplx* zs = w_of(A, b) + m.posOff;
    const cplx* x = A.x.at(b);
    for (int q = threadIdx.x; q < m.f; q += blockDim.x) {
      if (q < m.s) v[q] = zs[q];
      else {
        const cplx tv = __ldcg(&x[__ldg(&A.halo[m.haloOff + q - m.s])]);
        v[q] = cmake(-tv.x, -tv.y);
      }
    }
  }
  __syncthreads();
  front_bwd_rows(A, m, b, v, c * (LT / 32) + warp, nch * (LT / 32), lane);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(cnt + W.nfr + t, 1);
  }
}

// bottom subtrees: one CTA walks all fronts of one subtree (bottom-up / top-down)
__global__ void __launch_bounds__(256) k_nd_fwd_sub(SolveArgs A, const int* __restrict__ sub_ptr,
                                                    const int* __restrict__ sub_list) {
  extern __shared__ double4 smem_raw[];
  cplx* wsh = reinterpret_cast<cplx*>(smem_raw);
  const int b = blockIdx.y;
  if (A.st && A.st[b]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = sub_ptr[blockIdx.x]; k < sub_ptr[blockIdx.x + 1]; ++k) {
    const FrontMeta m = A.fr[sub_list[k]];
    front_gather(A, m, b, wsh, w_of(A, b) + m.posOff, m.s, threadIdx.x, blockDim.x);
    __syncthreads();
    front_fwd_rows(A, m, b, wsh, warp, 8, lane);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_nd_bwd_sub(SolveArgs A, const int* __restrict__ sub_ptr,
                                                    const int* __restrict__ sub_list) {
  extern __shared__ double4 smem_raw[];
  cplx* v = reinterpret_cast<cplx*>(smem_raw);
  const int b = blockIdx.y;
  if (A.st && A.st[b]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = sub_ptr[blockIdx.x + 1] - 1; k >= sub_ptr[blockIdx.x]; --k) {
    const FrontMeta m = A.fr[sub_list[k]];
    stage_bwd(A, m, b, v);
    __syncthreads();
    front_bwd_rows(A, m, b, v, warp, 8, lane);
    __syncthreads();
  }
}

// ============================================================ host plan
struct Box { int lo[3], hi[3]; };   // node index ranges [lo, hi)

struct HostFront {
  Box box;
  std::vector<int> sep, halo;
  int parent = -1;
  std::vector<int> children;
  int level = 0;
  int owner = 0;        // rank owning the front (distributed plans)
  bool top = false;     // interface-plane front of a distributed plan
};

int64_t box_count(const Box& b, int dim) {
  int64_t c = 1;
  for (int d = 0; d < dim; ++d) c *= (b.hi[d] - b.lo[d]);
  return c;
}

void push_box_nodes(const Box& b, int dim, int m, std::vector<int>& out) {
  int c[3] = {0, 0, 0};
  for (c[2] = (dim > 2 ? b.lo[2] : 0); c[2] < (dim > 2 ? b.hi[2] : 1); ++c[2])
    for (c[1] = b.lo[1]; c[1] < b.hi[1]; ++c[1])
      for (c[0] = b.lo[0]; c[0] < b.hi[0]; ++c[0]) {
        int64_t g = 0, st = 1;
        for (int d = 0; d < dim; ++d) { g += c[d] * st; st *= m; }
        out.push_back((int)g);
      }
}

void build_tree(const Box& b, int dim, int m, int parent, std::vector<HostFront>& out) {
  const int id = (int)out.size();
  out.push_back(HostFront());
  out[id].box = b;
  out[id].parent = parent;
  int ax = 0;
  for (int d = 1; d < dim; ++d)
    if (b.hi[d] - b.lo[d] > b.hi[ax] - b.lo[ax]) ax = d;
  const int ext = b.hi[ax] - b.lo[ax];
  static const int leaf = getenv("HH_ND_LEAF") ? atoi(getenv("HH_ND_LEAF")) : LEAF;
  if (box_count(b, dim) <= leaf || ext < 3) {   // leaf: all nodes, lexicographic
    push_box_nodes(b, dim, m, out[id].sep);
    return;
  }
  const int mid = (b.lo[ax] + b.hi[ax]) / 2;
  Box s = b; s.lo[ax] = mid; s.hi[ax] = mid + 1;
  push_box_nodes(s, dim, m, out[id].sep);
  Box l = b; l.hi[ax] = mid;
  Box r = b; r.lo[ax] = mid + 1;
  const int lid = (int)out.size();
  build_tree(l, dim, m, id, out);
  out[id].children.push_back(lid);
  const int rid = (int)out.size();
  build_tree(r, dim, m, id, out);
  out[id].children.push_back(rid);
}

// Slab-aligned nested dissection (distributed coarse solve, SURVEY.md 8(e)
// "second version" / 8(f) row 2): the coarse planes Zc[1..P-1] of the slowest
// axis (the slab boundaries of the fine decomposition, halved) are the top
// separators, taken middle-first over the chain of slabs [r0, r1), so the
// interface planes form a binary tree above the P slab interiors; each slab
// interior [Zc[r] + 1, Zc[r+1]) (rank 0: [0, Zc[1])) is an ordinary
// geometric ND subtree owned by rank r.  Interface plane Zc[k] is owned by rank
// k (the slab that restricts onto it: fine plane 2 Zc[k] belongs to slab k).
void build_tree_dist(const Box& b, int dim, int m, int parent, std::vector<HostFront>& out,
                     const std::vector<int>& Zc, int r0, int r1) {
  if (r1 - r0 == 1) {
    const size_t first = out.size();
    build_tree(b, dim, m, parent, out);
    for (size_t i = first; i < out.size(); ++i) out[i].owner = r0;
    return;
  }
  const int k = (r0 + r1) / 2;   // plane Zc[k]: ranks [r0, k) below, [k, r1) above
  const int ax = dim - 1;
  const int id = (int)out.size();
  out.push_back(HostFront());
  out[id].box = b;
  out[id].parent = parent;
  out[id].owner = k;
  out[id].top = true;
  Box sp = b; sp.lo[ax] = Zc[k]; sp.hi[ax] = Zc[k] + 1;
  push_box_nodes(sp, dim, m, out[id].sep);
  Box l = b; l.hi[ax] = Zc[k];
  Box r = b; r.lo[ax] = Zc[k] + 1;
  const int lid = (int)out.size();
  build_tree_dist(l, dim, m, id, out, Zc, r0, k);
  out[id].children.push_back(lid);
  const int rid = (int)out.size();
  build_tree_dist(r, dim, m, id, out, Zc, k, r1);
  out[id].children.push_back(rid);
}

}  // namespace

// ============================================================ host API
static hh_status plan_build(int dim, int m, const std::vector<int>* Zc, int rank, NDPlan** out);

hh_status nd_plan_create(int dim, int m, NDPlan** out) { return plan_build(dim, m, nullptr, 0, out); }

hh_status nd_plan_create_dist(int dim, int m, const std::vector<int>& Zc, int rank, NDPlan** out) {
  const int P = (int)Zc.size() - 1;
  if (P < 2 || rank < 0 || rank >= P || Zc[0] != 0 || Zc[P] != m) {
    hh_set_error("nd dist: bad plane bounds / rank");
    return HH_E_CONFIG;
  }
  for (int k = 0; k < P; ++k)
    if (Zc[k + 1] - Zc[k] < 2) {
      hh_set_error("nd dist: slab %d has %d coarse planes (need >= 2)", k, Zc[k + 1] - Zc[k]);
      return HH_E_CONFIG;
    }
  return plan_build(dim, m, &Zc, rank, out);
}

static hh_status plan_build(int dim, int m, const std::vector<int>* Zc, int rank, NDPlan** out) {
  NDPlan* nd = new NDPlan();
  nd->dim = dim; nd->m = m;
  nd->N = 1;
  for (int d = 0; d < dim; ++d) nd->N *= m;
  nd->S = dim == 2 ? 9 : 27;
  const bool dist = Zc != nullptr;
  std::vector<HostFront> tf;
  Box root;
  for (int d = 0; d < 3; ++d) { root.lo[d] = 0; root.hi[d] = (d < dim) ? m : 1; }
  if (dist) {
    nd->P = (int)Zc->size() - 1;
    nd->rank = rank;
    build_tree_dist(root, dim, m, -1, tf, *Zc, 0, nd->P);
  } else {
    build_tree(root, dim, m, -1, tf);
  }
  const int nf = (int)tf.size();
  // halo rings + levels (height above the leaves)
  for (int t = nf - 1; t >= 0; --t) {
    int lv = 0;
    for (int c : tf[t].children) lv = std::max(lv, tf[c].level + 1);
    tf[t].level = lv;
    const Box& b = tf[t].box;
    Box e = b;
    for (int d = 0; d < dim; ++d) { e.lo[d] = std::max(0, b.lo[d] - 1); e.hi[d] = std::min(m, b.hi[d] + 1); }
    int c[3] = {0, 0, 0};
    for (c[2] = (dim > 2 ? e.lo[2] : 0); c[2] < (dim > 2 ? e.hi[2] : 1); ++c[2])
      for (c[1] = e.lo[1]; c[1] < e.hi[1]; ++c[1])
        for (c[0] = e.lo[0]; c[0] < e.hi[0]; ++c[0]) {
          bool inside = true;
          for (int d = 0; d < dim; ++d) inside = inside && c[d] >= b.lo[d] && c[d] < b.hi[d];
          if (inside) continue;
          int64_t g = 0, st = 1;
          for (int d = 0; d < dim; ++d) { g += c[d] * st; st *= m; }
          tf[t].halo.push_back((int)g);
        }
  }
  // order fronts by level (stable)
  std::vector<int> order(nf);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {   // by level, then owner
    return tf[a].level != tf[b].level ? tf[a].level < tf[b].level : tf[a].owner < tf[b].owner;
  });
  std::vector<int> newid(nf);
  for (int i = 0; i < nf; ++i) newid[order[i]] = i;
  const int nlev = tf[order[nf - 1]].level + 1;

  // owner of every node: (front, position in sep)
  std::vector<int> owner(nd->N, -1), ownpos(nd->N, -1);
  for (int i = 0; i < nf; ++i) {
    const HostFront& h = tf[order[i]];
    for (size_t a = 0; a < h.sep.size(); ++a) { owner[h.sep[a]] = i; ownpos[h.sep[a]] = (int)a; }
  }
  for (int64_t g = 0; g < nd->N; ++g)
    if (owner[g] < 0) { delete nd; hh_set_error("nd: node %lld not covered", (long long)g); return HH_E_STATE; }

  nd->fronts.resize(nf);
  std::vector<int> sepAll, haloAll, eamap;
  std::vector<int4> asmE;
  int64_t Foff = 0, posOff = 0, outOff = 0, eaOff = 0;
  const int S = nd->S;
  std::vector<int> loc(nd->N, -1);
  for (int i = 0; i < nf; ++i) {
    const HostFront& h = tf[order[i]];
    FrontMeta& fm = nd->fronts[i];
    fm.s = (int)h.sep.size(); fm.u = (int)h.halo.size(); fm.f = fm.s + fm.u; fm.level = h.level;
    fm.Foff = Foff; Foff += (int64_t)fm.f * fm.f;
    fm.sepOff = (int64_t)sepAll.size(); sepAll.insert(sepAll.end(), h.sep.begin(), h.sep.end());
    fm.haloOff = (int64_t)haloAll.size(); haloAll.insert(haloAll.end(), h.halo.begin(), h.halo.end());
    fm.posOff = posOff; posOff += fm.f;
    fm.outOff = outOff; outOff += fm.u;
    fm.parent = h.parent >= 0 ? newid[h.parent] : -1;
    fm.pad = 0;
    for (int a = 0; a < fm.s; ++a) loc[h.sep[a]] = a;
    for (int b = 0; b < fm.u; ++b) loc[h.halo[b]] = fm.s + b;
    for (int a = 0; a < fm.s; ++a) {
      const int g = h.sep[a];
      int c[3] = {0, 0, 0};
      int64_t r = g;
      for (int d = 0; d < dim; ++d) { c[d] = (int)(r % m); r /= m; }
      for (int o = 0; o < S; ++o) {
        bool ok = true;
        int oo = o;
        int64_t gj = 0, st = 1;
        for (int d = 0; d < dim; ++d) {
          const int nbd = c[d] + oo % 3 - 1;
          oo /= 3;
          ok = ok && nbd >= 0 && nbd < m;
          gj += nbd * st; st *= m;
        }
        if (!ok) continue;
        const int lj = loc[gj];
        if (lj < 0) continue;                    // eliminated in a descendant
        asmE.push_back(make_int4(i, a, lj, (int)((int64_t)g * S + o)));
        if (lj >= fm.s) asmE.push_back(make_int4(i, lj, a, (int)((int64_t)g * S + o)));
      }
    }
    for (int a = 0; a < fm.s; ++a) loc[h.sep[a]] = -1;
    for (int b = 0; b < fm.u; ++b) loc[h.halo[b]] = -1;
  }
  // extend-add maps (child halo -> parent local)
  for (int i = 0; i < nf; ++i) {
    FrontMeta& fm = nd->fronts[i];
    fm.eaOff = eaOff;
    if (fm.parent < 0) continue;
    const HostFront& hp = tf[order[fm.parent]];
    const int ps = (int)hp.sep.size();
    for (int a = 0; a < ps; ++a) loc[hp.sep[a]] = a;
    for (size_t b = 0; b < hp.halo.size(); ++b) loc[hp.halo[b]] = ps + (int)b;
    const HostFront& h = tf[order[i]];
    for (int b = 0; b < fm.u; ++b) {
      const int lp = loc[h.halo[b]];
      if (lp < 0) { delete nd; hh_set_error("nd: halo node not in parent front"); return HH_E_STATE; }
      eamap.push_back(lp);
    }
    eaOff += fm.u;
    for (int a = 0; a < ps; ++a) loc[hp.sep[a]] = -1;
    for (size_t b = 0; b < hp.halo.size(); ++b) loc[hp.halo[b]] = -1;
  }
  // solve gather map: front position -> update-vector entry of child slot 0 / 1
  std::vector<int2> gmap(posOff, make_int2(-1, -1));
  for (int i = 0; i < nf; ++i) {
    const FrontMeta& fm = nd->fronts[i];
    if (fm.parent < 0) continue;
    const HostFront& hp = tf[order[fm.parent]];
    const int slot = (hp.children.size() > 1 && newid[hp.children[1]] == i) ? 1 : 0;
    const FrontMeta& pm = nd->fronts[fm.parent];
    for (int q = 0; q < fm.u; ++q) {
      int2& g = gmap[pm.posOff + eamap[fm.eaOff + q]];
      (slot ? g.y : g.x) = (int)(fm.outOff + q);
    }
  }
  // levels
  nd->levels.resize(nlev);
  std::vector<int> eaList;
  {
    int i = 0;
    int64_t ai = 0;
    for (int L = 0; L < nlev; ++L) {
      LevelInfo& li = nd->levels[L];
      li.begin = i; li.count = 0; li.max_s = li.max_u = li.max_f = 0;
      while (i < nf && nd->fronts[i].level == L) {
        li.max_s = std::max(li.max_s, nd->fronts[i].s);
        li.max_u = std::max(li.max_u, nd->fronts[i].u);
        li.max_f = std::max(li.max_f, nd->fronts[i].f);
        ++li.count; ++i;
      }
      const FrontMeta& f0 = nd->fronts[li.begin];
      const FrontMeta& fl = nd->fronts[li.begin + li.count - 1];
      li.Fbegin = f0.Foff;
      li.Fcount = fl.Foff + (int64_t)fl.f * fl.f - f0.Foff;
      li.asmBegin = ai;
      while (ai < (int64_t)asmE.size() && nd->fronts[asmE[ai].x].level == L) ++ai;
      li.asmCount = ai - li.asmBegin;
      for (int slot = 0; slot < 2; ++slot) {
        li.ea_list_off[slot] = (int64_t)eaList.size();
        li.ea_count[slot] = 0;
        for (int p = li.begin; p < li.begin + li.count; ++p) {
          const HostFront& hp = tf[order[p]];
          if ((int)hp.children.size() > slot) {
            eaList.push_back(newid[hp.children[slot]]);
            ++li.ea_count[slot];
          }
        }
      }
    }
  }
  // pivot column buffer offsets (level-local, indexed by front id)
  int64_t Cmax = 0;
  std::vector<int64_t> Coff(nf);
  for (auto& li : nd->levels) {
    int64_t o = 0;
    for (int t = li.begin; t < li.begin + li.count; ++t) { Coff[t] = o; o += (int64_t)nd->fronts[t].f * NB_MAX + NB_MAX * NB_MAX; }
    Cmax = std::max(Cmax, o);
  }
  nd->F_entries = Foff; nd->w_entries = posOff; nd->out_entries = outOff; nd->C_entries = Cmax;
  std::vector<int64_t> Koff(nf, 0);
  for (const LevelInfo& li : nd->levels) {
    int64_t ko = 0;
    for (int t = li.begin; t < li.begin + li.count; ++t) {
      Koff[t] = ko;
      ko += (int64_t)((nd->fronts[t].f + 2047) / 2048) * nd->fronts[t].s;
    }
    if (li.max_f > bwdk_f()) nd->Kmax = std::max(nd->Kmax, ko);
  }
  // distributed plan: keep the global level ranges for the packed-S offsets,
  // narrow `levels` to this rank's fronts, and record the exchange lists
  const std::vector<LevelInfo> glevels = nd->levels;
  if (dist) {
    nd->owner.resize(nf);
    for (int i = 0; i < nf; ++i) nd->owner[i] = tf[order[i]].owner;
    nd->xcross.assign(nlev, {});
    nd->xtop.assign(nlev, {});
    for (int L = 0; L < nlev; ++L) {
      LevelInfo& li = nd->levels[L];
      const int gb = li.begin, ge = li.begin + li.count;
      int b0 = gb;
      while (b0 < ge && nd->owner[b0] < rank) ++b0;
      int b1 = b0;
      while (b1 < ge && nd->owner[b1] == rank) ++b1;
      li.begin = b0;
      li.count = b1 - b0;
      li.max_s = li.max_u = li.max_f = 0;
      for (int t = b0; t < b1; ++t) {
        li.max_s = std::max(li.max_s, nd->fronts[t].s);
        li.max_u = std::max(li.max_u, nd->fronts[t].u);
        li.max_f = std::max(li.max_f, nd->fronts[t].f);
      }
      int64_t topsum = 0;
      for (int t = gb; t < ge; ++t) {
        const int p = nd->fronts[t].parent;
        if (p >= 0 && nd->owner[p] != nd->owner[t]) nd->xcross[L].push_back(t);
        if (tf[order[t]].top) {
          nd->xtop[L].push_back(t);
          topsum += nd->fronts[t].s;
        }
      }
      nd->top_sep_max = std::max(nd->top_sep_max, topsum);
    }
  }
  // lean storage for trees whose full fronts would not fit (3D coarse grids of
  // cfg4 size); HH_ND_LEAN=0/1 overrides, HH_ND_WMAX sets the workspace (entries)
  std::vector<FrontMeta> fronts_w;
  std::vector<int64_t> Coff_w(nf, 0), Soff(nf, 0), Poff(nf, 0);
  std::vector<int> eaListC;
  {
    const char* el = getenv("HH_ND_LEAN");
    nd->lean = dist || (el ? atoi(el) != 0 : 16.0 * (double)Foff > 24e9);   // distributed: always lean
  }
  if (nd->lean) {
    const int64_t Wlim = getenv("HH_ND_WMAX") ? atoll(getenv("HH_ND_WMAX")) : (int64_t)750000000;
    fronts_w = nd->fronts;
    int64_t xh = 0;
    std::vector<int64_t> asmFirst(nf + 1, (int64_t)asmE.size());
    for (int64_t q = (int64_t)asmE.size() - 1; q >= 0; --q) asmFirst[asmE[q].x] = q;
    for (int t = nf - 1; t >= 0; --t) asmFirst[t] = std::min(asmFirst[t], asmFirst[t + 1]);
    for (int L = 0; L < nlev; ++L) {
      const LevelInfo& li = nd->levels[L];
      int64_t so = 0, po = 0;
      int t = li.begin;
      const int tend = li.begin + li.count;
      while (t < tend) {
        Chunk ch;
        ch.level = L; ch.t0 = t;
        int64_t w = 0, co = 0;
        while (t < tend) {
          const int64_t ff = (int64_t)nd->fronts[t].f * nd->fronts[t].f;
          if (t > ch.t0 && w + ff > Wlim) break;
          fronts_w[t].Foff = w;
          w += ff;
          Coff_w[t] = co;
          co += (int64_t)nd->fronts[t].f * NB_MAX + NB_MAX * NB_MAX;
          ++t;
        }
        ch.t1 = t;
        ch.Wcount = w;
        nd->Wmax = std::max(nd->Wmax, w);
        nd->Cw = std::max(nd->Cw, co);
        ch.asmBegin = asmFirst[ch.t0];
        ch.asmCount = asmFirst[ch.t1] - asmFirst[ch.t0];
        for (int slot = 0; slot < 2; ++slot) {
          ch.ea_list_off[slot] = (int64_t)eaListC.size();
          ch.ea_count[slot] = 0;
          for (int pp = ch.t0; pp < ch.t1; ++pp) {
            const HostFront& hp = tf[order[pp]];
            if ((int)hp.children.size() > slot) {
              eaListC.push_back(newid[hp.children[slot]]);
              ++ch.ea_count[slot];
            }
          }
        }
        nd->chunks.push_back(ch);
      }
      for (int q = li.begin; q < tend; ++q) {
        FrontMeta& fm = nd->fronts[q];
        Poff[q] = po;
        po += (int64_t)((fm.s + 255) / 256) * fm.u;
        fm.Foff = xh;                      // the solve reads [X | H] here
        xh += (int64_t)fm.s * fm.f;
      }
      nd->Pmax = std::max(nd->Pmax, po);
      (void)so;
    }
    nd->F_entries = xh;
    // packed-S store: a front's S lives from its own level to its parent's level;
    // offsets by first-fit over the levels (S read by level L is freed after level L)
    std::map<int64_t, int64_t> freel;   // offset -> length
    int64_t top = 0;
    auto alloc = [&](int64_t n) -> int64_t {
      for (auto it = freel.begin(); it != freel.end(); ++it)
        if (it->second >= n) {
          const int64_t o = it->first, len = it->second;
          freel.erase(it);
          if (len > n) freel[o + n] = len - n;
          return o;
        }
      const int64_t o = top;
      top += n;
      return o;
    };
    auto release = [&](int64_t o, int64_t n) {
      auto it = freel.emplace(o, n).first;
      auto nx = std::next(it);
      if (nx != freel.end() && it->first + it->second == nx->first) { it->second += nx->second; freel.erase(nx); }
      if (it != freel.begin()) {
        auto pv = std::prev(it);
        if (pv->first + pv->second == it->first) { pv->second += it->second; freel.erase(it); }
      }
    };
    // distributed plans: only the S blocks this rank touches get a place -- its own
    // fronts' (sent on after their level when the parent lives elsewhere) and the
    // ones its fronts receive from children of other owners; every rank places
    // them in its own store (the transfers use each side's own offsets)
    auto own = [&](int q) { return !dist || nd->owner[q] == rank; };
    auto touches = [&](int q) {
      const int p = nd->fronts[q].parent;
      return p >= 0 && (own(q) || own(p));
    };
    std::vector<int> sent_prev;   // own fronts of the previous level whose S went to another rank
    for (int L = 0; L < nlev; ++L) {
      const LevelInfo& li = glevels[L];
      for (int q = li.begin; q < li.begin + li.count; ++q) {
        const FrontMeta& fm = nd->fronts[q];
        Soff[q] = touches(q) ? alloc((int64_t)fm.u * (fm.u + 1) / 2) : 0;
      }
      for (int q = li.begin; q < li.begin + li.count; ++q) {
        if (!own(q)) continue;
        for (int c : tf[order[q]].children) {   // consumed by this level's extend-add
          const FrontMeta& fc = nd->fronts[newid[c]];
          release(Soff[newid[c]], (int64_t)fc.u * (fc.u + 1) / 2);
        }
      }
      for (int q : sent_prev) {
        const FrontMeta& fc = nd->fronts[q];
        release(Soff[q], (int64_t)fc.u * (fc.u + 1) / 2);
      }
      sent_prev.clear();
      for (int q = li.begin; q < li.begin + li.count; ++q)
        if (dist && own(q) && touches(q) && !own(nd->fronts[q].parent)) sent_prev.push_back(q);
    }
    nd->Smax[0] = std::max<int64_t>(1, top);
    nd->Smax[1] = 0;
  }
  int64_t sb = 0;
  for (int t = 0; t < nf; ++t) {
    if (dist && nd->owner[t] != rank) continue;   // distributed: this rank's fronts only
    const FrontMeta& fm = nd->fronts[t];
    sb += (int64_t)fm.s * fm.f + (int64_t)fm.u * fm.s;
  }
  nd->stream_bytes = sb * (int64_t)sizeof(cplx);
  nd->Soff_h = Soff;

  // bottom-subtree decompositions for every cut level (not for distributed plans:
  // they always run the per-level lean schedule)
  std::vector<int> sptr_all, slist_all;
  if (!dist) {
    std::vector<std::vector<int>> kids(nf);
    for (int i = 0; i < nf; ++i)
      if (nd->fronts[i].parent >= 0) kids[nd->fronts[i].parent].push_back(i);
    for (int L = 0; L < nlev; ++L) {
      nd->sub_off.push_back((int64_t)sptr_all.size());
      nd->list_off.push_back((int64_t)slist_all.size());
      int cnt = 0, maxf = 0;
      double worst = 0;
      const int base = (int)slist_all.size();
      for (int r = 0; r < nf; ++r) {
        const FrontMeta& fm = nd->fronts[r];
        if (fm.level > L) continue;
        if (fm.parent >= 0 && nd->fronts[fm.parent].level <= L) continue;
        // subtree of r in bottom-up order: BFS then reverse
        std::vector<int> order_sub{r};
        for (size_t q = 0; q < order_sub.size(); ++q)
          for (int c : kids[order_sub[q]]) order_sub.push_back(c);
        std::reverse(order_sub.begin(), order_sub.end());
        sptr_all.push_back((int)slist_all.size() - base);
        double cost = 0;
        for (int t : order_sub) {
          const FrontMeta& ft = nd->fronts[t];
          maxf = std::max(maxf, ft.f);
          // measured on B200: ~5 us of dependent-load latency per front + ~40 GB/s per CTA
          cost += 5.0 + ((double)ft.s * ft.f + (double)ft.u * ft.s) * 16.0 / 4.0e4;
          slist_all.push_back(t);
        }
        worst = std::max(worst, cost);
        ++cnt;
      }
      sptr_all.push_back((int)slist_all.size() - base);
      nd->sub_cnt.push_back(cnt);
      nd->sub_cost_us.push_back(worst);
      nd->sub_maxf.push_back(maxf);
    }
  }
  // per-level ranges and entry -> front maps for the cluster solve
  std::vector<int> sep_front(sepAll.size()), halo_front(haloAll.size()), pos_front(posOff);
  std::vector<int64_t> lvr(6 * nlev);
  for (int i = 0; i < nf; ++i) {
    const FrontMeta& fm = nd->fronts[i];
    for (int a = 0; a < fm.s; ++a) sep_front[fm.sepOff + a] = i;
    for (int b = 0; b < fm.u; ++b) halo_front[fm.haloOff + b] = i;
    for (int p = 0; p < fm.f; ++p) pos_front[fm.posOff + p] = i;
  }
  nd->level_bytes.assign(nlev, 0.0);
  for (int L = 0; L < nlev; ++L) {
    const LevelInfo& li = nd->levels[L];
    if (li.count == 0) continue;
    const FrontMeta& f0 = nd->fronts[li.begin];
    const FrontMeta& fl = nd->fronts[li.begin + li.count - 1];
    lvr[6 * L] = f0.sepOff;
    lvr[6 * L + 1] = fl.sepOff + fl.s;
    lvr[6 * L + 2] = f0.haloOff;
    lvr[6 * L + 3] = fl.haloOff + fl.u;
    lvr[6 * L + 4] = f0.posOff;
    lvr[6 * L + 5] = fl.posOff + fl.f;
    for (int t = li.begin; t < li.begin + li.count; ++t)
      nd->level_bytes[L] += 16.0 * ((double)nd->fronts[t].s * nd->fronts[t].f + (double)nd->fronts[t].u * nd->fronts[t].s);
  }
  auto up = [&](auto** dptr, const auto& vec) -> hh_status {
    using T = typename std::remove_reference<decltype(vec)>::type::value_type;
    const size_t bytes = std::max<size_t>(1, vec.size()) * sizeof(T);
    if (cudaMalloc((void**)dptr, bytes) != cudaSuccess) {
      cudaGetLastError();
      hh_set_error("nd: cudaMalloc %zu B failed", bytes);
      return HH_E_OOM;
    }
    if (!vec.empty()) HH_CUDA_TRY(cudaMemcpy(*dptr, vec.data(), vec.size() * sizeof(T), cudaMemcpyHostToDevice));
    return HH_OK;
  };
  hh_status st = HH_OK;
  if (st == HH_OK) st = up(&nd->d_fronts, nd->fronts);
  if (st == HH_OK) st = up(&nd->d_sep, sepAll);
  if (st == HH_OK) st = up(&nd->d_halo, haloAll);
  if (st == HH_OK) st = up(&nd->d_asm, asmE);
  if (st == HH_OK) st = up(&nd->d_eamap, eamap);
  if (st == HH_OK) st = up(&nd->d_eaList, eaList);
  if (st == HH_OK) st = up(&nd->d_gmap, gmap);
  if (st == HH_OK) st = up(&nd->d_Coff, Coff);
  if (st == HH_OK) st = up(&nd->d_sub_ptr, sptr_all);
  if (st == HH_OK) st = up(&nd->d_sub_list, slist_all);
  if (st == HH_OK) st = up(&nd->d_sep_front, sep_front);
  if (st == HH_OK) st = up(&nd->d_halo_front, halo_front);
  if (st == HH_OK) st = up(&nd->d_pos_front, pos_front);
  if (st == HH_OK) st = up(&nd->d_Koff, Koff);
  if (st == HH_OK && nd->lean) st = up(&nd->d_fronts_w, fronts_w);
  if (st == HH_OK && nd->lean) st = up(&nd->d_Coff_w, Coff_w);
  if (st == HH_OK && nd->lean) st = up(&nd->d_Soff, Soff);
  if (st == HH_OK && nd->lean) st = up(&nd->d_Poff, Poff);
  if (st == HH_OK && nd->lean) st = up(&nd->d_eaListC, eaListC);
  if (st == HH_OK) st = up(&nd->d_lvr, lvr);
  {
    std::vector<int2> child(nd->fronts.size(), make_int2(-1, -1));
    for (size_t t = 0; t < nd->fronts.size(); ++t) {
      const int p = nd->fronts[t].parent;
      if (p < 0) continue;
      if (child[p].x < 0) child[p].x = (int)t; else child[p].y = (int)t;
    }
    std::vector<int> lvbeg(nd->levels.size());
    for (size_t L = 0; L < nd->levels.size(); ++L) lvbeg[L] = nd->levels[L].begin;
    if (st == HH_OK) st = up(&nd->d_child, child);
    if (st == HH_OK) st = up(&nd->d_lvbeg, lvbeg);
  }
  if (st != HH_OK) { nd_plan_destroy(nd); return st; }
  *out = nd;
  return HH_OK;
}

void nd_plan_destroy(NDPlan* nd) {
  if (!nd) return;
  cudaFree(nd->d_fronts); cudaFree(nd->d_sep); cudaFree(nd->d_halo); cudaFree(nd->d_asm);
  cudaFree(nd->d_eamap); cudaFree(nd->d_eaList); cudaFree(nd->d_gmap);
  cudaFree(nd->d_Coff); cudaFree(nd->d_sub_ptr); cudaFree(nd->d_sub_list);
  cudaFree(nd->d_sep_front); cudaFree(nd->d_halo_front); cudaFree(nd->d_pos_front);
  cudaFree(nd->d_lvr); cudaFree(nd->d_child); cudaFree(nd->d_lvbeg);
  cudaFree(nd->d_fronts_w); cudaFree(nd->d_Coff_w); cudaFree(nd->d_Soff); cudaFree(nd->d_Poff);
  cudaFree(nd->d_eaListC); cudaFree(nd->d_Koff);
  delete nd;
}

int64_t nd_front_entries(const NDPlan* p) { return p->F_entries; }
int64_t nd_stream_bytes(const NDPlan* p) { return p->stream_bytes; }
int nd_levels(const NDPlan* p) { return (int)p->levels.size(); }
// per sample: w | update vectors | lean forward partials | K-split backward partials
// flow-solve completion counters (2 ints per front) at the end of each sample's work
static int64_t flow_cnt_off(const NDPlan* p) {
  return p->w_entries + p->out_entries + (p->lean ? p->Pmax : 0) + p->Kmax;
}
static int64_t flow_cnt_entries(const NDPlan* p) {
  return p->lean ? 0 : ((int64_t)p->fronts.size() * 2 * (int64_t)sizeof(int) + 15) / 16;
}
int64_t nd_work_entries(const NDPlan* p) { return flow_cnt_off(p) + flow_cnt_entries(p); }
int64_t nd_cbuf_entries(const NDPlan* p) {
  if (p->lean) return p->Cw + p->Wmax + p->Smax[0] + p->Smax[1];
  return std::max<int64_t>(1, p->C_entries);
}

// The partial Gauss-Jordan sweep of `cnt` fronts (x Bn samples) starting at t0:
// pivot blocks of 32 on fronts of order >= HH_ND_NB32_F (default 1024), 16 below
// (64 from HH_ND_NB64_F, off by default) -- larger blocks mean fewer passes over
// the front and more multiply-adds per byte, smaller ones more CTAs.
static int nb32_f() {
  static const int v = getenv("HH_ND_NB32_F") ? atoi(getenv("HH_ND_NB32_F")) : 1024;
  return v;
}
static int nb64_f() {   // pivot blocks of 64 from this front order (HH_ND_NB64_F; compiled in only
                        // with NB_MAX = 64: 2 CTAs per SM and the longer serial inversion lost,
                        // cfg3 372 -> 398-405 ms)
  static const int v = getenv("HH_ND_NB64_F") ? atoi(getenv("HH_ND_NB64_F")) : (1 << 30);
  return v;
}
template <int NBT>
static size_t piv_smem() { return ((size_t)NBT * (NBT + 1) + 2 * NBT + (NBT > 16 ? (size_t)NBT * 32 : 0)) * sizeof(cplx); }
template <int UR, int NBT>
static size_t upd_smem() { return ((size_t)UR * NBT + (size_t)NBT * UT) * sizeof(cplx); }

static int ur64_f() {   // 64-row update tiles from this front order (HH_ND_UR64_F)
  static const int v = getenv("HH_ND_UR64_F") ? atoi(getenv("HH_ND_UR64_F")) : 1024;
  return v;
}
template <int NBT>
static void pivot_sweep_nb(const FrontMeta* fr, int t0, int cnt, int Bn, int ms, int mf, cplx* F, int64_t FE,
                           cplx* C, int64_t CE, const int64_t* coff, int* flag, cudaStream_t s) {
  const bool big = mf >= ur64_f();
  const int tiles = (mf + UT - 1) / UT;
  const dim3 gp(cnt, Bn, (mf + PIV_CHUNK - 1) / PIV_CHUNK);
  const dim3 gu((mf + (big ? 63 : 31)) / (big ? 64 : 32) * tiles, cnt, Bn);
  const size_t sp = piv_smem<NBT>() + (NBT == 16 && !ND_PIV_REG ? (size_t)NBT * 32 * sizeof(cplx) : 0), su = big ? upd_smem<64, NBT>() : upd_smem<32, NBT>();
  if (sp > 48 * 1024) smem_attr((const void*)k_nd_piv<NBT>, sp);
  if (su > 48 * 1024) smem_attr(big ? (const void*)k_nd_upd<64, NBT> : (const void*)k_nd_upd<32, NBT>, su);
  // FP64 tensor-core (DMMA) update (HH_ND_MMA: 0 = FMA kernels, 1 = DMMA on the 64-row
  // tiles only, 2 (default) = DMMA on all tiles)
  static const int use_mma = getenv("HH_ND_MMA") ? atoi(getenv("HH_ND_MMA")) : 2;
  const bool mma = (big ? use_mma >= 1 : use_mma >= 2) && NBT % 4 == 0;
  const size_t sm_mma = big ? upd_mma_smem<64, NBT>() : upd_mma_smem<32, NBT>();
  if (mma && sm_mma > 48 * 1024)
    smem_attr(big ? (const void*)k_nd_upd_mma<64, NBT> : (const void*)k_nd_upd_mma<32, NBT>, sm_mma);
  for (int kb = 0; kb < ms; kb += NBT) {
    k_nd_piv<NBT><<<gp, 256, sp, s>>>(fr, t0, kb, F, FE, C, CE, coff, flag);
    if (mma && big) k_nd_upd_mma<64, NBT><<<gu, 256, sm_mma, s>>>(fr, t0, kb, tiles, F, FE, C, CE, coff);
    else if (mma) k_nd_upd_mma<32, NBT><<<gu, 256, sm_mma, s>>>(fr, t0, kb, tiles, F, FE, C, CE, coff);
    else if (big) k_nd_upd<64, NBT><<<gu, 256, su, s>>>(fr, t0, kb, tiles, F, FE, C, CE, coff);
    else k_nd_upd<32, NBT><<<gu, 256, su, s>>>(fr, t0, kb, tiles, F, FE, C, CE, coff);
  }
}
static void pivot_sweep(const FrontMeta* fr, int t0, int cnt, int Bn, int ms, int mf, cplx* F, int64_t FE,
                        cplx* C, int64_t CE, const int64_t* coff, int* flag, cudaStream_t s) {
  if constexpr (NB_MAX >= 64) {
    if (mf >= nb64_f()) {
      pivot_sweep_nb<64>(fr, t0, cnt, Bn, ms, mf, F, FE, C, CE, coff, flag, s);
      return;
    }
  }
  if (mf >= nb32_f()) pivot_sweep_nb<32>(fr, t0, cnt, Bn, ms, mf, F, FE, C, CE, coff, flag, s);
  else pivot_sweep_nb<16>(fr, t0, cnt, Bn, ms, mf, F, FE, C, CE, coff, flag, s);
}

// one chunk of the lean factorisation: zero the workspace, assemble the coarse
// stencil entries, extend-add the children's packed Schur complements, Gauss-Jordan
// sweep, copy [X | H] and the packed S out
// C: pivot columns (nd->Cw entries), W: workspace (nd->Wmax), Sst: packed Schur
// complements (first-fit offsets, see the plan; nd->Smax[0] entries)
static hh_status lean_chunk(const NDPlan* nd, const Chunk& ch, const cplx* st, cplx* F, cplx* C, cplx* W,
                            cplx* Sst, int* flag, cudaStream_t s) {
  const int64_t stS = nd->N * nd->S;
  static const int lprof = getenv("HH_PROFILE_SETUP") ? atoi(getenv("HH_PROFILE_SETUP")) : 0;
  const int cnt = ch.t1 - ch.t0;
  int ms = 0, mf = 0;
  for (int t = ch.t0; t < ch.t1; ++t) { ms = std::max(ms, nd->fronts[t].s); mf = std::max(mf, nd->fronts[t].f); }
  cudaEvent_t ce0 = nullptr, ce1 = nullptr;   // HH_PROFILE_SETUP=2: per-chunk timing (diagnostics)
  if (lprof >= 2) {
    cudaEventCreate(&ce0); cudaEventCreate(&ce1);
    cudaEventRecord(ce0, s);
  }
  struct ChunkTimer {
    cudaEvent_t a, b; cudaStream_t st; const Chunk& c; int n, ms, mf; const NDPlan* p;
    ~ChunkTimer() {
      if (!a) return;
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms_ = 0;
      cudaEventElapsedTime(&ms_, a, b);
      double fl = 0;
      for (int t = c.t0; t < c.t1; ++t) fl += 8.0 * (double)p->fronts[t].s * p->fronts[t].f * p->fronts[t].f;
      fprintf(stderr, "[hh factor] lean m=%d level %d chunk: %d fronts max_s=%d max_f=%d %.3f ms %.2f TFLOP/s\n",
              p->m, c.level, n, ms, mf, ms_, fl / (ms_ * 1e-3) / 1e12);
      cudaEventDestroy(a); cudaEventDestroy(b);
    }
  } ctimer{ce0, ce1, s, ch, cnt, ms, mf, nd};
  {
    const unsigned gx = (unsigned)std::min<int64_t>(8192, (ch.Wcount + 255) / 256);
    k_nd_zero<<<dim3(gx, 1), 256, 0, s>>>(W, 0, 0, ch.Wcount);
  }
  if (ch.asmCount) {
    k_nd_assemble<<<dim3((unsigned)((ch.asmCount + 255) / 256), 1), 256, 0, s>>>(
        nd->d_asm + ch.asmBegin, ch.asmCount, nd->d_fronts_w, st, stS, W, 0);
  }
  for (int slot = 0; slot < 2; ++slot) {
    if (!ch.ea_count[slot]) continue;
    k_nd_ea_packed<<<dim3(ch.ea_count[slot], 64), 128, 0, s>>>(nd->d_eaListC + ch.ea_list_off[slot],
                                                               nd->d_fronts_w, nd->d_Soff, Sst,
                                                               nd->d_eamap, W);
  }
  pivot_sweep(nd->d_fronts_w, ch.t0, cnt, 1, ms, mf, W, 0, C, 0, nd->d_Coff_w + ch.t0, flag, s);
  k_nd_copyout<<<dim3(cnt, 64), 256, 0, s>>>(nd->d_fronts_w, nd->d_fronts, nd->d_Soff, ch.t0, W, F, Sst);
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

hh_status nd_factor(const NDPlan* nd, int B, const cplx* st, cplx* F, cplx* cbuf, int* flag,
                    cudaStream_t s) {
  const int64_t FE = nd->F_entries, CE = nd_cbuf_entries(nd);
  const int64_t stS = nd->N * nd->S;
  HH_CUDA_TRY(cudaMemsetAsync(flag, 0, B * sizeof(int), s));
  if (nd->lean) {
    if (B != 1) { hh_set_error("lean ND storage needs one problem per factorisation"); return HH_E_CONFIG; }
    for (const Chunk& ch : nd->chunks)
      HH_TRY(lean_chunk(nd, ch, st, F, cbuf, cbuf + nd->Cw, cbuf + nd->Cw + nd->Wmax, flag, s));
    return HH_OK;
  }
  static const int prof = getenv("HH_PROFILE_SETUP") ? atoi(getenv("HH_PROFILE_SETUP")) : 0;
  for (size_t L = 0; L < nd->levels.size(); ++L) {
    const LevelInfo& li = nd->levels[L];
    cudaEvent_t pe0 = nullptr, pe1 = nullptr;
    if (prof >= 2) {
      cudaEventCreate(&pe0); cudaEventCreate(&pe1);
      cudaEventRecord(pe0, s);
    }
    {
      const unsigned gx = (unsigned)std::min<int64_t>(4096, (li.Fcount + 255) / 256);
      k_nd_zero<<<dim3(gx, B), 256, 0, s>>>(F, FE, li.Fbegin, li.Fcount);
    }
    if (li.asmCount) {
      const int bs = 256;
      k_nd_assemble<<<dim3((unsigned)((li.asmCount + bs - 1) / bs), B), bs, 0, s>>>(
          nd->d_asm + li.asmBegin, li.asmCount, nd->d_fronts, st, stS, F, FE);
    }
    for (int slot = 0; slot < 2; ++slot) {
      if (!li.ea_count[slot]) continue;
      dim3 g(li.ea_count[slot], 32, B);
      k_nd_extend_add<<<g, 128, 0, s>>>(nd->d_eaList + li.ea_list_off[slot], nd->d_fronts,
                                        nd->d_eamap, F, FE);
    }
    pivot_sweep(nd->d_fronts, li.begin, li.count, B, li.max_s, li.max_f, F, FE, cbuf, CE, nd->d_Coff + li.begin,
                flag, s);
    HH_CUDA_TRY(cudaGetLastError());
    if (prof >= 2) {
      cudaEventRecord(pe1, s);
      cudaEventSynchronize(pe1);
      float ms = 0;
      cudaEventElapsedTime(&ms, pe0, pe1);
      double fl = 0;
      for (int t = li.begin; t < li.begin + li.count; ++t)
        fl += 8.0 * (double)nd->fronts[t].s * nd->fronts[t].f * nd->fronts[t].f;
      fprintf(stderr, "[hh factor] m=%d B=%d level %zu: %d fronts max_s=%d max_f=%d %.3f ms %.2f TFLOP/s\n",
              nd->m, B, L, li.count, li.max_s, li.max_f, ms, fl * B / (ms * 1e-3) / 1e12);
      cudaEventDestroy(pe0); cudaEventDestroy(pe1);
    }
  }
  return HH_OK;
}

// CTAs per sample in the cluster solve (16: non-portable cluster size, opted in below)
static int cluster_size() {
  static const int v = getenv("HH_ND_CLUSTER") ? atoi(getenv("HH_ND_CLUSTER")) : 16;
  return v;
}

static bool cached_cfg(NDPlan* nd, int key, SolveCfg* c) {
  std::lock_guard<std::mutex> lk(nd->cut_mu);
  for (auto& e : nd->cfg_cache)
    if (e.first == key) { *c = e.second; return true; }
  return false;
}

static int cfg_key(int B, bool conc) { return 2 * B + (conc ? 1 : 0); }
static SolveCfg get_cfg(NDPlan* nd, int B, bool conc) {
  SolveCfg c{-1, (int)nd->levels.size() - 1};
  if (const char* e = getenv("HH_ND_SPLIT")) c.split = std::min<int>(atoi(e), c.split);
  if (const char* e = getenv("HH_ND_CUT")) c.sub_cut = std::min<int>(atoi(e), c.split);
  if (const char* e = getenv("HH_ND_FLOW")) c.flow = atoi(e);
  if (nd->flow_disabled) c.flow = 0;
  if (getenv("HH_ND_SPLIT") || getenv("HH_ND_CUT")) return c;
  SolveCfg cc;
  if (cached_cfg(nd, cfg_key(B, conc), &cc)) return cc;
  return c;
}

// levels with at least this many rows per front run the wide path (HH_ND_WIDE)
static int wide_rows() {
  static const int v = getenv("HH_ND_WIDE") ? atoi(getenv("HH_ND_WIDE")) : 128;
  return v;
}

// ... and fronts of at least this order (HH_ND_WIDE_F): the 2D fronts (f <= ~770)
// are faster with the per-front gather in shared memory
static int wide_f() {
  static const int v = getenv("HH_ND_WIDE_F") ? atoi(getenv("HH_ND_WIDE_F")) : 1024;
  return v;
}

// launch with programmatic stream serialisation (PDL); HH_NO_PDL=1 disables it
static const bool g_pdl = getenv("HH_NO_PDL") == nullptr;
template <typename... Args>
static hh_status launch_pdl(void (*kern)(Args...), dim3 grid, int block, size_t smem, cudaStream_t s,
                            Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  HH_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args...));
  return HH_OK;
}

// CTAs per front of a per-level launch: one warp per row at most, and only as
// many as needed to put ~4 CTAs on every SM
static int g_fill_ctas = getenv("HH_ND_FILL") ? atoi(getenv("HH_ND_FILL")) : 4 * 148;
static int level_split(int rows, int count, int B, int len) {
  const int rpc = (LT / 32) * (32 / wide_group(std::max(1, len))) * ND_RB;   // rows per CTA pass
  const int by_rows = std::max(1, (rows + rpc - 1) / rpc);
  const int fill = std::max(1, (g_fill_ctas + count * B - 1) / (count * B));
  return std::max(1, std::min(std::min(by_rows, fill), 65535));
}

// the dataflow kernels cover levels (cut, Lb] when every one of them takes the
// narrow per-level path (front vectors staged in shared memory, no wide rows)
static bool flow_ok(const NDPlan* nd, int cut, int Lb) {
  if (nd->lean || nd->dim != 2 || Lb - cut < 1 || Lb - cut > FLOW_MAXL || getenv("HH_NO_FLOW")) return false;
  for (int L = cut + 1; L <= Lb; ++L) {
    const LevelInfo& li = nd->levels[L];
    if (li.max_f > nd_vmax()) return false;
    if ((li.max_u >= wide_rows() || li.max_s >= wide_rows()) && li.max_f >= wide_f()) return false;
  }
  return true;
}

static hh_status flow_launch(const NDPlan* nd, const SolveArgs& A, int B, int L0, int L1, bool fwd,
                             cudaStream_t s) {
  FlowArgs W;
  W.L0 = L0; W.nl = L1 - L0 + 1;
  W.cnt_off = flow_cnt_off(nd);
  W.nfr = (int)nd->fronts.size();
  {
    const char* e = getenv("HH_ND_FLOW_POLLS");   // 0: every wait fails (fault injection for tests)
    W.max_polls = e ? (unsigned)strtoul(e, nullptr, 10) : (1u << 24);
  }
  int maxf = 1;
  for (int j = 0; j < W.nl; ++j) {
    const LevelInfo& li = nd->levels[L0 + j];
    W.nch[j] = level_split(fwd ? li.max_u : li.max_s, li.count, B, fwd ? li.max_s : li.max_f);
    maxf = std::max(maxf, li.max_f);
  }
  int64_t tot = 0;
  for (int k = 0; k < W.nl; ++k) {
    const int j = fwd ? k : W.nl - 1 - k;
    W.lev[k] = j;
    W.base[k] = (int)tot;
    tot += (int64_t)nd->levels[L0 + j].count * B * W.nch[j];
  }
  W.base[W.nl] = (int)tot;
  if (tot > INT32_MAX) { hh_set_error("nd flow: too many CTAs"); return HH_E_CONFIG; }
  const size_t sm = (size_t)maxf * sizeof(cplx);
  if (fwd) {
    if (sm > 48 * 1024) HH_CUDA_TRY(smem_attr((const void*)k_nd_flow_fwd, sm));
    return launch_pdl(k_nd_flow_fwd, dim3((unsigned)tot), LT, sm, s, A, W, (const int*)nd->d_lvbeg,
                      (const int2*)nd->d_child, B);
  }
  if (sm > 48 * 1024) HH_CUDA_TRY(smem_attr((const void*)k_nd_flow_bwd, sm));
  return launch_pdl(k_nd_flow_bwd, dim3((unsigned)tot), LT, sm, s, A, W, (const int*)nd->d_lvbeg, B);
}

// one level of the forward solve on lean storage: gather w_t, then the update
// vectors upd_t = w_t[halo] - H^T z_s from the transposed [X | H] rows
static hh_status lean_fwd_level(const NDPlan* nd, const SolveArgs& A, const LevelInfo& li, int B, cudaStream_t s) {
  if (li.count == 0) return HH_OK;   // (distributed plans: no front of this rank on the level)
  dim3 gg(li.count, std::max(1, std::min(64, (li.max_f + 255) / 256)), B);
  HH_TRY(launch_pdl(k_nd_gather, gg, 256, 0, s, A, li.begin));
  if (li.max_u == 0) return HH_OK;
  const int ncb = (li.max_u + FT_COLS - 1) / FT_COLS, nrc = (li.max_s + FT_ROWS - 1) / FT_ROWS;
  const int64_t PE = nd->w_entries + nd->out_entries;
  HH_TRY(launch_pdl(k_nd_fwdT, dim3(ncb * nrc, li.count, B), FT_COLS, 0, s, A, li.begin,
                    (const int64_t*)nd->d_Poff, ncb, PE));
  HH_TRY(launch_pdl(k_nd_fwdT_red, dim3((li.max_u + 255) / 256, li.count, B), 256, 0, s, A, li.begin,
                    (const int64_t*)nd->d_Poff, PE));
  return HH_OK;
}

// one level of the backward solve: x[sep] = [X | H] [z_s ; -x[halo]]
static hh_status bwd_level(const NDPlan* nd, const SolveArgs& A, const LevelInfo& li, int B, cudaStream_t s) {
  if (li.count == 0) return HH_OK;
  if (li.max_f > A.vmax || (li.max_s >= wide_rows() && (nd->dim == 3 || li.max_f >= wide_f()))) {
    dim3 gg(li.count, std::max(1, std::min(64, (li.max_u + 255) / 256)), B);
    HH_TRY(launch_pdl(k_nd_bwd_stage, gg, 256, 0, s, A, li.begin));
    if (li.max_f > bwdk_f() && !getenv("HH_NO_BWDK")) {   // long rows: K-split over column chunks
      const int ncb = (li.max_f + KC - 1) / KC, nrb = (li.max_s + KR - 1) / KR;
      const int64_t KE = nd->w_entries + nd->out_entries + (nd->lean ? nd->Pmax : 0);
      HH_TRY(launch_pdl(k_nd_bwdK, dim3(nrb * ncb, li.count, B), LT, 0, s, A, li.begin, ncb,
                        (const int64_t*)nd->d_Koff, KE));
      HH_TRY(launch_pdl(k_nd_bwdK_red, dim3((li.max_s + 255) / 256, li.count, B), 256, 0, s, A, li.begin,
                        (const int64_t*)nd->d_Koff, KE));
      return HH_OK;
    }
    // fronts whose vector does not fit read it from L2: no shared memory then (occupancy)
    const size_t sm = li.max_f > A.vmax ? 0 : (size_t)li.max_f * sizeof(cplx);
    if (sm > 48 * 1024)
      HH_CUDA_TRY(smem_attr((const void*)k_nd_rows_wide<1>, sm));
    dim3 g(li.count, (li.max_s + WIDE_RPC - 1) / WIDE_RPC, B);
    HH_TRY(launch_pdl(k_nd_rows_wide<1>, g, LT, sm, s, A, li.begin, (int)(sm / sizeof(cplx))));
    return HH_OK;
  }
  const size_t sm = (size_t)std::min(li.max_f, A.vmax) * sizeof(cplx);
  if (sm > 48 * 1024) HH_CUDA_TRY(smem_attr((const void*)k_nd_bwd, sm));
  dim3 g(li.count, level_split(li.max_s, li.count, B, li.max_f), B);
  HH_TRY(launch_pdl(k_nd_bwd, g, LT, sm, s, A, li.begin));
  return HH_OK;
}

static hh_status solve_cfg(NDPlan* nd, int B, const int* st, const cplx* F, cplx* work, VArg rhs,
                           VArg x, cudaStream_t s, SolveCfg c, bool shareF, bool conc, int* fail = nullptr) {
  const int nlev = (int)nd->levels.size();
  // HH_ND_LEVEL_TIMING=1: per-level event timing (diagnostics; synchronises, never in graphs)
  static const bool lt = getenv("HH_ND_LEVEL_TIMING") != nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  const bool timing = lt && cap == cudaStreamCaptureStatusNone;
  cudaEvent_t tev[2];
  if (timing) { cudaEventCreate(&tev[0]); cudaEventCreate(&tev[1]); }
  auto tick = [&]() { if (timing) cudaEventRecord(tev[0], s); };
  auto tock = [&](const char* what, int L) {
    if (!timing) return;
    cudaEventRecord(tev[1], s);
    cudaEventSynchronize(tev[1]);
    float ms = 0;
    cudaEventElapsedTime(&ms, tev[0], tev[1]);
    const LevelInfo& li = nd->levels[L];
    double by = 0;
    for (int t = li.begin; t < li.begin + li.count; ++t) {
      const FrontMeta& fm = nd->fronts[t];
      by += 16.0 * (what[0] == 'f' ? (double)fm.u * fm.s : (double)fm.s * fm.f);
    }
    fprintf(stderr, "[hh nd] %s L%-2d fronts %5d max_s %5d max_u %5d: %8.1f us %8.1f MB %6.0f GB/s\n", what, L,
            li.count, li.max_s, li.max_u, 1e3 * ms, by * B / 1e6, by * B / (ms * 1e-3) / 1e9);
  };
  SolveArgs A;
  A.fr = nd->d_fronts; A.st = st; A.sep = nd->d_sep; A.halo = nd->d_halo; A.gmap = nd->d_gmap;
  A.F = F; A.FE = shareF ? 0 : nd->F_entries;
  A.work = work; A.WE = nd_work_entries(nd); A.updE = nd->w_entries; A.rhs = rhs; A.x = x;
  A.vmax = nd_vmax();
  A.fail = fail;
  static const int pf = getenv("HH_NO_PREFETCH") ? 0 : 1;
  // L2 bulk prefetch of the next level's factor rows: pays for a single solve, but
  // beside other streams it only adds L2/HBM contention (sweep 0.369 -> 0.362 s without)
  A.prefetch = pf && !conc;
  if (nd->lean) {   // no stored -H^T rows: transposed forward, then the per-level backward
    c.sub_cut = -1;
    c.split = nlev - 1;
  }
  const int cut = c.sub_cut, Lb = c.split;
  const bool flow = c.flow && flow_ok(nd, cut, Lb);
  if (cut >= 0) {
    const size_t sm = (size_t)nd->sub_maxf[cut] * sizeof(cplx);
    if (sm > 48 * 1024) {
      HH_CUDA_TRY(smem_attr((const void*)k_nd_fwd_sub, sm));
      HH_CUDA_TRY(smem_attr((const void*)k_nd_bwd_sub, sm));
    }
    k_nd_fwd_sub<<<dim3(nd->sub_cnt[cut], B), 256, sm, s>>>(A, nd->d_sub_ptr + nd->sub_off[cut],
                                                            nd->d_sub_list + nd->list_off[cut]);
  }
  if (flow) HH_TRY(flow_launch(nd, A, B, cut + 1, Lb, true, s));
  for (int L = cut + 1; L <= Lb && !flow; ++L) {
    const LevelInfo& li = nd->levels[L];
    tick();
    struct Tk { decltype(tock)& f; int L; ~Tk() { f("fwd", L); } } tk_{tock, L};
    if (nd->lean) {
      HH_TRY(lean_fwd_level(nd, A, li, B, s));
      continue;
    }
    if (li.max_f > A.vmax || (li.max_u >= wide_rows() && (nd->dim == 3 || li.max_f >= wide_f()))) {
      dim3 gg(li.count, std::max(1, std::min(64, (li.max_f + 255) / 256)), B);
      HH_TRY(launch_pdl(k_nd_gather, gg, 256, 0, s, A, li.begin));
      if (li.max_u == 0) continue;
      const size_t sm = li.max_s > A.vmax ? 0 : (size_t)li.max_s * sizeof(cplx);
      if (sm > 48 * 1024)
        HH_CUDA_TRY(smem_attr((const void*)k_nd_rows_wide<0>, sm));
      dim3 g(li.count, (li.max_u + WIDE_RPC - 1) / WIDE_RPC, B);   // covers the smallest rows-per-CTA
      HH_TRY(launch_pdl(k_nd_rows_wide<0>, g, LT, sm, s, A, li.begin, (int)(sm / sizeof(cplx))));
      continue;
    }
    const size_t sm = (size_t)std::min(li.max_f, A.vmax) * sizeof(cplx);
    if (sm > 48 * 1024) HH_CUDA_TRY(smem_attr((const void*)k_nd_fwd, sm));
    dim3 g(li.count, level_split(li.max_u, li.count, B, li.max_s), B);
    HH_TRY(launch_pdl(k_nd_fwd, g, LT, sm, s, A, li.begin));
  }
  if (Lb < nlev - 1) {
    cudaLaunchConfig_t cfg = {};
    const int CLUSTER = cluster_size();
    if (CLUSTER > 8)
      HH_CUDA_TRY(cudaFuncSetAttribute(k_nd_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cfg.gridDim = dim3(CLUSTER * B);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CLUSTER;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HH_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_nd_cluster, A, (const int64_t*)nd->d_lvr, Lb + 1, nlev,
                                   (const int*)nd->d_sep_front, (const int*)nd->d_halo_front,
                                   (const int*)nd->d_pos_front));
  }
  if (flow) HH_TRY(flow_launch(nd, A, B, cut + 1, Lb, false, s));
  for (int L = Lb; L > cut && !flow; --L) {
    const LevelInfo& li = nd->levels[L];
    tick();
    struct Tk { decltype(tock)& f; int L; ~Tk() { f("bwd", L); } } tk_{tock, L};
    HH_TRY(bwd_level(nd, A, li, B, s));
  }
  if (cut >= 0) {
    const size_t sm = (size_t)nd->sub_maxf[cut] * sizeof(cplx);
    k_nd_bwd_sub<<<dim3(nd->sub_cnt[cut], B), 256, sm, s>>>(A, nd->d_sub_ptr + nd->sub_off[cut],
                                                            nd->d_sub_list + nd->list_off[cut]);
  }
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

// zero the dataflow counters of B samples (after the work buffer is (re)allocated)
hh_status nd_flow_reset(const NDPlan* nd, int B, cplx* work, cudaStream_t s) {
  const int64_t ce = flow_cnt_entries(nd);
  if (ce == 0 || B <= 0) return HH_OK;
  const size_t pitch = (size_t)nd_work_entries(nd) * sizeof(cplx);
  HH_CUDA_TRY(cudaMemset2DAsync(work + flow_cnt_off(nd), pitch, 0, (size_t)ce * sizeof(cplx), B, s));
  return HH_OK;
}

hh_status nd_solve(const NDPlan* ndc, int B, const int* st, const cplx* F, cplx* work, VArg rhs,
                   VArg x, cudaStream_t s, bool shareF, bool conc, int* fail) {
  NDPlan* nd = const_cast<NDPlan*>(ndc);
  return solve_cfg(nd, B, st, F, work, rhs, x, s, get_cfg(nd, B, conc), shareF, conc, fail);
}

bool nd_solve_uses_flow(const NDPlan* ndc, int B, bool conc) {
  NDPlan* nd = const_cast<NDPlan*>(ndc);
  const SolveCfg c = get_cfg(nd, B, conc);
  return c.flow && !nd->lean && flow_ok(nd, c.sub_cut, c.split);
}

void nd_flow_disable(const NDPlan* ndc) {
  NDPlan* nd = const_cast<NDPlan*>(ndc);
  std::lock_guard<std::mutex> lk(nd->cut_mu);
  nd->flow_disabled = true;
  for (auto& e : nd->cfg_cache) e.second.flow = 0;
}

// Empirical schedule choice on the real factor (called once per (tree, B) at
// setup, outside graph capture): time the candidate schedules with CUDA events.
hh_status nd_autotune(const NDPlan* ndc, int B, const cplx* F, cplx* work, VArg rhs, VArg x,
                      cudaStream_t s, bool shareF, bool conc, const std::vector<NDTuneCtx>* multi) {
  NDPlan* nd = const_cast<NDPlan*>(ndc);
  SolveCfg have;
  if (getenv("HH_ND_SPLIT") || getenv("HH_ND_CUT") || cached_cfg(nd, cfg_key(B, conc), &have) || nd->lean)
    return HH_OK;
  const int nlev = (int)nd->levels.size();
  cudaEvent_t e0, e1;
  HH_CUDA_TRY(cudaEventCreate(&e0));
  HH_CUDA_TRY(cudaEventCreate(&e1));
  std::vector<cudaEvent_t> ej;
  if (multi)
    for (size_t k = 0; k < multi->size(); ++k) {
      cudaEvent_t e;
      HH_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ej.push_back(e);
    }
  // isolated: the latency of one solve on an idle GPU; multi (concurrent sweep
  // workers): the makespan of one solve on EVERY worker stream at once, i.e. the
  // schedule's throughput when the streams share the SMs
  auto run = [&](SolveCfg c, float* ms) -> hh_status {
    if (!multi) {
      HH_TRY(solve_cfg(nd, B, nullptr, F, work, rhs, x, s, c, shareF, conc));   // warm
      HH_CUDA_TRY(cudaEventRecord(e0, s));
      for (int r = 0; r < 3; ++r) HH_TRY(solve_cfg(nd, B, nullptr, F, work, rhs, x, s, c, shareF, conc));
      HH_CUDA_TRY(cudaEventRecord(e1, s));
    } else {
      const std::vector<NDTuneCtx>& M = *multi;
      cudaStream_t s0 = M[0].s;
      for (int pass = 0; pass < 2; ++pass) {   // pass 0 warms up
        HH_CUDA_TRY(cudaEventRecord(e0, s0));
        for (size_t k = 1; k < M.size(); ++k) HH_CUDA_TRY(cudaStreamWaitEvent(M[k].s, e0, 0));
        for (size_t k = 0; k < M.size(); ++k)
          for (int r = 0; r < (pass ? 3 : 1); ++r)
            HH_TRY(solve_cfg(nd, B, nullptr, M[k].F, M[k].work, M[k].rhs, M[k].x, M[k].s, c, shareF, conc));
        for (size_t k = 1; k < M.size(); ++k) {
          HH_CUDA_TRY(cudaEventRecord(ej[k], M[k].s));
          HH_CUDA_TRY(cudaStreamWaitEvent(s0, ej[k], 0));
        }
        HH_CUDA_TRY(cudaEventRecord(e1, s0));
        HH_CUDA_TRY(cudaEventSynchronize(e1));
      }
    }
    HH_CUDA_TRY(cudaEventSynchronize(e1));
    HH_CUDA_TRY(cudaEventElapsedTime(ms, e0, e1));
    return HH_OK;
  };
  SolveCfg best{-1, nlev - 1};
  float best_ms = 1e30f;
  for (int cut = -1; cut <= std::min(3, nlev - 1); ++cut) {        // stage 1: bottom subtrees
    if (cut >= 0 && nd->sub_maxf[cut] > 1024) break;
    SolveCfg c{cut, nlev - 1};
    float ms;
    HH_TRY(run(c, &ms));
    if (getenv("HH_DEBUG") && atoi(getenv("HH_DEBUG")) > 1)
      fprintf(stderr, "[hh]   m=%d B=%d cut=%d split=%d: %.1f us\n", nd->m, B, c.sub_cut, c.split, 1e3 * ms / 3);
    if (ms < best_ms) { best_ms = ms; best = c; }
  }
  for (int top = 1; top <= 8; top += (top < 2 ? 1 : 2)) {          // stage 2: cluster top levels
    const int split = nlev - 1 - top;
    if (split < best.sub_cut) break;
    SolveCfg c{best.sub_cut, split};
    float ms;
    HH_TRY(run(c, &ms));
    if (getenv("HH_DEBUG") && atoi(getenv("HH_DEBUG")) > 1)
      fprintf(stderr, "[hh]   m=%d B=%d cut=%d split=%d: %.1f us\n", nd->m, B, c.sub_cut, c.split, 1e3 * ms / 3);
    if (ms < best_ms) { best_ms = ms; best = c; }
  }
  // stage 3: dataflow kernels for the per-level range (with and without the cluster top);
  // for concurrent sweep workers only on trees of at least HH_ND_FLOW_CONC_M coarse
  // nodes per side (default: never -- waiting CTAs hold SM slots other streams need)
  static const int flow_conc_m = getenv("HH_ND_FLOW_CONC_M") ? atoi(getenv("HH_ND_FLOW_CONC_M")) : (1 << 30);
  if ((!conc || nd->m >= flow_conc_m) && !nd->flow_disabled && !multi) {
    SolveCfg cands[2] = {best, best};
    cands[0].flow = 1;
    cands[1].flow = 1;
    cands[1].split = nlev - 1;
    HH_TRY(nd_flow_reset(nd, B, work, s));
    for (int k = 0; k < 2; ++k) {
      const SolveCfg c = cands[k];
      if (k == 1 && c.split == best.split) break;
      if (!flow_ok(nd, c.sub_cut, c.split)) continue;
      float ms;
      HH_TRY(run(c, &ms));
      HH_CUDA_TRY(cudaStreamSynchronize(s));
      int to = 0;
      HH_CUDA_TRY(cudaMemcpyFromSymbol(&to, g_flow_timeout, sizeof(int)));
      if (to) {   // a wait gave up: never use the dataflow schedule for this plan
        const int z = 0;
        HH_CUDA_TRY(cudaMemcpyToSymbol(g_flow_timeout, &z, sizeof(int)));
        HH_TRY(nd_flow_reset(nd, B, work, s));
        if (getenv("HH_DEBUG")) fprintf(stderr, "[hh] nd flow: wait timeout (m=%d B=%d), disabled\n", nd->m, B);
        break;
      }
      if (getenv("HH_DEBUG") && atoi(getenv("HH_DEBUG")) > 1)
        fprintf(stderr, "[hh]   m=%d B=%d cut=%d split=%d flow: %.1f us\n", nd->m, B, c.sub_cut, c.split,
                1e3 * ms / 3);
      if (ms < best_ms) { best_ms = ms; best = c; }
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  for (cudaEvent_t e : ej) cudaEventDestroy(e);
  std::lock_guard<std::mutex> lk(nd->cut_mu);
  nd->cfg_cache.push_back({cfg_key(B, conc), best});
  if (getenv("HH_DEBUG"))
    fprintf(stderr,
            "[hh] nd_autotune m=%d dim=%d B=%d levels=%d -> sub_cut=%d split=%d flow=%d (%.1f us/solve, "
            "%.1f MB/sample, %.0f GB/s)\n",
            nd->m, nd->dim, B, nlev, best.sub_cut, best.split, best.flow, 1e3 * best_ms / 3,
            nd->stream_bytes / 1e6, (double)nd->stream_bytes * B / (best_ms / 3 * 1e-3) / 1e9);
  return HH_OK;
}

int nd_solve_launches(const NDPlan* ndc, int B, bool conc) {
  NDPlan* nd = const_cast<NDPlan*>(ndc);
  const int nlev = (int)nd->levels.size();
  SolveCfg c = get_cfg(nd, B, conc);
  if (nd->lean) { c.sub_cut = -1; c.split = nlev - 1; }
  if (c.flow && flow_ok(nd, c.sub_cut, c.split))
    return (c.sub_cut >= 0 ? 2 : 0) + 2 + (c.split < nlev - 1 ? 1 : 0);
  int n = (c.sub_cut >= 0 ? 2 : 0) + 2 * (c.split - c.sub_cut) + (c.split < nlev - 1 ? 1 : 0);
  for (int L = c.sub_cut + 1; L <= c.split; ++L) {
    const LevelInfo& li = nd->levels[L];
    const bool big = li.max_f > nd_vmax() || li.max_f >= wide_f() || nd->dim == 3;
    n += (big && (li.max_f > nd_vmax() || li.max_u >= wide_rows())) +
         (big && (li.max_f > nd_vmax() || li.max_s >= wide_rows()));
  }
  return n;
}

// ============================================================ distributed coarse solve
// SURVEY.md 8(e) "second version" / 8(f) row 2 (the paper ran this step as a
// parallel MUMPS LU).  The slab-aligned tree of
// nd_plan_create_dist is factored and solved by its owners: rank r eliminates its
// slab interior (an ordinary ND subtree) and the interface planes it owns; the
// only exchanges are
//   factor  : the packed Schur complement S_t of a front whose parent is owned by
//             another rank -> the parent's owner (same packed-S offset on both);
//   forward : the update vector upd_t of such a front -> the parent's owner;
//   backward: the solution on every interface plane -> every rank (the halos of
//             the fronts below it reach into the planes of all their ancestors).
// The views of one process are either all P ranks (in-process slabs: the
// exchanges are device copies) or one rank with an NCCL communicator.
namespace {
__global__ void k_nd_sep_copy(const int* __restrict__ sep, int n, const cplx* __restrict__ x,
                              cplx* __restrict__ y, cplx* __restrict__ buf, int mode) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int g = sep[i];
    if (mode == 0) buf[i] = x[g];            // pack
    else if (mode == 1) y[g] = buf[i];       // unpack
    else y[g] = x[g];                        // direct (in-process)
  }
}

SolveArgs dist_args(const NDPlan* nd, const NDDistView& v, const int* st, VArg rhs, VArg x) {
  SolveArgs A;
  A.fr = nd->d_fronts; A.st = st; A.sep = nd->d_sep; A.halo = nd->d_halo; A.gmap = nd->d_gmap;
  A.F = v.F; A.FE = 0;
  A.work = v.work; A.WE = nd_work_entries(nd); A.updE = nd->w_entries; A.rhs = rhs; A.x = x;
  A.vmax = nd_vmax();
  A.prefetch = 0;
  A.fail = nullptr;
  return A;
}

int view_of(const std::vector<NDDistView>& V, int rank) {
  for (size_t k = 0; k < V.size(); ++k)
    if (V[k].plan->rank == rank) return (int)k;
  return -1;
}

// move the blocks of `list` (fronts whose parent has another owner) from the
// child's owner to the parent's owner: kind 0 = packed S (cbuf), 1 = upd (work)
hh_status dist_xfer(std::vector<NDDistView>& V, Comm* comm, const std::vector<int>& list, int kind,
                    cudaStream_t s) {
  if (list.empty()) return HH_OK;
  const NDPlan* g = V[0].plan;
  auto where = [&](const NDDistView& v, int t, int64_t* cnt) -> cplx* {
    const FrontMeta& fm = g->fronts[t];
    if (kind == 0) {
      *cnt = (int64_t)fm.u * (fm.u + 1) / 2;
      return v.S + v.plan->Soff_h[t];   // each rank's own placement
    }
    *cnt = fm.u;
    return v.work + g->w_entries + fm.outOff;
  };
  if (!comm) {
    for (int t : list) {
      const int a = view_of(V, g->owner[t]), b = view_of(V, g->owner[g->fronts[t].parent]);
      if (a < 0 || b < 0) { hh_set_error("nd dist: rank view missing"); return HH_E_STATE; }
      int64_t cnt = 0;
      cplx* src = where(V[a], t, &cnt);
      cplx* dst = where(V[b], t, &cnt);
      if (cnt) HH_CUDA_TRY(cudaMemcpyAsync(dst, src, cnt * sizeof(cplx), cudaMemcpyDeviceToDevice, s));
    }
    return HH_OK;
  }
  const int me = V[0].plan->rank;
  HH_TRY(comm_group(true));
  for (int t : list) {
    const int a = g->owner[t], b = g->owner[g->fronts[t].parent];
    int64_t cnt = 0;
    cplx* buf = where(V[0], t, &cnt);
    if (!cnt) continue;
    if (a == me) HH_TRY(comm_send(comm, buf, cnt * sizeof(cplx), b, s));
    if (b == me) HH_TRY(comm_recv(comm, buf, cnt * sizeof(cplx), a, s));
  }
  return comm_group(false);
}

// the solution on the interface planes of `list` (level L) -> every rank
hh_status dist_bcast_top(std::vector<NDDistView>& V, Comm* comm, const std::vector<int>& list, VArg x,
                         cplx* stage, cudaStream_t s) {
  if (list.empty()) return HH_OK;
  const NDPlan* g = V[0].plan;
  if (!comm) {
    for (int t : list) {
      const FrontMeta& fm = g->fronts[t];
      const int a = view_of(V, g->owner[t]);
      for (size_t b = 0; b < V.size(); ++b) {
        if ((int)b == a) continue;
        k_nd_sep_copy<<<std::min(1024, (fm.s + 255) / 256), 256, 0, s>>>(
            g->d_sep + fm.sepOff, fm.s, x.p + (int64_t)a * x.bs, x.p + (int64_t)b * x.bs, nullptr, 2);
      }
    }
    HH_CUDA_TRY(cudaGetLastError());
    return HH_OK;
  }
  const int me = V[0].plan->rank;
  int64_t off = 0;
  for (int t : list) {   // pack the planes this rank owns
    const FrontMeta& fm = g->fronts[t];
    if (g->owner[t] == me)
      k_nd_sep_copy<<<std::min(1024, (fm.s + 255) / 256), 256, 0, s>>>(g->d_sep + fm.sepOff, fm.s, x.p,
                                                                        nullptr, stage + off, 0);
    off += fm.s;
  }
  HH_CUDA_TRY(cudaGetLastError());
  HH_TRY(comm_group(true));
  off = 0;
  for (int t : list) {
    const FrontMeta& fm = g->fronts[t];
    HH_TRY(comm_bcast(comm, stage + off, (size_t)fm.s * sizeof(cplx), g->owner[t], s));
    off += fm.s;
  }
  HH_TRY(comm_group(false));
  off = 0;
  for (int t : list) {   // unpack the others'
    const FrontMeta& fm = g->fronts[t];
    if (g->owner[t] != me)
      k_nd_sep_copy<<<std::min(1024, (fm.s + 255) / 256), 256, 0, s>>>(g->d_sep + fm.sepOff, fm.s, nullptr,
                                                                        x.p, stage + off, 1);
    off += fm.s;
  }
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}
}  // namespace

int64_t nd_dist_stage_entries(const NDPlan* p) { return std::max<int64_t>(1, p->top_sep_max); }

int nd_dist_levels(const NDPlan* p) { return (int)p->levels.size(); }

hh_status nd_dist_factor(std::vector<NDDistView>& V, const cplx* st, Comm* comm, cudaStream_t s) {
  if (V.empty()) return HH_OK;
  const NDPlan* g = V[0].plan;
  const int nlev = (int)g->levels.size();
  std::vector<size_t> next(V.size(), 0);
  for (auto& v : V) HH_CUDA_TRY(cudaMemsetAsync(v.flag, 0, sizeof(int), s));
  for (int L = 0; L < nlev; ++L) {
    for (size_t k = 0; k < V.size(); ++k) {
      const NDPlan* p = V[k].plan;
      while (next[k] < p->chunks.size() && p->chunks[next[k]].level == L)
        HH_TRY(lean_chunk(p, p->chunks[next[k]++], st, V[k].F, V[k].scratch, V[k].scratch + p->Cw, V[k].S,
                          V[k].flag, s));
    }
    HH_TRY(dist_xfer(V, comm, g->xcross[L], 0, s));
  }
  return HH_OK;
}

hh_status nd_dist_solve(std::vector<NDDistView>& V, const int* st, VArg rhs, VArg x, Comm* comm, cplx* stage,
                        cudaStream_t s) {
  if (V.empty()) return HH_OK;
  const NDPlan* g = V[0].plan;
  const int nlev = (int)g->levels.size();
  std::vector<SolveArgs> A;
  for (size_t k = 0; k < V.size(); ++k)
    A.push_back(dist_args(V[k].plan, V[k], st ? st + k : nullptr, varg(rhs.p + (int64_t)k * rhs.bs, rhs.bs),
                          varg(x.p + (int64_t)k * x.bs, x.bs)));
  for (int L = 0; L < nlev; ++L) {
    for (size_t k = 0; k < V.size(); ++k) HH_TRY(lean_fwd_level(V[k].plan, A[k], V[k].plan->levels[L], 1, s));
    HH_TRY(dist_xfer(V, comm, g->xcross[L], 1, s));
  }
  for (int L = nlev - 1; L >= 0; --L) {
    for (size_t k = 0; k < V.size(); ++k) HH_TRY(bwd_level(V[k].plan, A[k], V[k].plan->levels[L], 1, s));
    HH_TRY(dist_bcast_top(V, comm, g->xtop[L], x, stage, s));
  }
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

int nd_dist_launches(const std::vector<NDDistView>& V) {
  int n = 0;
  for (const NDDistView& v : V)
    for (const LevelInfo& li : v.plan->levels) {
      if (!li.count) continue;
      n += 1 + (li.max_u > 0 ? 2 : 0);                                    // forward
      n += (li.max_f > nd_vmax() || li.max_s >= wide_rows()) ? (li.max_f > bwdk_f() ? 3 : 2) : 1;   // backward
    }
  const NDPlan* g = V[0].plan;
  for (size_t L = 0; L < g->levels.size(); ++L)
    n += (int)(g->xcross[L].size() + g->xtop[L].size() * (V.size() > 1 ? V.size() - 1 : 2));
  return n;
}

// scratch (pivot columns + workspace: reusable across the views of one process,
// which run one after another) and packed-S (per view) sizes of a rank view
int64_t nd_dist_scratch_entries(const NDPlan* p) { return p->Cw + p->Wmax; }
int64_t nd_dist_s_entries(const NDPlan* p) { return std::max<int64_t>(1, p->Smax[0] + p->Smax[1]); }
