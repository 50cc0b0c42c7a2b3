// Coarse-grid direct solver for A_eps^{(1)} (Alg. 1 line 3, PAPER.md:374;
// factor once, reuse every V-cycle: PAPER.md:511-512).
//
// B200 design (differs from the paper's MUMPS LU):
//  * geometric nested dissection of the structured (m)^d coarse node grid:
//    recursive bisection of boxes by a separator line/plane; leaves <= 64 nodes.
//    Front(t) = sep(t) (eliminated at t) + halo(t) (1-ring of box(t), clipped).
//  * multifrontal elimination WITHOUT pivoting (reading C18: the Hermitian part
//    of i*A_eps is eps*M + k*B, positive definite for eps > 0, so every
//    principal submatrix is non-singular), all fronts of one tree level in one
//    batched launch.  Each front is "swept" on its separator block by partial
//    Gauss-Jordan (block size NB): afterwards the dense front holds
//        [ X = F_ss^{-1}      H = F_ss^{-1} F_su ]
//        [ -H^T               S = F_uu - F_us X F_su ]
//    and S is extend-added into the parent front.
//  * solve = two sweeps of batched GEMVs over the stored blocks (explicit
//    inverses, no triangular recurrences):
//        forward (leaves -> root):  z_s = r[sep] + sum_children-of-halo contributions,
//                                   contribution_t = -H^T z_s  (gathered, no atomics)
//        backward (root -> leaves): x[sep] = X z_s - H x[halo]
//    Bytes streamed per solve ~ 16 * sum_t (s_t f_t + u_t s_t), the same as a
//    triangular LDL^T solve; every launch is fully parallel.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <unordered_map>
#include "hh_internal.cuh"

namespace {
constexpr int NB = 16;      // pivot block of the partial Gauss-Jordan sweep
constexpr int LEAF = 64;    // max nodes of a leaf box

struct FrontMeta {          // device-visible per-front data
  int s, u, f, level;
  int64_t Foff;             // offset (complex entries) of the f x f front
  int64_t sepOff, haloOff;  // into sep / halo index arrays
  int64_t zsOff, outOff;    // into the solve work vectors
  int64_t gptrOff;          // into gptr (s+1 entries)
  int64_t eaOff;            // into extend-add map (u entries)
  int parent;
  int pad;
};

struct LevelInfo {
  int begin, count;         // fronts [begin, begin+count)
  int max_s, max_u, max_f;
  int64_t asmBegin, asmCount;       // assembly entries
  int ea_count[2];                   // children per slot
  int64_t ea_list_off[2];            // offsets into eaList
};
}  // namespace

struct NDFactor {
  int dim = 2, m = 0;            // coarse grid nodes per side
  int64_t N = 0;                 // coarse nodes
  std::vector<FrontMeta> fronts; // host copy
  std::vector<LevelInfo> levels;
  FrontMeta* d_fronts = nullptr;
  int* d_sep = nullptr;
  int* d_halo = nullptr;
  int4* d_asm = nullptr;         // (front, a, b, stencil index)
  int* d_eamap = nullptr;        // child halo pos -> parent front pos
  int* d_eaList = nullptr;       // child front ids grouped by (level, slot)
  int64_t* d_gptr = nullptr;     // CSR over all separator entries
  int64_t* d_gidx = nullptr;     // index into out buffer
  cplx* d_F = nullptr;           // all fronts
  cplx* d_C = nullptr;           // saved column block (per level, f x NB per front)
  int64_t* d_Coff = nullptr;     // per front offset into d_C (level-local)
  cplx* d_zs = nullptr;          // forward solve values per separator entry
  cplx* d_out = nullptr;         // forward contributions per halo entry
  int* d_flag = nullptr;         // zero-pivot flag
  int64_t F_entries = 0, zs_entries = 0, out_entries = 0;
  int64_t stream_bytes = 0;
};

// ============================================================ device kernels
namespace {

__global__ void k_nd_assemble(const int4* __restrict__ e, int64_t cnt,
                              const FrontMeta* __restrict__ fr, const cplx* __restrict__ st,
                              cplx* __restrict__ F) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  const int4 v = e[i];
  const FrontMeta m = fr[v.x];
  F[m.Foff + (int64_t)v.y * m.f + v.z] = st[v.w];
}

// extend-add of the child update matrices S_c into the parents (one child per parent per launch)
__global__ void k_nd_extend_add(const int* __restrict__ list, const FrontMeta* __restrict__ fr,
                                const int* __restrict__ eamap, cplx* __restrict__ F) {
  const int c = list[blockIdx.x];
  const FrontMeta mc = fr[c];
  const FrontMeta mp = fr[mc.parent];
  const int* map = eamap + mc.eaOff;
  for (int a = blockIdx.y; a < mc.u; a += gridDim.y) {
    const cplx* src = F + mc.Foff + (int64_t)(mc.s + a) * mc.f + mc.s;
    cplx* dst = F + mp.Foff + (int64_t)map[a] * mp.f;
    for (int b = threadIdx.x; b < mc.u; b += blockDim.x) {
      cplx v = src[b];
      cplx& d = dst[map[b]];
      d.x += v.x;
      d.y += v.y;
    }
  }
}

// pivot step: P = F[K,K]^{-1}; save column block C = F[:,K]; rows K <- P F[K,:], F[K,K] <- P
__global__ void __launch_bounds__(256) k_nd_piv(const FrontMeta* __restrict__ fr, int begin,
                                                int kb, cplx* __restrict__ F,
                                                cplx* __restrict__ Cbuf,
                                                const int64_t* __restrict__ Coff,
                                                int* __restrict__ flag) {
  const int t = begin + blockIdx.x;
  const FrontMeta m = fr[t];
  if (kb >= m.s) return;
  const int nb = min(NB, m.s - kb);
  const int f = m.f;
  cplx* A = F + m.Foff;
  cplx* C = Cbuf + Coff[blockIdx.x];
  __shared__ cplx P[NB][NB + 1];
  const int ti = threadIdx.x / NB, tj = threadIdx.x % NB;   // 16 x 16
  if (ti < nb && tj < nb) P[ti][tj] = A[(int64_t)(kb + ti) * f + kb + tj];
  // save column block (rows outside K only are used later)
  for (int idx = threadIdx.x; idx < f * nb; idx += blockDim.x) {
    const int i = idx / nb, k = idx % nb;
    C[(int64_t)i * NB + k] = A[(int64_t)i * f + kb + k];
  }
  __syncthreads();
  // in-place Gauss-Jordan inversion of the nb x nb pivot block (sweep operator)
  for (int p = 0; p < nb; ++p) {
    const cplx piv = P[p][p];
    if (cabs2(piv) == 0.0) {
      if (threadIdx.x == 0) atomicExch(flag, 1);
    }
    const cplx pinv = cinv(piv);
    __syncthreads();
    cplx rowp = (ti == p && tj < nb && tj != p) ? cmul(P[p][tj], pinv) : cmake(0, 0);
    __syncthreads();
    if (ti == p && tj < nb && tj != p) P[p][tj] = rowp;
    __syncthreads();
    cplx newv = cmake(0, 0);
    bool wr = false;
    if (ti < nb && tj < nb && ti != p) {
      const cplx fac = P[ti][p];
      if (tj != p) {
        newv = P[ti][tj];
        cfms(newv, fac, P[p][tj]);
      } else {
        newv = cmul(fac, pinv);
        newv.x = -newv.x; newv.y = -newv.y;
      }
      wr = true;
    }
    __syncthreads();
    if (wr) P[ti][tj] = newv;
    if (threadIdx.x == 0) P[p][p] = pinv;
    __syncthreads();
  }
  // rows K: R[k][j] = sum_l P[k][l] A[kb+l][j] for j not in K; P for j in K
  for (int j = threadIdx.x; j < f; j += blockDim.x) {
    if (j >= kb && j < kb + nb) {
      for (int k = 0; k < nb; ++k) A[(int64_t)(kb + k) * f + j] = P[k][j - kb];
      continue;
    }
    cplx col[NB];
#pragma unroll
    for (int l = 0; l < NB; ++l) col[l] = (l < nb) ? A[(int64_t)(kb + l) * f + j] : cmake(0, 0);
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      if (k >= nb) break;
      cplx acc = cmake(0, 0);
#pragma unroll
      for (int l = 0; l < NB; ++l)
        if (l < nb) cfma(acc, P[k][l], col[l]);
      A[(int64_t)(kb + k) * f + j] = acc;
    }
  }
}

// rank-nb update of all rows outside K:
//   F[i][j] <- (j in K ? 0 : F[i][j]) - sum_k C[i][k] * F[kb+k][j]
constexpr int UT = 32;   // update tile (UT x UT outputs per CTA, 256 threads)
__global__ void __launch_bounds__(256) k_nd_upd(const FrontMeta* __restrict__ fr, int begin,
                                                int kb, cplx* __restrict__ F,
                                                const cplx* __restrict__ Cbuf,
                                                const int64_t* __restrict__ Coff) {
  const int t = begin + blockIdx.z;
  const FrontMeta m = fr[t];
  if (kb >= m.s) return;
  const int f = m.f;
  const int i0 = blockIdx.y * UT, j0 = blockIdx.x * UT;
  if (i0 >= f || j0 >= f) return;
  const int nb = min(NB, m.s - kb);
  cplx* A = F + m.Foff;
  const cplx* C = Cbuf + Coff[blockIdx.z];
  __shared__ cplx Cs[UT][NB + 1];
  __shared__ cplx Rs[NB][UT + 1];
  for (int idx = threadIdx.x; idx < UT * NB; idx += 256) {
    const int i = idx / NB, k = idx % NB;
    Cs[i][k] = (i0 + i < f && k < nb) ? C[(int64_t)(i0 + i) * NB + k] : cmake(0, 0);
  }
  for (int idx = threadIdx.x; idx < NB * UT; idx += 256) {
    const int k = idx / UT, j = idx % UT;
    Rs[k][j] = (k < nb && j0 + j < f) ? A[(int64_t)(kb + k) * f + j0 + j] : cmake(0, 0);
  }
  __syncthreads();
  const int tx = threadIdx.x % UT, ty = threadIdx.x / UT;   // 32 x 8
  const int j = j0 + tx;
  if (j >= f) return;
  const bool jK = (j >= kb && j < kb + nb);
#pragma unroll
  for (int r = 0; r < UT / 8; ++r) {
    const int il = ty + 8 * r;
    const int i = i0 + il;
    if (i >= f || (i >= kb && i < kb + nb)) continue;
    cplx acc = jK ? cmake(0, 0) : A[(int64_t)i * f + j];
#pragma unroll
    for (int k = 0; k < NB; ++k) cfms(acc, Cs[il][k], Rs[k][tx]);
    A[(int64_t)i * f + j] = acc;
  }
}

// forward: gather z_s = r[sep] + sum of descendant contributions
__global__ void k_nd_gather(const FrontMeta* __restrict__ fr, int begin,
                            const int* __restrict__ sep, const int64_t* __restrict__ gptr,
                            const int64_t* __restrict__ gidx, const cplx* __restrict__ rhs,
                            const cplx* __restrict__ out, cplx* __restrict__ zs) {
  const FrontMeta m = fr[begin + blockIdx.x];
  for (int a = threadIdx.x + blockIdx.y * blockDim.x; a < m.s; a += blockDim.x * gridDim.y) {
    cplx v = rhs[sep[m.sepOff + a]];
    const int64_t p0 = gptr[m.gptrOff + a], p1 = gptr[m.gptrOff + a + 1];
    for (int64_t p = p0; p < p1; ++p) {
      const cplx c = out[gidx[p]];
      v.x += c.x;
      v.y += c.y;
    }
    zs[m.zsOff + a] = v;
  }
}

// warp-per-row GEMV helpers
__device__ __forceinline__ cplx warp_sum(cplx v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// forward contributions out[b] = sum_a F[s+b][a] zs[a]   (F[u][s] = -H^T)
__global__ void __launch_bounds__(256) k_nd_fwd(const FrontMeta* __restrict__ fr, int begin,
                                                const cplx* __restrict__ F,
                                                const cplx* __restrict__ zs,
                                                cplx* __restrict__ out) {
  const FrontMeta m = fr[begin + blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const cplx* z = zs + m.zsOff;
  for (int b = blockIdx.y * 8 + warp; b < m.u; b += gridDim.y * 8) {
    const cplx* row = F + m.Foff + (int64_t)(m.s + b) * m.f;
    cplx acc = cmake(0, 0);
    for (int a = lane; a < m.s; a += 32) cfma(acc, row[a], z[a]);
    acc = warp_sum(acc);
    if (lane == 0) out[m.outOff + b] = acc;
  }
}

// backward: x[sep[a]] = sum_b F[a][b] v[b],  v = [z_s ; -x[halo]]
__global__ void __launch_bounds__(256) k_nd_bwd(const FrontMeta* __restrict__ fr, int begin,
                                                const cplx* __restrict__ F,
                                                const cplx* __restrict__ zs,
                                                const int* __restrict__ sep,
                                                const int* __restrict__ halo,
                                                cplx* __restrict__ x) {
  const FrontMeta m = fr[begin + blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const cplx* z = zs + m.zsOff;
  const int* hl = halo + m.haloOff;
  for (int a = blockIdx.y * 8 + warp; a < m.s; a += gridDim.y * 8) {
    const cplx* row = F + m.Foff + (int64_t)a * m.f;
    cplx acc = cmake(0, 0);
    for (int b = lane; b < m.s; b += 32) cfma(acc, row[b], z[b]);
    for (int b = lane; b < m.u; b += 32) cfms(acc, row[m.s + b], x[hl[b]]);
    acc = warp_sum(acc);
    if (lane == 0) x[sep[m.sepOff + a]] = acc;
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
};

int64_t box_count(const Box& b, int dim) {
  int64_t c = 1;
  for (int d = 0; d < dim; ++d) c *= (b.hi[d] - b.lo[d]);
  return c;
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
  const int64_t cnt = box_count(b, dim);
  auto idx = [&](const int* c) {
    int64_t g = 0, st = 1;
    for (int d = 0; d < dim; ++d) { g += c[d] * st; st *= m; }
    return (int)g;
  };
  if (cnt <= LEAF || ext < 3) {
    // leaf: all nodes, lexicographic
    int c[3] = {0, 0, 0};
    for (c[2] = (dim > 2 ? b.lo[2] : 0); c[2] < (dim > 2 ? b.hi[2] : 1); ++c[2])
      for (c[1] = b.lo[1]; c[1] < b.hi[1]; ++c[1])
        for (c[0] = b.lo[0]; c[0] < b.hi[0]; ++c[0]) out[id].sep.push_back(idx(c));
    return;
  }
  const int mid = (b.lo[ax] + b.hi[ax]) / 2;
  Box s = b; s.lo[ax] = mid; s.hi[ax] = mid + 1;
  {
    int c[3] = {0, 0, 0};
    for (c[2] = (dim > 2 ? s.lo[2] : 0); c[2] < (dim > 2 ? s.hi[2] : 1); ++c[2])
      for (c[1] = s.lo[1]; c[1] < s.hi[1]; ++c[1])
        for (c[0] = s.lo[0]; c[0] < s.hi[0]; ++c[0]) out[id].sep.push_back(idx(c));
  }
  Box l = b; l.hi[ax] = mid;
  Box r = b; r.lo[ax] = mid + 1;
  const int lid = (int)out.size();
  build_tree(l, dim, m, id, out);
  out[id].children.push_back(lid);
  const int rid = (int)out.size();
  build_tree(r, dim, m, id, out);
  out[id].children.push_back(rid);
}

}  // namespace

// ============================================================ host API
hh_status nd_create(const Level& C, NDFactor** out, cudaStream_t s) {
  (void)s;
  NDFactor* nd = new NDFactor();
  const int dim = C.dim, m = C.n + 1;
  nd->dim = dim; nd->m = m; nd->N = C.nodes;
  std::vector<HostFront> tf;
  Box root;
  for (int d = 0; d < 3; ++d) { root.lo[d] = 0; root.hi[d] = (d < dim) ? m : 1; }
  build_tree(root, dim, m, -1, tf);
  const int nf = (int)tf.size();
  // halo rings + levels (height)
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
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tf[a].level < tf[b].level; });
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
  int64_t Foff = 0, zsOff = 0, outOff = 0, eaOff = 0;
  const int S = (dim == 2) ? 9 : 27;
  std::vector<int> loc(nd->N, -1);
  // assembly entries grouped per level: collect per front then concatenate (fronts ordered by level)
  for (int i = 0; i < nf; ++i) {
    const HostFront& h = tf[order[i]];
    FrontMeta& fm = nd->fronts[i];
    fm.s = (int)h.sep.size(); fm.u = (int)h.halo.size(); fm.f = fm.s + fm.u; fm.level = h.level;
    fm.Foff = Foff; Foff += (int64_t)fm.f * fm.f;
    fm.sepOff = (int64_t)sepAll.size(); sepAll.insert(sepAll.end(), h.sep.begin(), h.sep.end());
    fm.haloOff = (int64_t)haloAll.size(); haloAll.insert(haloAll.end(), h.halo.begin(), h.halo.end());
    fm.zsOff = zsOff; zsOff += fm.s;
    fm.outOff = outOff; outOff += fm.u;
    fm.parent = h.parent >= 0 ? newid[h.parent] : -1;
    // local map
    for (int a = 0; a < fm.s; ++a) loc[h.sep[a]] = a;
    for (int b = 0; b < fm.u; ++b) loc[h.halo[b]] = fm.s + b;
    for (int a = 0; a < fm.s; ++a) {
      const int g = h.sep[a];
      int c[3] = {0, 0, 0};
      int64_t r = g;
      for (int d = 0; d < dim; ++d) { c[d] = (int)(r % m); r /= m; }
      for (int o = 0; o < S; ++o) {
        int nb[3] = {0, 0, 0};
        bool ok = true;
        int oo = o;
        int64_t gj = 0, st = 1;
        for (int d = 0; d < dim; ++d) {
          const int dd = oo % 3 - 1; oo /= 3;
          nb[d] = c[d] + dd;
          ok = ok && nb[d] >= 0 && nb[d] < m;
          gj += nb[d] * st; st *= m;
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
  // gather CSR: for every separator entry (front t, a): contributions (front d, halo pos b)
  std::vector<std::vector<int64_t>> contrib(sepAll.size());
  for (int d = 0; d < nf; ++d) {
    const FrontMeta& fm = nd->fronts[d];
    const HostFront& h = tf[order[d]];
    for (int b = 0; b < fm.u; ++b) {
      const int g = h.halo[b];
      const int t = owner[g];
      contrib[nd->fronts[t].sepOff + ownpos[g]].push_back(fm.outOff + b);
    }
  }
  std::vector<int64_t> gptr(sepAll.size() + 1, 0), gidx;
  for (size_t e = 0; e < sepAll.size(); ++e) {
    gptr[e + 1] = gptr[e] + (int64_t)contrib[e].size();
    gidx.insert(gidx.end(), contrib[e].begin(), contrib[e].end());
  }
  for (int i = 0; i < nf; ++i) nd->fronts[i].gptrOff = nd->fronts[i].sepOff;   // gptr indexed per sep entry
  // levels
  nd->levels.resize(nlev);
  {
    int i = 0;
    int64_t ai = 0;
    std::vector<int> eaList;
    for (int L = 0; L < nlev; ++L) {
      LevelInfo& li = nd->levels[L];
      li.begin = i; li.count = 0; li.max_s = li.max_u = li.max_f = 0;
      while (i < nf && nd->fronts[i].level == L) {
        li.max_s = std::max(li.max_s, nd->fronts[i].s);
        li.max_u = std::max(li.max_u, nd->fronts[i].u);
        li.max_f = std::max(li.max_f, nd->fronts[i].f);
        ++li.count; ++i;
      }
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
    HH_CUDA_TRY(cudaMalloc(&nd->d_eaList, std::max<size_t>(1, eaList.size()) * sizeof(int)));
    HH_CUDA_TRY(cudaMemcpy(nd->d_eaList, eaList.data(), eaList.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  // C buffer offsets (level-local)
  int64_t Cmax = 0;
  std::vector<int64_t> Coff(nf);
  for (auto& li : nd->levels) {
    int64_t o = 0;
    for (int t = li.begin; t < li.begin + li.count; ++t) { Coff[t - li.begin + li.begin] = o; o += (int64_t)nd->fronts[t].f * NB; }
    Cmax = std::max(Cmax, o);
  }
  // device Coff array indexed by blockIdx (level-local): store per front, pass pointer at level begin
  nd->F_entries = Foff; nd->zs_entries = zsOff; nd->out_entries = outOff;
  int64_t sb = 0;
  for (auto& fm : nd->fronts) sb += (int64_t)fm.s * fm.f + (int64_t)fm.u * fm.s;
  nd->stream_bytes = sb * (int64_t)sizeof(cplx);

  auto up = [&](auto** dptr, const auto& vec) -> hh_status {
    using T = typename std::remove_reference<decltype(vec)>::type::value_type;
    const size_t bytes = std::max<size_t>(1, vec.size()) * sizeof(T);
    if (cudaMalloc((void**)dptr, bytes) != cudaSuccess) { hh_set_error("nd: cudaMalloc %zu B failed", bytes); return HH_E_OOM; }
    if (!vec.empty()) HH_CUDA_TRY(cudaMemcpy(*dptr, vec.data(), vec.size() * sizeof(T), cudaMemcpyHostToDevice));
    return HH_OK;
  };
  HH_TRY(up(&nd->d_fronts, nd->fronts));
  HH_TRY(up(&nd->d_sep, sepAll));
  HH_TRY(up(&nd->d_halo, haloAll));
  HH_TRY(up(&nd->d_asm, asmE));
  HH_TRY(up(&nd->d_eamap, eamap));
  HH_TRY(up(&nd->d_gptr, gptr));
  HH_TRY(up(&nd->d_gidx, gidx));
  HH_TRY(up(&nd->d_Coff, Coff));
  if (cudaMalloc(&nd->d_F, std::max<int64_t>(1, Foff) * sizeof(cplx)) != cudaSuccess) {
    hh_set_error("nd: cannot allocate %.3f GB of fronts", Foff * 16.0 / 1e9);
    return HH_E_OOM;
  }
  if (cudaMalloc(&nd->d_C, std::max<int64_t>(1, Cmax) * sizeof(cplx)) != cudaSuccess) return HH_E_OOM;
  HH_CUDA_TRY(cudaMalloc(&nd->d_zs, std::max<int64_t>(1, zsOff) * sizeof(cplx)));
  HH_CUDA_TRY(cudaMalloc(&nd->d_out, std::max<int64_t>(1, outOff) * sizeof(cplx)));
  HH_CUDA_TRY(cudaMalloc(&nd->d_flag, sizeof(int)));
  *out = nd;
  return HH_OK;
}

hh_status nd_factor(NDFactor* nd, const cplx* st, cudaStream_t s) {
  HH_CUDA_TRY(cudaMemsetAsync(nd->d_flag, 0, sizeof(int), s));
  for (size_t L = 0; L < nd->levels.size(); ++L) {
    const LevelInfo& li = nd->levels[L];
    const FrontMeta& f0 = nd->fronts[li.begin];
    const FrontMeta& fl = nd->fronts[li.begin + li.count - 1];
    const int64_t lvEntries = fl.Foff + (int64_t)fl.f * fl.f - f0.Foff;
    HH_CUDA_TRY(cudaMemsetAsync(nd->d_F + f0.Foff, 0, lvEntries * sizeof(cplx), s));
    if (li.asmCount) {
      const int bs = 256;
      k_nd_assemble<<<(unsigned)((li.asmCount + bs - 1) / bs), bs, 0, s>>>(
          nd->d_asm + li.asmBegin, li.asmCount, nd->d_fronts, st, nd->d_F);
    }
    for (int slot = 0; slot < 2; ++slot) {
      if (!li.ea_count[slot]) continue;
      dim3 g(li.ea_count[slot], std::min(64, std::max(1, nd->levels[0].max_u)));
      k_nd_extend_add<<<g, 128, 0, s>>>(nd->d_eaList + li.ea_list_off[slot], nd->d_fronts,
                                        nd->d_eamap, nd->d_F);
    }
    for (int kb = 0; kb < li.max_s; kb += NB) {
      k_nd_piv<<<li.count, 256, 0, s>>>(nd->d_fronts, li.begin, kb, nd->d_F, nd->d_C,
                                        nd->d_Coff + li.begin, nd->d_flag);
      const int tiles = (li.max_f + UT - 1) / UT;
      dim3 g(tiles, tiles, li.count);
      k_nd_upd<<<g, 256, 0, s>>>(nd->d_fronts, li.begin, kb, nd->d_F, nd->d_C,
                                 nd->d_Coff + li.begin);
    }
    HH_CUDA_TRY(cudaGetLastError());
  }
  int flag = 0;
  HH_CUDA_TRY(cudaMemcpyAsync(&flag, nd->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  HH_CUDA_TRY(cudaStreamSynchronize(s));
  if (flag) { hh_set_error("nd: zero pivot in the coarse factorisation"); return HH_E_SINGULAR; }
  return HH_OK;
}

hh_status nd_solve(NDFactor* nd, const cplx* rhs, cplx* x, cudaStream_t s) {
  const int nlev = (int)nd->levels.size();
  for (int L = 0; L < nlev; ++L) {
    const LevelInfo& li = nd->levels[L];
    dim3 gg(li.count, std::max(1, std::min(32, (li.max_s + 255) / 256)));
    k_nd_gather<<<gg, 256, 0, s>>>(nd->d_fronts, li.begin, nd->d_sep, nd->d_gptr, nd->d_gidx,
                                   rhs, nd->d_out, nd->d_zs);
    if (li.max_u > 0) {
      dim3 g(li.count, std::max(1, std::min(1024, (li.max_u + 7) / 8)));
      k_nd_fwd<<<g, 256, 0, s>>>(nd->d_fronts, li.begin, nd->d_F, nd->d_zs, nd->d_out);
    }
  }
  for (int L = nlev - 1; L >= 0; --L) {
    const LevelInfo& li = nd->levels[L];
    dim3 g(li.count, std::max(1, std::min(1024, (li.max_s + 7) / 8)));
    k_nd_bwd<<<g, 256, 0, s>>>(nd->d_fronts, li.begin, nd->d_F, nd->d_zs, nd->d_sep, nd->d_halo, x);
  }
  HH_CUDA_TRY(cudaGetLastError());
  return HH_OK;
}

void nd_destroy(NDFactor* nd) {
  if (!nd) return;
  cudaFree(nd->d_fronts); cudaFree(nd->d_sep); cudaFree(nd->d_halo); cudaFree(nd->d_asm);
  cudaFree(nd->d_eamap); cudaFree(nd->d_eaList); cudaFree(nd->d_gptr); cudaFree(nd->d_gidx);
  cudaFree(nd->d_F); cudaFree(nd->d_C); cudaFree(nd->d_Coff); cudaFree(nd->d_zs);
  cudaFree(nd->d_out); cudaFree(nd->d_flag);
  delete nd;
}

int64_t nd_factor_bytes(const NDFactor* nd) { return nd ? nd->stream_bytes : 0; }
int nd_levels(const NDFactor* nd) { return nd ? (int)nd->levels.size() : 0; }
