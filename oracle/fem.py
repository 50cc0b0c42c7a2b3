"""Oracle: Q1 finite elements on the uniform grid of (0,1)^d, d in {2,3}.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:82-91 (section 2, sesquilinear form)
    a_eps(u,v) = int grad u . grad v  -  int (k^2 + i eps) u v  -  i int_bdry k u v
PAPER.md:100-113 (Eq. discreteproblem / sys_matrix)
    A(k, eps) = K - M(k, eps) - i B(k)
PAPER.md:94-99: Q_p elements on squares/cubes; here p = 1 (BASELINE.json).

Readings: element-constant coefficients k_e (C1), eps_e = beta
k_e^sigma pointwise (C2), boundary faces use the k_e of the adjacent element
(C3), exact integration of the bilinear/trilinear basis.

Node numbering: x fastest, node (i, j[, l]) -> i + (n+1) j [+ (n+1)^2 l].
Element numbering: e (i, j[, l]) -> i + n j [+ n^2 l].
Local node a of an element: bit d of a = offset along axis d.
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp


def q1_1d(h: float):
    """1D linear element stiffness and mass on an interval of length h."""
    k1 = np.array([[1.0, -1.0], [-1.0, 1.0]]) / h
    m1 = np.array([[2.0, 1.0], [1.0, 2.0]]) * (h / 6.0)
    return k1, m1


def _kron_axes(mats):
    """Kronecker product with axis 0 FASTEST: mats = [A_x, A_y(, A_z)];
    local index a = a_x + 2 a_y (+ 4 a_z)."""
    out = np.array([[1.0]])
    for m in mats:            # x first -> ends up fastest
        out = np.kron(m, out)
    return out


def element_matrices(dim: int, h: float):
    """Exact Q1 element stiffness K^e, mass M^e (2^d x 2^d) and boundary-face
    mass B^f (2^(d-1) x 2^(d-1)) for a cell of edge h (tensor products of the
    1D forms)."""
    k1, m1 = q1_1d(h)
    Ke = np.zeros((2 ** dim, 2 ** dim))
    for d in range(dim):
        Ke += _kron_axes([k1 if e == d else m1 for e in range(dim)])
    Me = _kron_axes([m1] * dim)
    Bf = _kron_axes([m1] * (dim - 1))
    return Ke, Me, Bf


def _local_offsets(dim: int, n: int):
    """Global node offset of local node a relative to the element's first node."""
    N1 = n + 1
    offs = []
    for a in range(2 ** dim):
        o = 0
        for d in range(dim):
            o += ((a >> d) & 1) * N1 ** d
        offs.append(o)
    return np.asarray(offs, dtype=np.int64)


def _element_first_nodes(dim: int, n: int):
    """Global index of local node 0 of every element (element order x fastest)."""
    N1 = n + 1
    idx = np.zeros([n] * dim, dtype=np.int64)
    grids = np.meshgrid(*([np.arange(n)] * dim), indexing="ij")  # slow..fast
    for d in range(dim):
        idx += grids[dim - 1 - d] * N1 ** d   # grids[dim-1] is x
    return idx.reshape(-1)


def _element_index_grids(dim: int, n: int):
    """Integer coordinates (x, y[, z]) of every element, element order."""
    grids = np.meshgrid(*([np.arange(n)] * dim), indexing="ij")
    return [g.reshape(-1) for g in reversed(grids)]


def assemble(dim: int, n: int, k_elem, eps_elem):
    """Element-loop CSR assembly of K, M(k,eps) and B(k).

    k_elem, eps_elem: per-element arrays (n^dim,), or scalars.
    Returns (K, Mlam, B) with Mlam = sum_e (k_e^2 + i eps_e) M^e and
    B = sum_f k_f B^f (complex CSR matrices, (n+1)^dim square)."""
    h = 1.0 / n
    ne = n ** dim
    N = (n + 1) ** dim
    k_elem = np.broadcast_to(np.asarray(k_elem, dtype=np.float64), (ne,))
    eps_elem = np.broadcast_to(np.asarray(eps_elem, dtype=np.float64), (ne,))
    lam = k_elem ** 2 + 1j * eps_elem
    Ke, Me, Bf = element_matrices(dim, h)
    first = _element_first_nodes(dim, n)
    offs = _local_offsets(dim, n)
    nl = 2 ** dim

    rows, cols, kv, mv = [], [], [], []
    for a in range(nl):              # element loop, vectorised over elements
        for b in range(nl):
            rows.append(first + offs[a])
            cols.append(first + offs[b])
            kv.append(np.full(ne, Ke[a, b]))
            mv.append(lam * Me[a, b])
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    K = sp.csr_matrix((np.concatenate(kv).astype(np.complex128), (r, c)), shape=(N, N))
    Mlam = sp.csr_matrix((np.concatenate(mv), (r, c)), shape=(N, N))

    # boundary faces: for every axis d and side s in {0, 1}, the elements with
    # coordinate 0 (s=0) or n-1 (s=1) along d own a face on the boundary.
    coords = _element_index_grids(dim, n)
    brow, bcol, bv = [], [], []
    for d in range(dim):
        for side in (0, 1):
            sel = np.nonzero(coords[d] == (0 if side == 0 else n - 1))[0]
            # local nodes of the face: bit d fixed to `side`
            face_local = [a for a in range(nl) if ((a >> d) & 1) == side]
            for fa, a in enumerate(face_local):
                for fb, b in enumerate(face_local):
                    brow.append(first[sel] + offs[a])
                    bcol.append(first[sel] + offs[b])
                    bv.append(k_elem[sel] * Bf[fa, fb])
    B = sp.csr_matrix((np.concatenate(bv).astype(np.complex128),
                       (np.concatenate(brow), np.concatenate(bcol))), shape=(N, N))
    return K, Mlam, B


def system_matrix(dim: int, n: int, k_elem, eps_elem):
    """A(k, eps) = K - M(k, eps) - i B(k)   (Eq. sys_matrix)."""
    K, Mlam, B = assemble(dim, n, k_elem, eps_elem)
    return (K - Mlam - 1j * B).tocsr()


def prolongation(dim: int, n: int):
    """Canonical interpolation I: V_{2h} -> V_h:
    P_1D(2i, i) = 1, P_1D(2i+1, i) = P_1D(2i+1, i+1) = 1/2, tensorised."""
    nc = n // 2
    P1 = sp.lil_matrix((n + 1, nc + 1))
    for i in range(nc + 1):
        P1[2 * i, i] = 1.0
        if i < nc:
            P1[2 * i + 1, i] = 0.5
            P1[2 * i + 1, i + 1] = 0.5
    P1 = P1.tocsr()
    P = sp.csr_matrix(np.ones((1, 1)))
    for _ in range(dim):
        P = sp.kron(P1, P).tocsr()
    return P.astype(np.complex128)


def node_coords(dim: int, n: int):
    """Coordinates (x, y[, z]) of all nodes, node order (x fastest)."""
    c = np.arange(n + 1) / n
    grids = np.meshgrid(*([c] * dim), indexing="ij")
    return [g.reshape(-1) for g in reversed(grids)]


def shifts(k_elem, beta: float, sigma: float):
    """eps_e = beta * k_e^sigma (reading C2; the paper's eps = k^sigma has beta=1,
    PAPER.md:27, 532)."""
    return beta * np.asarray(k_elem, dtype=np.float64) ** sigma


def apply_rows(dim: int, n: int, k_elem, eps_elem, x, rows):
    """Rows `rows` of A(k, eps) x by a direct element loop around each node
    (the same element and face matrices as `assemble`), for
    sampled checks at sizes where assembling A is impractical."""
    h = 1.0 / n
    N1 = n + 1
    Ke, Me, Bf = element_matrices(dim, h)
    k_elem = np.asarray(k_elem, dtype=np.float64)
    eps_elem = np.asarray(eps_elem, dtype=np.float64)
    scalar = k_elem.ndim == 0
    out = np.zeros(len(rows), dtype=np.complex128)
    for r, node in enumerate(rows):
        c = [(int(node) // N1 ** d) % N1 for d in range(dim)]
        acc = 0.0 + 0.0j
        for a in range(2 ** dim):                       # node = local node a of element e
            e = [c[d] - ((a >> d) & 1) for d in range(dim)]
            if any(v < 0 or v >= n for v in e):
                continue
            eidx = sum(e[d] * n ** d for d in range(dim))
            ke = float(k_elem) if scalar else float(k_elem[eidx])
            ee = float(eps_elem) if eps_elem.ndim == 0 else float(eps_elem[eidx])
            lam = ke * ke + 1j * ee
            first = sum(e[d] * N1 ** d for d in range(dim))
            for b in range(2 ** dim):
                gb = first + sum(((b >> d) & 1) * N1 ** d for d in range(dim))
                acc += (Ke[a, b] - lam * Me[a, b]) * x[gb]
            for d in range(dim):                        # boundary faces of this element
                side = (a >> d) & 1
                if not ((side == 0 and e[d] == 0) or (side == 1 and e[d] == n - 1)):
                    continue
                face = [q for q in range(2 ** dim) if ((q >> d) & 1) == side]
                fa = face.index(a)
                for fb, b in enumerate(face):
                    gb = first + sum(((b >> dd) & 1) * N1 ** dd for dd in range(dim))
                    acc += -1j * ke * Bf[fa, fb] * x[gb]
        out[r] = acc
    return out
