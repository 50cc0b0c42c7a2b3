"""Pins of oracle/fem.py against what the paper and the mathematics fix.

-m "not gpu".  Each test names its source; none re-types the assembly code.
"""
import os

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import fem
from oracle import lfa

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read_blocks(path):
    blocks, cur = {}, None
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line[0].isalpha():
            cur = line
            blocks[cur] = []
        else:
            blocks[cur].append([float(v) for v in line.split()])
    return {k: np.array(v) for k, v in blocks.items()}


def _row_stencil(Amat, dim, n, node):
    """Entries of row `node` arranged as a 3^dim stencil, axis order (.., y, x)."""
    N1 = n + 1
    out = np.zeros([3] * dim, dtype=np.complex128)
    row = Amat.getrow(node).tocoo()
    coords = []
    rem = node
    for d in range(dim):
        coords.append(rem % N1)
        rem //= N1
    for j, v in zip(row.col, row.data):
        c = []
        rem = j
        for d in range(dim):
            c.append(rem % N1 - coords[d] + 1)
            rem //= N1
        out[tuple(reversed(c))] += v
    return out


def test_2d_interior_stencils_match_paper():
    """interior rows of K and M are the printed 9-point stencils."""
    g = _read_blocks(os.path.join(GOLD, "q1_stencils_2d.txt"))
    n, h = 8, 1.0 / 8
    K, M, B = fem.assemble(2, n, 1.0, 0.0)          # k = 1 -> M(k,0) = M
    node = 4 + 9 * 4
    # golden rows run y = +1..-1, ours y = -1..+1
    np.testing.assert_allclose(_row_stencil(K, 2, n, node).real * 3, g["stiffness_times_3"][::-1],
                               atol=1e-13)
    np.testing.assert_allclose(_row_stencil(M, 2, n, node).real * 36 / h ** 2,
                               g["mass_times_36_over_h2"][::-1], atol=1e-12)
    assert abs(B.getrow(node)).sum() == 0.0


def test_3d_interior_stencils_closed_form():
    """3D Q1 (tensor product of 1D P1): K centre 8h/3, face 0, edge -h/6,
    corner -h/12; M centre 8h^3/27 and row sum h^3 (SURVEY 8(c) pin table)."""
    n, h = 6, 1.0 / 6
    K, M, B = fem.assemble(3, n, 1.0, 0.0)
    node = 3 + 7 * 3 + 49 * 3
    s = _row_stencil(K, 3, n, node).real
    for idx in np.ndindex(3, 3, 3):
        nz = sum(1 for i in idx if i != 1)
        want = {0: 8 * h / 3, 1: 0.0, 2: -h / 6, 3: -h / 12}[nz]
        assert abs(s[idx] - want) < 1e-14
    m = _row_stencil(M, 3, n, node).real
    assert abs(m[1, 1, 1] - 8 * h ** 3 / 27) < 1e-16
    assert abs(m.sum() - h ** 3) < 1e-16


@pytest.mark.parametrize("dim,n", [(2, 8), (2, 10), (3, 4)])
def test_row_sums(dim, n):
    """K 1 = 0; M 1 = h^d at interior nodes; B 1 = h on every 2D boundary node;
    3D: h^2 on face and edge nodes, 3h^2/4 at corners (derived)."""
    h = 1.0 / n
    K, M, B = fem.assemble(dim, n, 1.0, 0.0)
    one = np.ones(K.shape[0])
    assert np.abs(K @ one).max() < 1e-12
    coords = fem.node_coords(dim, n)
    on_bdry = np.zeros(K.shape[0], bool)
    n_faces = np.zeros(K.shape[0], int)
    for c in coords:
        e = (np.isclose(c, 0) | np.isclose(c, 1))
        on_bdry |= e
        n_faces += e
    mrow = (M @ one).real
    np.testing.assert_allclose(mrow[~on_bdry], h ** dim, rtol=1e-13)
    brow = (B @ one).real
    assert np.all(brow[~on_bdry] == 0)
    if dim == 2:
        np.testing.assert_allclose(brow[on_bdry], h, rtol=1e-13)
    else:
        np.testing.assert_allclose(brow[(n_faces == 1) | (n_faces == 2)], h * h, rtol=1e-13)
        np.testing.assert_allclose(brow[n_faces == 3], 0.75 * h * h, rtol=1e-13)


@pytest.mark.parametrize("dim", [2, 3])
def test_complex_symmetric_not_hermitian(dim):
    """A(k,eps) = A^T (real basis) and A != A^H."""
    n = 6 if dim == 2 else 4
    rng = np.random.default_rng(1)
    k = rng.uniform(2, 9, n ** dim)
    A = fem.system_matrix(dim, n, k, 0.5 * k ** 1.5)
    x = rng.standard_normal(A.shape[0]) + 1j * rng.standard_normal(A.shape[0])
    y = rng.standard_normal(A.shape[0]) + 1j * rng.standard_normal(A.shape[0])
    assert abs(x @ (A @ y) - y @ (A @ x)) <= 1e-13 * abs(x @ (A @ y))
    assert abs(A - A.T).max() <= 1e-14 * abs(A).max()
    assert abs(A - A.conj().T).max() > 1e-3


def test_fourier_mode_2d_matches_paper_symbol():
    """Interior rows: A e^{i theta x/h} = L~_h(theta) e^{i theta x/h} with the
    paper's symbol, lambda = k^2 + i eps."""
    n, k, eps = 64, 20.0, 20.0 ** 1.5
    h = 1.0 / n
    A = fem.system_matrix(2, n, k, eps)
    x, y = fem.node_coords(2, n)
    for th in [(0.37, -1.1), (2.5, 0.2), (-3.0, 3.1)]:
        u = np.exp(1j * (th[0] * x + th[1] * y) / h)
        Au = A @ u
        inner = (x > 1e-9) & (x < 1 - 1e-9) & (y > 1e-9) & (y < 1 - 1e-9)
        sym = lfa.L_h(th[0], th[1], k * k + 1j * eps, h)
        np.testing.assert_allclose(Au[inner], sym * u[inner], rtol=1e-12, atol=1e-12 * abs(sym))


def test_fourier_mode_3d_tensor_symbol():
    """3D tensor-product extension of the symbol:
    L~ = (h/36) sum_d (2-2cos t_d) prod_{e!=d} (4+2cos t_e) - lam (h^3/216) prod (4+2cos t_d)."""
    n, k, eps = 12, 5.0, 3.0
    h = 1.0 / n
    A = fem.system_matrix(3, n, k, eps)
    x, y, z = fem.node_coords(3, n)
    th = (0.4, -1.3, 2.2)
    u = np.exp(1j * (th[0] * x + th[1] * y + th[2] * z) / h)
    c = [np.cos(t) for t in th]
    lam = k * k + 1j * eps
    stiff = sum((2 - 2 * c[d]) * np.prod([4 + 2 * c[e] for e in range(3) if e != d])
                for d in range(3)) * h / 36
    sym = stiff - lam * h ** 3 / 216 * np.prod([4 + 2 * cc for cc in c])
    inner = np.ones_like(x, bool)
    for cc in (x, y, z):
        inner &= (cc > 1e-9) & (cc < 1 - 1e-9)
    np.testing.assert_allclose((A @ u)[inner], sym * u[inner], rtol=1e-12, atol=1e-13)


def _plane_wave_error(n, k=6.0, ang=0.3):
    """Discrete L2 (RMS nodal) error of the Q1 solution of -Lap u - k^2 u = 0,
    du/dn - iku = g with the exact plane wave u = e^{ik d.x} (manufactured)."""
    d = np.array([np.cos(ang), np.sin(ang)])
    h = 1.0 / n
    A = fem.system_matrix(2, n, k, 0.0)
    F = np.zeros(A.shape[0], dtype=np.complex128)
    gx, gw = np.polynomial.legendre.leggauss(6)
    N1 = n + 1
    # boundary load F_i = int_bdry g phi_i, g = ik(d.n - 1) u, by 6-point Gauss per edge
    sides = [((0, None), np.array([-1.0, 0.0])), ((n, None), np.array([1.0, 0.0])),
             ((None, 0), np.array([0.0, -1.0])), ((None, n), np.array([0.0, 1.0]))]
    for (fx, fy), nrm in sides:
        for e in range(n):
            s = (gx + 1) / 2 * h + e * h
            w = gw * h / 2
            if fx is not None:
                px, py = np.full_like(s, fx * h), s
                nodes = [fx + N1 * e, fx + N1 * (e + 1)]
            else:
                px, py = s, np.full_like(s, fy * h)
                nodes = [e + N1 * fy, e + 1 + N1 * fy]
            u = np.exp(1j * k * (d[0] * px + d[1] * py))
            g = 1j * k * (d @ nrm - 1.0) * u
            t = (s - e * h) / h
            F[nodes[0]] += np.sum(w * g * (1 - t))
            F[nodes[1]] += np.sum(w * g * t)
    uh = spla.spsolve(A.tocsc(), F)
    x, y = fem.node_coords(2, n)
    ue = np.exp(1j * k * (d[0] * x + d[1] * y))
    return np.sqrt(np.mean(np.abs(uh - ue) ** 2))


def test_manufactured_plane_wave_second_order():
    """Q1 nodal error falls 4x per halving of h (second order; BASELINE.json
    north_star 'manufactured-solution convergence rate')."""
    errs = [_plane_wave_error(n) for n in (16, 32, 64)]
    rates = [np.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(1.9 <= r <= 2.1 for r in rates), (errs, rates)


def test_dof_counts_match_paper():
    """Tables 2 and 6 print the real DoF counts of the Q1 grids (2 reals per node)."""
    for line in open(os.path.join(GOLD, "dof_counts.txt")):
        if line.startswith("#") or not line.strip():
            continue
        dim, n, dofs = (int(v) for v in line.split()[:3])
        A = None  # counting only: nodes of the Q1 grid
        assert 2 * (n + 1) ** dim == dofs


def test_apply_rows_equals_assembled_rows():
    """The sampled-row apply used for full-size checks equals rows of the
    element-loop CSR assembly (brute force, 2D and 3D, constant and per-element k)."""
    from oracle import fem as F
    rng = np.random.default_rng(7)
    for dim, n in [(2, 6), (3, 4)]:
        ne, N = n ** dim, (n + 1) ** dim
        for kk, ee in [(3.0, 1.5), (rng.uniform(1, 4, ne), rng.uniform(0, 2, ne))]:
            A = F.system_matrix(dim, n, kk, ee)
            x = rng.standard_normal(N) + 1j * rng.standard_normal(N)
            rows = np.arange(N)
            assert np.allclose(F.apply_rows(dim, n, kk, ee, x, rows), (A @ x)[rows], rtol=1e-13, atol=1e-13)
