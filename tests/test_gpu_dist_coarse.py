"""Distributed exact coarse solve (SURVEY.md 8(f) row 2 / 8(e) "second
version"; the paper's parallel MUMPS LU) through
the C ABI (-m gpu): coarse_solver = HH_COARSE_ND_DIST on in-process slabs, i.e.
the same rank views, Schur-complement / update-vector transfers and interface
broadcasts as S processes, with device copies for the exchanges.

Each slab factors only its slab interior and its interface plane; the results
must match the oracle's (pivoted sparse LU) coarse solve and V-cycle at 1e-10,
FGMRES at +-1 iteration / 1e-8, and the replicated-factor slab solve."""
import numpy as np
import pytest
import torch

from oracle.solve import OracleProblem
from workloads import config_spec
from workloads.vectors import random_complex

pytestmark = pytest.mark.gpu

hh = pytest.importorskip("paper_2104_01439_b200.hh") if torch.cuda.is_available() else None


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).cuda()


def _host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _scaled(name, n):
    spec = config_spec(name, n=n)
    full = config_spec(name)
    spec.k_const = full.k_const * n / full.n
    return spec


CASES = [
    ("cfg0_n64_S2", lambda: config_spec("cfg0", n=64), 2),
    ("cfg0_n64_S5", lambda: config_spec("cfg0", n=64), 5),      # ragged slabs, odd chain
    ("cfg2_n64_S4", lambda: config_spec("cfg2", n=64), 4),      # 2D heterogeneous
    ("cfg3_n16_S2", lambda: _scaled("cfg3", 16), 2),             # 3D constant k
    ("cfg3_n24_S3", lambda: _scaled("cfg3", 24), 3),
    ("cfg4_n16_S4", lambda: config_spec("cfg4", n=16), 4),       # 3D heterogeneous
    ("cfg4_n24_S6", lambda: config_spec("cfg4", n=24), 6),
]


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def trio(request):
    _, mk, S = request.param
    spec = mk()
    orc = OracleProblem(spec)
    gd = hh.Problem.from_spec(spec, nslabs_local=S, coarse_solver=hh.HH_COARSE_ND_DIST)
    gr = hh.Problem.from_spec(spec, nslabs_local=S)      # replicated factor
    yield spec, orc, gd, gr, S
    gd.close()
    gr.close()


def test_dist_coarse_solve_parity(trio):
    spec, orc, gd, gr, _ = trio
    r = random_complex(spec.n_coarse_nodes, 21)
    e = _host(gd.coarse_solve(_dev(r)))
    assert _rel(e, orc.tg.coarse.solve(r)) <= 1e-10
    assert _rel(orc.tg.Ac @ e, r) <= 1e-11
    assert _rel(e, _host(gr.coarse_solve(_dev(r)))) <= 1e-11


def test_dist_vcycle_parity(trio):
    spec, orc, gd, _, _ = trio
    f = random_complex(spec.n_nodes, 22)
    z = _host(gd.vcycle(_dev(f)))
    assert _rel(z, orc.vcycle(f)) <= 1e-10


def test_dist_fgmres_parity(trio):
    spec, orc, gd, gr, _ = trio
    b = spec.rhs()
    xo, ro = orc.solve(b)
    o = hh.opts(restart=spec.restart, rtol=spec.rtol, max_iters=spec.max_iters)
    x, r = gd.fgmres_solve(_dev(b), o=o)
    assert abs(r["iterations"] - ro.iterations) <= 1 and r["converged"] == 1
    xr, rr = gr.fgmres_solve(_dev(b), o=o)
    assert r["iterations"] == rr["iterations"]
    if r["iterations"] != ro.iterations:
        x, r = gd.fgmres_solve(_dev(b), o=hh.opts(restart=spec.restart, rtol=spec.rtol,
                                                  fixed_iters=ro.iterations))
    assert _rel(_host(x), xo) <= 1e-8


def test_dist_needs_slabs():
    spec = config_spec("cfg0", n=16)
    with pytest.raises(hh.HHError) as e:
        hh.Problem.from_spec(spec, coarse_solver=hh.HH_COARSE_ND_DIST)
    assert e.value.status == 2
    with pytest.raises(hh.HHError) as e:   # a slab with a single coarse plane
        hh.Problem.from_spec(config_spec("cfg0", n=8), nslabs_local=4, coarse_solver=hh.HH_COARSE_ND_DIST)
    assert e.value.status in (2, 10)


@pytest.mark.parametrize("name,n,S", [("cfg4", 256, 2), ("cfg4", 128, 4), ("cfg4", 128, 8), ("cfg3", 128, 4)])
def test_dist_fullsize(name, n, S):
    """BASELINE configs[4] at full size (257^3 fine / 129^3 coarse, S = 2) and the
    129^3 grids (cfg4 medium at n = 128, cfg3; S = 4, 8) with the coarse factor
    distributed over S in-process slabs: the same iteration count as the
    single-GPU solve (+-1), converged, and the true residual below rtol."""
    spec = config_spec(name, n=n)
    o = hh.opts(restart=spec.restart, rtol=spec.rtol)
    b = _dev(spec.rhs())
    g1 = hh.Problem.from_spec(spec)
    _, r1 = g1.fgmres_solve(b, o=o)
    g1.close()
    torch.cuda.empty_cache()
    gd = hh.Problem.from_spec(spec, nslabs_local=S, coarse_solver=hh.HH_COARSE_ND_DIST)
    x, rd = gd.fgmres_solve(b, o=o)
    gd.close()
    assert rd["converged"] == 1 and rd["rel_res_true"] <= spec.rtol
    assert abs(rd["iterations"] - r1["iterations"]) <= 1, (rd, r1)
