"""Slab decomposition of one solve (north_star "Large single
solves use a slab decomposition, with NCCL halo exchange ... and allreduce for
Arnoldi inner products"), through the C ABI (-m gpu).

The in-process slab mode runs the same kernels, ghost planes, replicated coarse
solve and split Arnoldi reductions as S processes, with device copies for the
exchange steps; it is checked against the CPU oracle at the parity bars, and a
one-rank NCCL communicator exercises the NCCL calls of the multi-GPU path."""
import numpy as np
import pytest
import torch

from oracle.solve import OracleProblem
from workloads import config_spec

pytestmark = pytest.mark.gpu

hh = pytest.importorskip("paper_2104_01439_b200.hh") if torch.cuda.is_available() else None


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).cuda()


def _host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _rand(n, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal(n) + 1j * r.standard_normal(n)


def _scaled(name, n):
    spec = config_spec(name, n=n)
    full = config_spec(name)
    spec.k_const = full.k_const * n / full.n
    return spec


CASES = [
    ("cfg0_n64_S2", lambda: config_spec("cfg0", n=64), 2),
    ("cfg0_n64_S5", lambda: config_spec("cfg0", n=64), 5),       # ragged slabs, partial tiles
    ("cfg2_n64_S3", lambda: config_spec("cfg2", n=64), 3),       # 2D heterogeneous
    ("cfg3_n14_S2", lambda: _scaled("cfg3", 14), 2),              # 3D constant k
    ("cfg4_n12_S3", lambda: config_spec("cfg4", n=12), 3),        # 3D heterogeneous
]


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def trio(request):
    _, mk, S = request.param
    spec = mk()
    orc = OracleProblem(spec)
    gs = hh.Problem.from_spec(spec, nslabs_local=S)
    g1 = hh.Problem.from_spec(spec)
    yield spec, orc, gs, g1, S
    gs.close()
    g1.close()


def test_slab_layout_covers_the_grid(trio):
    spec, _, gs, _, S = trio
    n_local, first, n_planes = gs.local_layout()
    assert (n_local, first, n_planes) == (spec.n_nodes, 0, spec.n + 1)
    z = hh.slab_bounds(spec.n, S)
    assert z[0] == 0 and z[-1] == spec.n + 1 and all(v % 2 == 0 for v in z[:-1])
    assert all(b - a >= 3 for a, b in zip(z, z[1:]))


def test_slab_apply_parity(trio):
    spec, orc, gs, _, _ = trio
    x = _rand(spec.n_nodes, 11)
    for op in (hh.HH_OP_A0, hh.HH_OP_AEPS):
        y = _host(gs.apply_op(op, _dev(x)))
        assert _rel(y, orc.apply(op, x)) <= 1e-10, op


def test_slab_vcycle_parity(trio):
    spec, orc, gs, _, _ = trio
    f = _rand(spec.n_nodes, 12)
    z = _host(gs.vcycle(_dev(f)))
    assert _rel(z, orc.vcycle(f)) <= 1e-10


def test_slab_fgmres_matches_oracle_and_single_slab(trio):
    spec, orc, gs, g1, _ = trio
    b = spec.rhs()
    o = hh.opts(restart=spec.restart, rtol=spec.rtol)
    xs, rs = gs.fgmres_solve(_dev(b), o=o)
    x1, r1 = g1.fgmres_solve(_dev(b), o=o)
    xo, ro = OracleProblem(spec).solve(b)
    assert abs(rs["iterations"] - ro.iterations) <= 1
    assert rs["iterations"] == r1["iterations"]
    assert _rel(_host(xs), _host(x1)) <= 1e-10       # same arithmetic up to summation order
    xf, rf = gs.fgmres_solve(_dev(b), o=hh.opts(restart=spec.restart, rtol=spec.rtol,
                                                 fixed_iters=ro.iterations))
    assert _rel(_host(xf), xo) <= 1e-8
    assert rs["rel_res_true"] <= spec.rtol * 1.01


def test_too_many_slabs_is_a_config_error():
    spec = config_spec("cfg0", n=8)
    with pytest.raises(hh.HHError) as e:
        hh.Problem.from_spec(spec, nslabs_local=3)      # 9 planes -> slabs of 2 < G = 3
    assert e.value.status == 2


def test_single_rank_nccl_communicator():
    """NCCL path (communicator from hh_nccl_unique_id, allreduces in the Arnoldi
    step) with one rank: same iterations and solution as the plain handle."""
    spec = config_spec("cfg0", n=32)
    nid = hh.nccl_unique_id()
    assert len(nid) == 128
    gn = hh.Problem.from_spec(spec, nccl_id=nid, rank=0, nranks=1)
    g1 = hh.Problem.from_spec(spec)
    b = _dev(spec.rhs())
    o = hh.opts(restart=spec.restart, rtol=spec.rtol)
    xn, rn = gn.fgmres_solve(b, o=o)
    x1, r1 = g1.fgmres_solve(b, o=o)
    assert rn["iterations"] == r1["iterations"]
    assert _rel(_host(xn), _host(x1)) <= 1e-12
    gn.close()
    g1.close()
