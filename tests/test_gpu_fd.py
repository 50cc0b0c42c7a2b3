"""Coarse solve by fast diagonalisation (fd.cu, HH_COARSE_FD) against the CPU
oracle through the C ABI (-m gpu).

The FD path is the same exact coarse solve e_c = (A_eps^(1))^{-1} r_c as the
oracle's sparse LU (Alg. 1 line 3), computed from the Kronecker
structure of the constant-k Q1 operator.  Bars: the
coarse solve <= 1e-10 relative to the oracle and residual <= 1e-11 (the ND
bars); V-cycle <= 1e-10; FD and ND coarse solves of the same handle data agree
to round-off.  Cases cover even and odd coarse cell counts (odd nc has no
centre line, even nc has one), the smallest grids, every cfg1 (k, kh) class,
strong and weak shifts, 3D, slabs and the failure / fallback paths."""
import numpy as np
import pytest
import torch

from oracle.solve import OracleProblem
from workloads import config_spec
from workloads.configs import sweep_sample_spec

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


def _spec(dim, n, k, beta, sigma):
    s = config_spec("cfg0" if dim == 2 else "cfg3", n=n)
    s.k_const, s.beta, s.sigma = float(k), float(beta), float(sigma)
    return s


# (dim, n, k, beta, sigma): nc = n/2 even and odd, tiny grids, the cfg1 extremes
# (k = 160 at kh 0.3 / 0.6: nc = 267 / 134), weakest and strongest cfg1 shifts
CASES_2D = [
    (2, 4, 1.5, 0.5, 1.5),        # nc = 2: 3 x 3 coarse nodes
    (2, 6, 2.0, 1.0, 1.0),        # nc = 3 (odd)
    (2, 10, 3.0, 0.1, 1.0),       # nc = 5
    (2, 34, 10.0, 0.1, 1.0),      # cfg1 k = 10, kh 0.3
    (2, 66, 20.0, 1.0, 2.0),      # nc = 33
    (2, 64, 20.0, 1.0, 1.5),      # cfg0
    (2, 130, 40.0, 0.5, 1.5),     # nc = 65
    (2, 268, 160.0, 0.1, 1.0),    # cfg1 k = 160, kh 0.6, weakest shift
    (2, 534, 160.0, 0.1, 1.0),    # cfg1 k = 160, kh 0.3 (nc = 267, odd)
    (2, 534, 160.0, 1.0, 2.0),    # strongest shift
]
CASES_3D = [
    (3, 4, 1.25, 0.5, 1.5),       # nc = 2
    (3, 6, 1.9, 0.5, 1.5),        # nc = 3
    (3, 14, 4.4, 0.5, 1.5),       # cfg3 kh, nc = 7
    (3, 22, 6.9, 0.1, 1.0),
    (3, 32, 10.0, 0.5, 1.5),      # nc = 16
]
CASES = CASES_2D + CASES_3D


@pytest.fixture(scope="module", params=CASES, ids=[f"d{c[0]}_n{c[1]}_k{c[2]}_b{c[3]}_s{c[4]}" for c in CASES])
def fd_case(request):
    spec = _spec(*request.param)
    orc = OracleProblem(spec)
    gp = hh.Problem.from_spec(spec, coarse_solver=hh.HH_COARSE_FD)
    assert gp.coarse_kind() == hh.HH_COARSE_FD
    yield spec, orc, gp
    gp.close()


def test_fd_coarse_solve_matches_oracle(fd_case):
    spec, orc, gp = fd_case
    for seed in (3, 4):
        r = _rand(spec.n_coarse_nodes, seed)
        e = _host(gp.coarse_solve(_dev(r)))
        assert _rel(e, orc.tg.coarse.solve(r)) <= 1e-10
        assert _rel(orc.tg.Ac @ e, r) <= 1e-11


def test_fd_coarse_solve_symmetric_and_point_data(fd_case):
    """Data with the grid's mirror symmetries and a single node (one folded block
    nonzero / every block nonzero) -- each parity block is exercised alone."""
    spec, orc, gp = fd_case
    m = spec.n // 2 + 1
    sh = (m,) * spec.dim
    r = np.zeros(sh, dtype=np.complex128)
    r[(0,) * spec.dim] = 1.0 - 0.5j                  # corner node
    e = _host(gp.coarse_solve(_dev(r.ravel())))
    assert _rel(e, orc.tg.coarse.solve(r.ravel())) <= 1e-10
    g = _rand(spec.n_coarse_nodes, 9).reshape(sh)
    for ax in range(spec.dim):                       # symmetric in every axis
        g = g + np.flip(g, axis=ax)
    e = _host(gp.coarse_solve(_dev(g.ravel())))
    assert _rel(e, orc.tg.coarse.solve(g.ravel())) <= 1e-10


def test_fd_vcycle_matches_oracle(fd_case):
    spec, orc, gp = fd_case
    f = _rand(spec.n_nodes, 5)
    assert _rel(_host(gp.vcycle(_dev(f))), orc.vcycle(f)) <= 1e-10


@pytest.mark.parametrize("case", [CASES_2D[5], CASES_2D[8], CASES_3D[2]],
                         ids=["cfg0", "k160_nc267", "d3_n14"])
def test_fd_equals_nd(case):
    """FD and the ND factor solve the same system: equal to round-off."""
    spec = _spec(*case)
    a = hh.Problem.from_spec(spec, coarse_solver=hh.HH_COARSE_FD)
    b = hh.Problem.from_spec(spec, coarse_solver=hh.HH_COARSE_ND)
    assert a.coarse_kind() == hh.HH_COARSE_FD and b.coarse_kind() == hh.HH_COARSE_ND
    r = _rand(spec.n_coarse_nodes, 6)
    ea, eb = _host(a.coarse_solve(_dev(r))), _host(b.coarse_solve(_dev(r)))
    assert _rel(ea, eb) <= 1e-12
    f = _rand(spec.n_nodes, 7)
    assert _rel(_host(a.vcycle(_dev(f))), _host(b.vcycle(_dev(f)))) <= 1e-12
    o = hh.opts(restart=spec.restart, rtol=spec.rtol)
    _, ra = a.fgmres_solve(_dev(spec.rhs()), o=o)
    _, rb = b.fgmres_solve(_dev(spec.rhs()), o=o)
    assert ra["iterations"] == rb["iterations"]
    a.close()
    b.close()


def test_fd_fgmres_cfg0_and_hardest_sweep_sample():
    """FGMRES through the FD coarse solve: iterations +-1, x <= 1e-8 at equal counts."""
    for spec in (config_spec("cfg0"),
                 sweep_sample_spec({"id": 0, "n": 268, "k": 160.0, "beta": 0.1, "sigma": 1.0,
                                    "kh_target": 0.6})):
        orc = OracleProblem(spec)
        gp = hh.Problem.from_spec(spec)
        assert gp.coarse_kind() == hh.HH_COARSE_FD
        xo, ro = orc.solve()
        o = hh.opts(restart=spec.restart, rtol=spec.rtol, max_iters=spec.max_iters)
        x, r = gp.fgmres_solve(_dev(spec.rhs()), o=o)
        assert abs(r["iterations"] - ro.iterations) <= 1
        if r["iterations"] != ro.iterations:
            x, r = gp.fgmres_solve(_dev(spec.rhs()), o=hh.opts(restart=spec.restart, fixed_iters=ro.iterations))
        assert _rel(_host(x), xo) <= 1e-8
        gp.close()


def test_fd_with_slabs_equals_unsliced():
    """The replicated coarse solve of in-process slabs shares one eigenbasis."""
    spec = config_spec("cfg0", n=64)
    g1 = hh.Problem.from_spec(spec)
    gs = hh.Problem.from_spec(spec, nslabs_local=3)
    assert gs.coarse_kind() == hh.HH_COARSE_FD
    f = _rand(spec.n_nodes, 8)
    z1 = _host(g1.vcycle(_dev(f)))
    zs = _host(gs.vcycle(_dev(f)))
    assert _rel(zs, z1) <= 1e-12
    _, r1 = g1.fgmres_solve(_dev(spec.rhs()))
    _, rs = gs.fgmres_solve(_dev(spec.rhs()))
    assert abs(r1["iterations"] - rs["iterations"]) <= 1
    g1.close()
    gs.close()


def test_fd_validation_failure_falls_back_or_fails_loudly(monkeypatch):
    """HH_FD_FAIL=1 marks the eigen-decomposition failed (fault injection): AUTO
    must fall back to the ND factor (same results), an explicit HH_COARSE_FD
    must fail with HH_E_SINGULAR -- never a wrong coarse correction."""
    spec = config_spec("cfg0", n=48)
    orc = OracleProblem(spec)
    monkeypatch.setenv("HH_FD_FAIL", "1")
    gp = hh.Problem.from_spec(spec)
    assert gp.coarse_kind() == hh.HH_COARSE_ND
    r = _rand(spec.n_coarse_nodes, 10)
    assert _rel(_host(gp.coarse_solve(_dev(r))), orc.tg.coarse.solve(r)) <= 1e-10
    gp.close()
    with pytest.raises(hh.HHError) as e:
        hh.Problem.from_spec(spec, coarse_solver=hh.HH_COARSE_FD)
    assert e.value.status == 7 and "validation" in str(e.value)
    samples = [{"id": i, "dim": 2, "n": 48, "k": 15.0, "kh_target": 0.3, "sigma": 1.5,
                "beta": 0.5} for i in range(3)]
    res = hh.sweep(samples)            # AUTO: the batch falls back to ND
    monkeypatch.delenv("HH_FD_FAIL")
    ref = hh.sweep(samples, coarse_solver=hh.HH_COARSE_ND)
    for a, b in zip(res, ref):
        assert a["status"] == 0 and a["iterations"] == b["iterations"]


def test_fd_unresolved_coarse_grid_is_correct_either_way():
    """k h_c = 2: AUTO picks FD; if the secular continuation loses a root the
    validation sends the problem to the ND factor.  Either way the coarse
    solve matches the oracle."""
    spec = _spec(2, 402, 400.0, 0.5, 1.5)
    orc = OracleProblem(spec)
    gp = hh.Problem.from_spec(spec)
    assert gp.coarse_kind() in (hh.HH_COARSE_FD, hh.HH_COARSE_ND)
    r = _rand(spec.n_coarse_nodes, 11)
    e = _host(gp.coarse_solve(_dev(r)))
    assert _rel(e, orc.tg.coarse.solve(r)) <= 1e-10
    gp.close()


def test_fd_heterogeneous_is_rejected():
    spec = config_spec("cfg2", n=32)
    with pytest.raises(hh.HHError) as e:
        hh.Problem.from_spec(spec, coarse_solver=hh.HH_COARSE_FD)
    assert e.value.status == 2
    gp = hh.Problem.from_spec(spec)               # AUTO -> ND for heterogeneous k
    assert gp.coarse_kind() == hh.HH_COARSE_ND
    gp.close()


def test_fd_flops_are_accounted():
    spec = config_spec("cfg0")
    gp = hh.Problem.from_spec(spec)
    gp.reset_timers(True)
    gp.fgmres_solve(_dev(spec.rhs()))
    t, a = hh.coarse_flops(gp)
    P = spec.n // 4 + 1
    its = gp.read_timers()["coarse"]["launches"]
    assert its > 0 and abs(t - its * 128.0 * P ** 3) <= 1e-6 * t
    assert a >= t > 0
    gp.reset_timers(False)
    gp.close()
    gn = hh.Problem.from_spec(spec, coarse_solver=hh.HH_COARSE_ND)
    gn.reset_timers(True)
    gn.fgmres_solve(_dev(spec.rhs()))
    assert hh.coarse_flops(gn) == (0.0, 0.0)
    gn.close()


def test_fd_sweep_equals_nd_sweep():
    """hh_sweep with the FD coarse solve forced and with the ND factor forced on a
    strided subset of cfg1 (every grid size class, both kh, weak and strong
    shifts, two k sharing a grid -> two basis slots in one batch): the same
    iteration counts (+-1: the coarse solves agree to ~1e-14) and true residuals."""
    from workloads import sweep_samples
    samples = sweep_samples()[::53]
    fd = hh.sweep(samples, coarse_solver=hh.HH_COARSE_FD)
    nd = hh.sweep(samples, coarse_solver=hh.HH_COARSE_ND)
    for s, a, b in zip(samples, fd, nd):
        assert a["status"] == 0 and b["status"] == 0, (s, a, b)
        assert abs(a["iterations"] - b["iterations"]) <= 1, (s, a, b)
        assert a["converged"] == b["converged"] == 1
        if a["iterations"] == b["iterations"]:
            assert abs(a["rel_res_true"] - b["rel_res_true"]) <= 1e-6 * b["rel_res_true"]
