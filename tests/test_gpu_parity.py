"""GPU <-> oracle parity through the C ABI (-m gpu).

Bars (BASELINE.json north_star): operator apply and V-cycle <= 1e-10 relative
2-norm; FGMRES iteration counts equal or +-1; solution <= 1e-8 relative (at
equal iteration counts, reading C12)."""
import numpy as np
import pytest
import torch

from oracle import fem
from oracle.solve import OracleProblem, coefficients
from oracle.twogrid import CoarseSolver
from workloads import config_spec, sweep_samples
from workloads.configs import ProblemSpec, sweep_sample_spec

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
    """Small-grid analogue of a constant-k config at the config's k*h."""
    spec = config_spec(name, n=n)
    full = config_spec(name)
    spec.k_const = full.k_const * n / full.n
    return spec


SPECS = [
    ("cfg0", lambda: config_spec("cfg0")),
    ("cfg0_n4", lambda: config_spec("cfg0", n=4)),
    ("cfg0_n6", lambda: config_spec("cfg0", n=6)),
    ("cfg0_n70", lambda: config_spec("cfg0", n=70)),            # ragged tiles
    ("cfg2_n64", lambda: config_spec("cfg2", n=64)),            # heterogeneous
    ("cfg2_n130", lambda: config_spec("cfg2", n=130)),
    ("cfg3_n8", lambda: _scaled("cfg3", 8)),                      # 3D constant k (cfg3 kh)
    ("cfg3_n14", lambda: _scaled("cfg3", 14)),
    ("cfg4_n12", lambda: config_spec("cfg4", n=12)),              # 3D heterogeneous
    ("sweep_k160_kh06", lambda: sweep_sample_spec(
        {"id": 0, "n": 268, "k": 160.0, "beta": 0.1, "sigma": 1.0, "kh_target": 0.6})),
]


# constant-k specs run twice: the default coarse solver (AUTO -> fast
# diagonalisation, fd.cu) and the nested-dissection factor forced (coarse_nd.cu);
# heterogeneous specs have the ND factor only
_CONST = {"cfg0", "cfg0_n4", "cfg0_n6", "cfg0_n70", "cfg3_n8", "cfg3_n14", "sweep_k160_kh06"}
PAIRS = [(name, mk, "auto") for name, mk in SPECS] + \
        [(name, mk, "nd") for name, mk in SPECS if name in _CONST]


@pytest.fixture(scope="module", params=PAIRS, ids=[f"{p[0]}-{p[2]}" for p in PAIRS])
def pair(request):
    name, mk, coarse = request.param
    spec = mk()
    orc = OracleProblem(spec)
    cs = hh.HH_COARSE_ND if coarse == "nd" else hh.HH_COARSE_AUTO
    gp = hh.Problem.from_spec(spec, coarse_solver=cs)
    # AUTO takes FD for constant k on resolved coarse grids (k h_c <= 2.5, include/hh.h)
    fd = coarse == "auto" and name in _CONST and spec.k_const / (spec.n // 2) <= 2.5
    want = hh.HH_COARSE_FD if fd else hh.HH_COARSE_ND
    assert gp.coarse_kind() == want, (name, coarse, gp.coarse_kind())
    yield spec, orc, gp
    gp.close()


def test_apply_op_parity(pair):
    spec, orc, gp = pair
    x = _rand(spec.n_nodes, 1)
    for op in (hh.HH_OP_A0, hh.HH_OP_AEPS):
        y = _host(gp.apply_op(op, _dev(x)))
        assert _rel(y, orc.apply(op, x)) <= 1e-10, op
    xc = _rand(spec.n_coarse_nodes, 2)
    yc = _host(gp.apply_op(hh.HH_OP_AEPS_COARSE, _dev(xc)))
    assert _rel(yc, orc.apply(2, xc)) <= 1e-10


def test_coarse_solve_parity(pair):
    spec, orc, gp = pair
    r = _rand(spec.n_coarse_nodes, 3)
    e = _host(gp.coarse_solve(_dev(r)))
    assert _rel(e, orc.tg.coarse.solve(r)) <= 1e-10
    assert _rel(orc.tg.Ac @ e, r) <= 1e-11


def test_vcycle_parity(pair):
    spec, orc, gp = pair
    for seed in (4, 5):
        f = _rand(spec.n_nodes, seed)
        z = _host(gp.vcycle(_dev(f)))
        assert _rel(z, orc.vcycle(f)) <= 1e-10


def test_fgmres_parity(pair):
    spec, orc, gp = pair
    b = spec.rhs()
    xo, ro = orc.solve(b)
    o = hh.opts(restart=spec.restart, rtol=spec.rtol, max_iters=spec.max_iters)
    xg, rg = gp.fgmres_solve(_dev(b), o=o, history=True)
    assert abs(rg["iterations"] - ro.iterations) <= 1, (rg, ro)
    assert rg["converged"] == int(ro.converged) == 1, (rg, ro)
    assert rg["rel_res_true"] <= 1.01 * spec.rtol
    if rg["iterations"] != ro.iterations:   # reading C12: compare at equal counts
        o2 = hh.opts(restart=spec.restart, rtol=spec.rtol, max_iters=spec.max_iters,
                     fixed_iters=ro.iterations)
        xg, rg = gp.fgmres_solve(_dev(b), o=o2)
    assert _rel(_host(xg), xo) <= 1e-8
    h = rg.get("history")
    if h:
        assert all(h[i + 1] <= h[i] * (1 + 1e-12) for i in range(len(h) - 1))


def test_fgmres_host_entry_point():
    spec = config_spec("cfg0")
    gp = hh.Problem.from_spec(spec)
    b = spec.rhs()
    x = np.zeros_like(b)
    rep = gp.fgmres_solve_host(b, x, hh.opts(restart=100, rtol=1e-6))
    xo, ro = OracleProblem(spec).solve(b)
    assert abs(rep["iterations"] - ro.iterations) <= 1
    if rep["iterations"] == ro.iterations:
        assert _rel(x, xo) <= 1e-8
    gp.close()


def test_errors_are_reported():
    with pytest.raises(hh.HHError) as e:
        hh.Problem(2, 7, k_const=10.0)          # odd n
    assert e.value.status == 2
    with pytest.raises(hh.HHError):
        hh.Problem(2, 8, k_const=10.0, omega=1.5)
    gp = hh.Problem(2, 8, k_const=10.0)
    with pytest.raises(ValueError):
        gp.apply_op(0, torch.zeros(5, dtype=torch.complex128, device="cuda"))
    gp.close()


def test_sweep_subset_matches_oracle():
    """hh_sweep on a strided subset of the cfg1 sweep: iteration counts +-1."""
    samples = sweep_samples()[::97][:24]
    res = hh.sweep(samples)
    for s, r in zip(samples, res):
        assert r["status"] == 0
        _, ro = OracleProblem(sweep_sample_spec(s)).solve()
        assert abs(r["iterations"] - ro.iterations) <= 1, (s, r, ro.iterations)
        assert r["converged"] == int(ro.converged)


def test_sweep_batch_equals_single_problem():
    """A batch of equal-n samples gives the same per-sample results as solving
    each sample alone (every kernel is sample-independent)."""
    samples = [s for s in sweep_samples() if s["n"] == 68][:12]
    res = hh.sweep(samples)
    for s, r in zip(samples, res):
        spec = sweep_sample_spec(s)
        gp = hh.Problem.from_spec(spec)
        _, rg = gp.fgmres_solve(_dev(spec.rhs()), o=hh.opts(restart=100, rtol=1e-6))
        gp.close()
        assert r["iterations"] == rg["iterations"], (s, r, rg)
        # reduction partitions differ with the batch size: equal up to round-off
        assert abs(r["rel_res_true"] - rg["rel_res_true"]) <= 1e-6 * rg["rel_res_true"] + 1e-18


def test_restarted_fgmres_parity():
    """Short restart cycles exercise the restart path (r = b - A_0 x, new basis)."""
    spec = config_spec("cfg0", n=32)
    spec.restart = 4
    orc = OracleProblem(spec)
    xo, ro = orc.solve()
    gp = hh.Problem.from_spec(spec, max_restart=8)
    xg, rg = gp.fgmres_solve(_dev(spec.rhs()), o=hh.opts(restart=4, rtol=spec.rtol))
    assert ro.restarts >= 1 and rg["restarts"] >= 1
    assert abs(rg["iterations"] - ro.iterations) <= 1, (rg, ro.iterations)
    if rg["iterations"] == ro.iterations:
        assert _rel(_host(xg), xo) <= 1e-8
    gp.close()


def test_fixed_iters_threshold_parity():
    """fixed_iters reproduces the oracle's iterate after exactly k steps (reading C12)."""
    spec = config_spec("cfg2", n=64)
    orc = OracleProblem(spec)
    gp = hh.Problem.from_spec(spec)
    for k in (1, 3, 7):
        xo, ro = orc.solve(fixed_iters=k)
        xg, rg = gp.fgmres_solve(_dev(spec.rhs()), o=hh.opts(fixed_iters=k))
        assert rg["iterations"] == k == ro.iterations
        assert _rel(_host(xg), xo) <= 1e-9
        assert abs(rg["rel_res_true"] - ro.rel_res_true) <= 1e-8 * ro.rel_res_true
    gp.close()


def test_zero_rhs_and_linearity_of_vcycle():
    """b = 0 returns x = 0 immediately; the V-cycle is linear."""
    spec = config_spec("cfg0", n=16)
    gp = hh.Problem.from_spec(spec)
    x, r = gp.fgmres_solve(torch.zeros(spec.n_nodes, dtype=torch.complex128, device="cuda"))
    assert r["iterations"] == 0 and r["converged"] == 1
    assert float(torch.linalg.vector_norm(x)) == 0.0
    f1, f2 = _rand(spec.n_nodes, 11), _rand(spec.n_nodes, 12)
    a, b2 = 0.7 - 0.3j, -1.1 + 2.0j
    z = _host(gp.vcycle(_dev(a * f1 + b2 * f2)))
    z12 = a * _host(gp.vcycle(_dev(f1))) + b2 * _host(gp.vcycle(_dev(f2)))
    assert _rel(z, z12) <= 1e-12
    gp.close()


def test_sweep_empty_and_smallest_grid():
    """An empty sweep is a no-op; the smallest grid (n = 4, one coarse cell per
    side... 3x3 coarse nodes) solves at the parity bar."""
    assert hh.sweep([]) == []
    s = {"id": 7, "dim": 2, "n": 4, "k": 1.5, "kh_target": 0.6, "sigma": 1.5, "beta": 0.5}
    r = hh.sweep([s])[0]
    _, ro = OracleProblem(sweep_sample_spec(s)).solve()
    assert r["status"] == 0 and abs(r["iterations"] - ro.iterations) <= 1


def test_nonconvergence_is_a_result():
    """Hitting max_iters is a result (converged = 0, status OK), not an error."""
    spec = config_spec("cfg0")
    gp = hh.Problem.from_spec(spec)
    x, r = gp.fgmres_solve(_dev(spec.rhs()), o=hh.opts(max_iters=3, rtol=1e-12))
    assert r["iterations"] == 3 and r["converged"] == 0 and r["rel_res_true"] > 1e-12
    xo, ro = OracleProblem(spec).solve(fixed_iters=3)
    assert _rel(_host(x), xo) <= 1e-9
    gp.close()


def test_lean_storage_with_slabs(monkeypatch):
    """Lean ND storage (cfg4's mode: chunked factorisation, packed Schur store,
    transposed forward) combined with in-process slabs, on a 3D heterogeneous
    grid whose coarse tree is created here for the first time."""
    monkeypatch.setenv("HH_ND_LEAN", "1")
    monkeypatch.setenv("HH_ND_WMAX", "30000")
    spec = config_spec("cfg4", n=18)
    gp = hh.Problem.from_spec(spec, nslabs_local=3)
    orc = OracleProblem(spec)
    x, r = gp.fgmres_solve(_dev(spec.rhs()), o=hh.opts(restart=spec.restart, rtol=spec.rtol))
    xo, ro = orc.solve()
    assert abs(r["iterations"] - ro.iterations) <= 1
    xf, _ = gp.fgmres_solve(_dev(spec.rhs()), o=hh.opts(restart=spec.restart, fixed_iters=ro.iterations))
    assert _rel(_host(xf), xo) <= 1e-8
    f = _rand(spec.n_nodes, 31)
    assert _rel(_host(gp.vcycle(_dev(f))), orc.vcycle(f)) <= 1e-10
    gp.close()
