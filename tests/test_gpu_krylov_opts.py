"""FGMRES options of the boundary against the oracle (-m gpu):
  * reorth = 1 (selective DGKS, threshold 1/sqrt 2: the oracle's own variant,
    reading C11) and reorth = 2 (CGS2): iterations +-1 and solution <= 1e-8 at
    equal counts;
  * x0 (PAPER.md:416 u^(0)): the solve starts from the given guess -- counts
    and solution match the oracle started from the same x0;
  * Arnoldi orthogonality of the GPU's single-pass CGS basis:
    max |<v_a, v_c> - delta_ac| <= 1e-8 (SURVEY.md 8(c) FGMRES pin)
    on the cfg2 medium and on the hardest sweep sample (sigma = 2, beta = 1,
    k = 160, n = 534), and <= 1e-12 with reorth = 2."""
import numpy as np
import pytest
import torch

from oracle.fgmres import fgmres
from oracle.solve import OracleProblem
from workloads import config_spec
from workloads.configs import sweep_sample_spec
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


@pytest.fixture(scope="module")
def cfg2m():
    spec = config_spec("cfg2", n=128)
    orc = OracleProblem(spec)
    gp = hh.Problem.from_spec(spec)
    yield spec, orc, gp
    gp.close()


@pytest.mark.parametrize("reorth", [1, 2])
def test_reorth_parity(cfg2m, reorth):
    spec, orc, gp = cfg2m
    b = spec.rhs()
    xo, ro = orc.solve(b)
    o = hh.opts(restart=spec.restart, rtol=spec.rtol, reorth=reorth)
    x, r = gp.fgmres_solve(_dev(b), o=o)
    assert abs(r["iterations"] - ro.iterations) <= 1 and r["converged"] == 1
    if r["iterations"] != ro.iterations:
        o = hh.opts(restart=spec.restart, rtol=spec.rtol, reorth=reorth, fixed_iters=ro.iterations)
        x, r = gp.fgmres_solve(_dev(b), o=o)
    assert _rel(_host(x), xo) <= 1e-8
    loss, nv = gp.arnoldi_orthogonality()
    assert nv == ro.iterations + 1 or nv == r["iterations"] + 1
    assert loss <= (1e-12 if reorth == 2 else 1e-10), loss


def test_reorth_short_restart_parity():
    """Restarted FGMRES(5) with reorth = 1: restart bookkeeping + second passes."""
    spec = config_spec("cfg0")
    spec.restart = 5
    orc = OracleProblem(spec)
    gp = hh.Problem.from_spec(spec)
    b = spec.rhs()
    xo, ro = orc.solve(b)
    o = hh.opts(restart=5, rtol=spec.rtol, reorth=1, fixed_iters=ro.iterations)
    x, r = gp.fgmres_solve(_dev(b), o=o)
    assert r["iterations"] == ro.iterations and r["restarts"] == ro.restarts
    assert _rel(_host(x), xo) <= 1e-8
    gp.close()


def test_x0_parity(cfg2m):
    spec, orc, gp = cfg2m
    b = spec.rhs()
    x0 = 1e-4 * random_complex(spec.n_nodes, 41)
    xo, ro = fgmres(lambda v: orc.A0 @ v, orc.tg.vcycle, b, restart=spec.restart, rtol=spec.rtol,
                    max_iters=spec.max_iters, x0=x0)
    x, r = gp.fgmres_solve(_dev(b), x=_dev(x0), o=hh.opts(restart=spec.restart, rtol=spec.rtol))
    assert abs(r["iterations"] - ro.iterations) <= 1 and r["converged"] == 1
    if r["iterations"] != ro.iterations:
        x, r = gp.fgmres_solve(_dev(b), x=_dev(x0), o=hh.opts(restart=spec.restart, rtol=spec.rtol,
                                                              fixed_iters=ro.iterations))
    assert _rel(_host(x), xo) <= 1e-8


def test_x0_exact_solution_converges_at_once(cfg2m):
    """x0 = the converged solution: r_0 is already below rtol ||b||, no Arnoldi step."""
    spec, orc, gp = cfg2m
    b = spec.rhs()
    x, r = gp.fgmres_solve(_dev(b), o=hh.opts(restart=spec.restart, rtol=1e-10))
    x2, r2 = gp.fgmres_solve(_dev(b), x=x.clone(), o=hh.opts(restart=spec.restart, rtol=1e-6))
    assert r2["iterations"] == 0 and r2["converged"] == 1
    assert _rel(_host(x2), _host(x)) == 0.0


def test_x0_host_entry_point(cfg2m):
    spec, orc, gp = cfg2m
    b = spec.rhs()
    x0 = 1e-4 * random_complex(spec.n_nodes, 42)
    xh = x0.copy()
    rep = gp.fgmres_solve_host(b, xh, hh.opts(restart=spec.restart, rtol=spec.rtol))
    xd, rd = gp.fgmres_solve(_dev(b), x=_dev(x0), o=hh.opts(restart=spec.restart, rtol=spec.rtol))
    assert rep["iterations"] == rd["iterations"]
    assert _rel(xh, _host(xd)) <= 1e-14


def test_single_pass_cgs_orthogonality_cfg2(cfg2m):
    spec, orc, gp = cfg2m
    gp.fgmres_solve(_dev(spec.rhs()), o=hh.opts(restart=spec.restart, rtol=spec.rtol))
    loss, nv = gp.arnoldi_orthogonality()
    assert nv > 5 and loss <= 1e-8, (loss, nv)


def test_single_pass_cgs_orthogonality_hardest_sweep_sample():
    s = {"id": 3409, "n": 534, "k": 160.0, "beta": 1.0, "sigma": 2.0, "kh_target": 0.3}
    spec = sweep_sample_spec(s)
    gp = hh.Problem.from_spec(spec)
    _, r = gp.fgmres_solve(_dev(spec.rhs()), o=hh.opts(restart=100, rtol=1e-6))
    assert r["converged"] == 1
    loss, nv = gp.arnoldi_orthogonality()
    assert nv > 50 and loss <= 1e-8, (loss, nv)
    gp.close()


def test_bad_options_are_config_errors(cfg2m):
    spec, orc, gp = cfg2m
    with pytest.raises(hh.HHError) as e:
        gp.fgmres_solve(_dev(spec.rhs()), o=hh.opts(reorth=3))
    assert e.value.status == 2
    with pytest.raises(hh.HHError) as e:
        hh.sweep([{"id": 0, "n": 8, "k": 5.0, "beta": 0.5, "sigma": 1.5}], o=hh.opts(restart=200))
    assert e.value.status == 2
    with pytest.raises(hh.HHError) as e:
        hh.sweep([{"id": 0, "n": 8, "k": 5.0, "beta": 0.5, "sigma": 1.5}], omega=1.5)
    assert e.value.status == 2
