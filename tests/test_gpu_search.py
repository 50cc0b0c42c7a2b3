"""GPU shift search (hh_shift_search) vs the oracle golden-section search (-m gpu)."""
import numpy as np
import pytest
import torch

from oracle.shift_search import rho_of, search_sample
from workloads.configs import search_rhs, search_sample_spec

pytestmark = pytest.mark.gpu

hh = pytest.importorskip("paper_2104_01439_b200.hh") if torch.cuda.is_available() else None

SAMPLES = [{"id": 0, "n": 16, "l": 4, "k": 8.0, "beta": 1.0},
           {"id": 1, "n": 16, "l": 4, "k": 11.5, "beta": 1.0},
           {"id": 2, "n": 32, "l": 5, "k": 20.0, "beta": 1.0},
           {"id": 3, "n": 32, "l": 5, "k": 9.0, "beta": 1.0}]


def test_shift_search_matches_oracle():
    rhs = [search_rhs(x, seed=0) for x in SAMPLES]
    res = hh.shift_search(SAMPLES, rhs)
    for x, r, b in zip(SAMPLES, res, rhs):
        so, ev = search_sample(search_sample_spec(x), b)
        assert r["status"] == 0 and r["evaluations"] == len(ev) == 12
        assert abs(r["sigma_hat"] - so) <= 1e-2
        assert abs(r["rho_best"] - min(v for _, v in ev)) <= 1e-3


def test_rho_parity_at_fixed_sigma():
    """One evaluation = one batched sweep solve with the sample's own rhs: rho
    equals the oracle's to 1e-8 relative when the iteration counts agree."""
    x = SAMPLES[2]
    b = search_rhs(x, seed=0)
    res = hh.shift_search([x], [b], lo=1.4, hi=1.4 + 1e-9, tol=1e-8)   # evaluates 1.4 + tiny
    r_o, its_o = rho_of(search_sample_spec(x), res[0]["sigma_best"], b)
    assert abs(res[0]["rho_best"] - r_o) <= 1e-8 * r_o


@pytest.mark.parametrize("name,n", [("cfg0", 64), ("cfg2", 64), ("cfg4", 12)])
def test_shift_map_solve_parity(name, n):
    """eps_e = beta k_e^{sigma_p(k_e, log2 n)} (Table 1 p = 1)
    evaluated per element on the device: A_eps, V-cycle and FGMRES vs the oracle."""
    from dataclasses import replace
    from oracle.solve import OracleProblem
    from workloads import config_spec
    spec = replace(config_spec(name, n=n), shift_map=1)
    orc = OracleProblem(spec)
    gp = hh.Problem.from_spec(spec)
    rng = np.random.default_rng(5)
    x = rng.standard_normal(spec.n_nodes) + 1j * rng.standard_normal(spec.n_nodes)
    y = gp.apply_op(hh.HH_OP_AEPS, torch.from_numpy(x).cuda()).cpu().numpy()
    ref = orc.apply(1, x)
    assert np.linalg.norm(y - ref) <= 1e-10 * np.linalg.norm(ref)
    z = gp.vcycle(torch.from_numpy(x).cuda()).cpu().numpy()
    zr = orc.vcycle(x)
    assert np.linalg.norm(z - zr) <= 1e-10 * np.linalg.norm(zr)
    _, rg = gp.fgmres_solve(torch.from_numpy(spec.rhs()).cuda(),
                            o=hh.opts(restart=spec.restart, rtol=spec.rtol))
    _, ro = orc.solve()
    assert abs(rg["iterations"] - ro.iterations) <= 1
    gp.close()
