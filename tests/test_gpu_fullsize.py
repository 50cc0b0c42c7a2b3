"""Full-size checks (-m gpu) where the oracle cannot solve: BASELINE configs[4]
(cfg4: 257^3 fine nodes, 129^3 coarse, heterogeneous) and configs[2] (cfg2,
1025^2), in the launch configuration bench.py times, against the oracle on
SAMPLED outputs (oracle.fem.apply_rows evaluates single rows of A by the
element loop):
  * A_0 x and A_eps x on random x: sampled rows <= 1e-12 relative;
  * the FGMRES solution: sampled rows of b - A_0 x are below the rtol bound
    (|r_i| <= ||r||_2 <= rtol ||b||, a property at any size)."""
import numpy as np
import pytest
import torch

from oracle import fem
from oracle.solve import coefficients
from workloads import config_spec

pytestmark = pytest.mark.gpu

hh = pytest.importorskip("paper_2104_01439_b200.hh") if torch.cuda.is_available() else None


@pytest.fixture(scope="module", params=["cfg2", "cfg4"])
def full(request):
    spec = config_spec(request.param)
    gp = hh.Problem.from_spec(spec)
    yield spec, gp
    gp.close()


def _rows(spec, count, seed):
    rng = np.random.default_rng(seed)
    N1 = spec.n + 1
    rows = list(rng.integers(0, spec.n_nodes, count))
    # plus boundary / corner nodes and the source neighbourhood
    rows += [0, spec.n_nodes - 1, N1 - 1, spec.n // 2 * (N1 ** (spec.dim - 1))]
    return np.array(sorted(set(int(r) for r in rows)), dtype=np.int64)


def test_fullsize_apply_sampled_rows(full):
    spec, gp = full
    kf, ef, _, _ = coefficients(spec)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(spec.n_nodes) + 1j * rng.standard_normal(spec.n_nodes)
    xd = torch.from_numpy(x).cuda()
    rows = _rows(spec, 150, 4)
    for op, eps in ((hh.HH_OP_A0, 0.0 * ef), (hh.HH_OP_AEPS, ef)):
        y = gp.apply_op(op, xd)
        torch.cuda.synchronize()
        yr = y[torch.from_numpy(rows).cuda()].cpu().numpy()
        ref = fem.apply_rows(spec.dim, spec.n, kf, eps, x, rows)
        assert np.max(np.abs(yr - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_fullsize_solution_sampled_residual(full):
    spec, gp = full
    kf, _, _, _ = coefficients(spec)
    b = spec.rhs()
    x, r = gp.fgmres_solve(torch.from_numpy(b).cuda(), o=hh.opts(restart=spec.restart, rtol=spec.rtol))
    torch.cuda.synchronize()
    assert r["converged"] == 1 and r["rel_res_true"] <= spec.rtol
    xh = x.cpu().numpy()
    rows = _rows(spec, 150, 5)
    src = np.nonzero(b)[0]
    rows = np.unique(np.concatenate([rows, src]))
    res = b[rows] - fem.apply_rows(spec.dim, spec.n, kf, np.zeros_like(kf), xh, rows)
    assert np.max(np.abs(res)) <= spec.rtol * np.linalg.norm(b)

