"""Dataflow ND solve (one forward and one backward kernel over the per-level
range, CTAs released by per-front completion counters) against the CPU oracle
at the parity bars, under forced schedules (-m gpu).

The schedule variables are read at every solve, so each case switches the
schedule of the same handle; alternating schedules also checks that the
completion counters return to zero after every solve (a stale counter would
release a CTA before its children finished and break parity)."""
import numpy as np
import pytest
import torch

from oracle.solve import OracleProblem
from workloads import config_spec

pytestmark = pytest.mark.gpu

hh = pytest.importorskip("paper_2104_01439_b200.hh") if torch.cuda.is_available() else None

SCHEDULES = [   # (HH_ND_FLOW, HH_ND_CUT, HH_ND_SPLIT)
    ("1", "-1", "99"),    # every level in the dataflow kernels
    ("1", "1", "99"),     # subtree walk below, dataflow above
    ("1", "0", "4"),      # dataflow in the middle, cluster kernel on top
    ("0", "-1", "99"),    # per-level kernels (counters untouched)
]


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


@pytest.fixture(scope="module", params=["cfg0", "cfg2_n128"])
def pair(request):
    spec = config_spec("cfg0") if request.param == "cfg0" else config_spec("cfg2", n=128)
    orc = OracleProblem(spec)
    gp = hh.Problem.from_spec(spec)
    yield spec, orc, gp
    gp.close()


def _set(monkeypatch, sched):
    flow, cut, split = sched
    monkeypatch.setenv("HH_ND_FLOW", flow)
    monkeypatch.setenv("HH_ND_CUT", cut)
    monkeypatch.setenv("HH_ND_SPLIT", split)


def test_flow_coarse_solve_parity(pair, monkeypatch):
    spec, orc, gp = pair
    r = _rand(spec.n_coarse_nodes, 3)
    ref = orc.tg.coarse.solve(r)
    for rep in range(2):
        for sched in SCHEDULES:
            _set(monkeypatch, sched)
            e = _host(gp.coarse_solve(_dev(r)))
            assert _rel(e, ref) <= 1e-10, (sched, rep)


def test_flow_fgmres_parity(pair, monkeypatch):
    spec, orc, gp = pair
    b = spec.rhs()
    xo, ro = orc.solve(b)
    for sched in SCHEDULES[:3]:
        _set(monkeypatch, sched)
        x, r = gp.fgmres_solve(_dev(b), o=hh.opts(restart=spec.restart, rtol=spec.rtol,
                                                  fixed_iters=ro.iterations))
        assert _rel(_host(x), xo) <= 1e-8, sched


def test_flow_batched_sweep(monkeypatch):
    """A batch of samples (several sweep entries per launch, masked samples
    once they converge) through the dataflow kernels, single stream."""
    monkeypatch.setenv("HH_SWEEP_STREAMS", "1")
    _set(monkeypatch, SCHEDULES[0])
    samples = [{"id": i, "dim": 2, "n": 64, "k": 6.0 + i, "kh_target": 0.6, "sigma": 1.0 + 0.1 * i,
                "beta": 0.5} for i in range(6)]
    res = hh.sweep(samples)
    _set(monkeypatch, SCHEDULES[3])
    ref = hh.sweep(samples)
    for a, c in zip(res, ref):
        assert a["status"] == 0 and a["iterations"] == c["iterations"]
        assert abs(a["rel_res_true"] - c["rel_res_true"]) <= 1e-8 * max(c["rel_res_true"], 1e-300) + 1e-14
