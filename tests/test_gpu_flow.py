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
    gp = hh.Problem.from_spec(spec, coarse_solver=hh.HH_COARSE_ND)
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
    res = hh.sweep(samples, coarse_solver=hh.HH_COARSE_ND)
    _set(monkeypatch, SCHEDULES[3])
    ref = hh.sweep(samples, coarse_solver=hh.HH_COARSE_ND)
    for a, c in zip(res, ref):
        assert a["status"] == 0 and a["iterations"] == c["iterations"]
        assert abs(a["rel_res_true"] - c["rel_res_true"]) <= 1e-8 * max(c["rel_res_true"], 1e-300) + 1e-14


# ---------------------------------------------------------------- failure path
# HH_ND_FLOW_POLLS=0 makes every dataflow dependency wait fail (fault injection).
# A failed wait must surface as an error (never a silent wrong coarse correction),
# and the handle must recover: counters reset, the schedule disabled for that
# tree.  Each case uses its own grid size, because the disable is per tree.
FORCE_FLOW = ("1", "-1", "99")


def test_flow_failure_fgmres_raises_then_recovers(monkeypatch):
    spec = config_spec("cfg0", n=96)
    gp = hh.Problem.from_spec(spec, coarse_solver=hh.HH_COARSE_ND)
    b = spec.rhs()
    _set(monkeypatch, FORCE_FLOW)
    monkeypatch.setenv("HH_ND_FLOW_POLLS", "0")
    with pytest.raises(hh.HHError) as e:
        gp.fgmres_solve(_dev(b), o=hh.opts(restart=spec.restart, rtol=spec.rtol))
    assert e.value.status == 4 and "dataflow" in str(e.value)
    monkeypatch.delenv("HH_ND_FLOW_POLLS")
    xo, ro = OracleProblem(spec).solve(b)
    x, r = gp.fgmres_solve(_dev(b), o=hh.opts(restart=spec.restart, rtol=spec.rtol,
                                              fixed_iters=ro.iterations))
    assert _rel(_host(x), xo) <= 1e-8
    gp.close()


def test_flow_failure_coarse_solve_raises_then_recovers(monkeypatch):
    spec = config_spec("cfg0", n=80)
    gp = hh.Problem.from_spec(spec, coarse_solver=hh.HH_COARSE_ND)
    orc = OracleProblem(spec)
    r = _rand(spec.n_coarse_nodes, 7)
    _set(monkeypatch, FORCE_FLOW)
    monkeypatch.setenv("HH_ND_FLOW_POLLS", "0")
    with pytest.raises(hh.HHError) as e:
        gp.coarse_solve(_dev(r))
    assert e.value.status == 4
    monkeypatch.delenv("HH_ND_FLOW_POLLS")
    e2 = _host(gp.coarse_solve(_dev(r)))
    assert _rel(e2, orc.tg.coarse.solve(r)) <= 1e-10
    gp.close()


def test_flow_failure_in_sweep_is_a_per_sample_error(monkeypatch):
    monkeypatch.setenv("HH_SWEEP_STREAMS", "1")
    _set(monkeypatch, FORCE_FLOW)
    monkeypatch.setenv("HH_ND_FLOW_POLLS", "0")
    samples = [{"id": i, "dim": 2, "n": 72, "k": 8.0 + i, "kh_target": 0.6, "sigma": 1.5,
                "beta": 0.5} for i in range(3)]
    res = hh.sweep(samples, coarse_solver=hh.HH_COARSE_ND)
    assert all(r["status"] == 4 and r["converged"] == 0 for r in res), res
    monkeypatch.delenv("HH_ND_FLOW_POLLS")
    res = hh.sweep(samples, coarse_solver=hh.HH_COARSE_ND)
    from workloads.configs import sweep_sample_spec
    for s, r in zip(samples, res):
        assert r["status"] == 0
        ro = OracleProblem(sweep_sample_spec(s)).solve()[1]
        assert abs(r["iterations"] - ro.iterations) <= 1
