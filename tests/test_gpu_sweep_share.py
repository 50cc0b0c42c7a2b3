"""The bench step itself at full size (-m gpu): rank 0's share of the cfg1 sweep
(440 samples, n up to 534, 8 engine streams, batched lockstep solves).  In its own
module so that no full-size handle of another test holds device memory."""
import pytest
import torch

pytestmark = pytest.mark.gpu

hh = pytest.importorskip("paper_2104_01439_b200.hh") if torch.cuda.is_available() else None


def test_fullsize_sweep_share_in_bench_configuration():
    """The bench step itself (rank 0's share of the cfg1 sweep: 440 samples, n up
    to 534, 8 engine streams, batched lockstep solves): every sample converges
    with rel_res_true <= rtol (a property at any size), and two of the largest
    samples (the fastest and the slowest to converge at the top grid size)
    match the oracle's iteration counts within +-1 (BASELINE tolerance)."""
    from oracle.solve import OracleProblem
    from workloads import sweep_samples
    from workloads.configs import sweep_sample_spec
    share = [s for s in sweep_samples() if s["id"] % 8 == 0]
    res = hh.sweep(share, o=hh.opts(restart=100, rtol=1e-6, max_iters=500))
    assert len(res) == len(share) == 440
    for s, r in zip(share, res):
        assert r["status"] == 0 and r["converged"] == 1, (s, r)
        assert r["rel_res_true"] <= 1.01e-6, (s, r)
    top = max(s["n"] for s in share)
    big = [(r["iterations"], i) for i, (s, r) in enumerate(zip(share, res)) if s["n"] == top]
    for _, i in (min(big), max(big)):
        _, ro = OracleProblem(sweep_sample_spec(share[i])).solve()
        assert abs(res[i]["iterations"] - ro.iterations) <= 1, (share[i], res[i], ro.iterations)
