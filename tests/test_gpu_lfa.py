"""LFA engine (hh_lfa_rho / hh_lfa_sigma_c) against
the oracle's transcription of the paper's symbols (oracle/lfa.py, numpy
eigenvalues) -- -m gpu, through the C ABI.

Tolerance: rho_loc is a maximum of spectral radii over the same theta grid on
both sides; the GPU takes the roots of the characteristic polynomial of the
diagonal-minus-rank-one symbol by Aberth iterations, whose accuracy near a
double root is ~sqrt(eps) ~ 1e-8, hence 1e-7 absolute.  sigma_c: both sides
bisect with the same midpoints, so they agree exactly unless a decision
rho < 1 falls within that tolerance of 1 (then within one bracket width)."""
import math

import pytest
import torch

from oracle import lfa

pytestmark = pytest.mark.gpu

hh = pytest.importorskip("paper_2104_01439_b200.hh") if torch.cuda.is_available() else None

H = 2.0 ** -5
QUERIES = [
    dict(k=0.3 / H, h=H, beta=1.0, sigma=1.0, omega=0.6, nu1=2, nu2=2, m=16),
    dict(k=0.5 / H, h=H, beta=1.0, sigma=1.5, omega=0.6, nu1=2, nu2=2, m=33),   # odd m: theta grid without 0
    dict(k=0.7 / H, h=H, beta=0.5, sigma=2.0, omega=0.6, nu1=1, nu2=1, m=24),
    dict(k=0.9 / H, h=H, beta=1.0, sigma=1.0, omega=1.0, nu1=0, nu2=2, m=20),   # divergent two-grid
    dict(k=0.6 / (2 * H), h=2 * H, beta=2.0, sigma=1.2, omega=0.8, nu1=3, nu2=1, m=12),
    dict(k=1.0, h=2.0 ** -8, beta=1.0, sigma=1.0, omega=0.6, nu1=2, nu2=2, m=8),  # Laplace-like limit
]


def _oracle_rho(q):
    return lfa.rho_loc(lfa.lam_of(q["k"], q["beta"], q["sigma"]), q["h"], q["omega"], q["nu1"], q["nu2"],
                       m=q["m"])


def test_lfa_rho_parity():
    got = hh.lfa_rho(QUERIES)
    for q, g in zip(QUERIES, got):
        assert abs(g - _oracle_rho(q)) <= 1e-7, (q, g)


def test_lfa_rho_batch_is_independent_of_batching():
    one = [hh.lfa_rho([q])[0] for q in QUERIES]
    assert one == hh.lfa_rho(QUERIES)


def test_lfa_sigma_c_parity():
    qs = [dict(k=kh / H, h=H, beta=1.0, omega=0.6, nu1=2, nu2=2, m=24) for kh in (0.2, 0.6, 0.8, 0.9)]
    got = hh.lfa_sigma_c(qs, tol=1e-2)
    for q, g in zip(qs, got):
        o = lfa.sigma_c(q["k"], q["h"], beta=q["beta"], omega=q["omega"], nu1=q["nu1"], nu2=q["nu2"],
                        m=q["m"], tol=1e-2)
        assert (math.isnan(o) and math.isnan(g)) or abs(g - o) <= 1e-2, (q, g, o)
    nan = hh.lfa_sigma_c([dict(k=0.9 / H, h=H, m=16)], hi=1.05, tol=1e-2)[0]
    assert math.isnan(nan)


def test_lfa_edge_cases():
    assert hh.lfa_rho([]) == []
    assert hh.lfa_sigma_c([]) == []
    with pytest.raises(hh.HHError) as e:
        hh.lfa_rho([dict(k=10.0, h=H, m=1)])
    assert e.value.status == 2
    with pytest.raises(hh.HHError) as e:
        hh.lfa_sigma_c([dict(k=10.0, h=H, m=8)], lo=2.0, hi=1.0)
    assert e.value.status == 2


def test_lfa_many_queries_span_launch_chunks():
    """More queries than one launch's grid.y (65,535): the host splits them."""
    n = 70000
    qs = [dict(k=(0.1 + 0.6 * (i % 7) / 6) / H, h=H, sigma=1.0 + (i % 5) * 0.25, m=4) for i in range(n)]
    got = hh.lfa_rho(qs)
    assert len(got) == n
    for i in (0, 1, 65534, 65535, 65536, n - 1):
        assert abs(got[i] - _oracle_rho(dict(qs[i], beta=1.0, omega=0.6, nu1=2, nu2=2))) <= 1e-7, i
