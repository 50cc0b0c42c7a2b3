"""Pins of the shift-search oracle and its input recipe."""
import math

import numpy as np
import pytest

from oracle.shift_search import golden_section, rho_of, search_sample
from workloads.configs import search_rhs, search_sample_spec, search_samples

PHI1 = (math.sqrt(5) - 1) / 2


def test_quadratic_minimum():
    s, ev = golden_section(lambda x: (x - 1.3) ** 2, 1.0, 2.0, 1e-2)
    assert abs(s - 1.3) <= 1e-2
    # ceil(log(tol / (b - a)) / log(1/phi)) reductions + 2 initial evaluations
    assert len(ev) == math.ceil(math.log(1e-2) / math.log(PHI1)) + 2 == 12


def test_boundary_minimum_and_bracket():
    s, ev = golden_section(lambda x: x, 1.0, 2.0, 1e-2)
    assert abs(s - 1.0) <= 1e-2
    assert all(1.0 <= x <= 2.0 for x, _ in ev)


def test_against_dense_scan():
    f = lambda x: abs(x - PHI1 - 1)           # minimum at 1.618...
    s, _ = golden_section(f, 1.0, 2.0, 1e-2)
    grid = np.linspace(1, 2, 1001)
    assert abs(s - grid[np.argmin([f(x) for x in grid])]) <= 1e-2


def test_bracket_shrinks_by_inverse_golden_ratio():
    # one evaluation per reduction by 1/phi: count = ceil(log(tol / width) / log(1/phi)) + 2
    for a, b, tol in [(0.0, 4.0, 1e-3), (1.0, 2.0, 0.3), (-5.0, 7.0, 1e-6)]:
        _, ev = golden_section(lambda x: (x - 0.77) ** 2, a, b, tol)
        assert len(ev) == math.ceil(math.log(tol / (b - a)) / math.log(PHI1) - 1e-12) + 2


def test_tie_keeps_right_bracket():
    s, _ = golden_section(lambda x: 0.0, 1.0, 2.0, 1e-2)
    assert s > 1.99


def test_search_recipe():
    smp = search_samples(50, seed=3)
    assert [x["id"] for x in smp] == list(range(50))
    for x in smp:
        assert x["n"] == 2 ** x["l"] and 4 <= x["l"] <= 10
        assert 3 * x["n"] / 16 <= x["k"] <= 3 * x["n"] / 4
    r = search_rhs(smp[0], seed=3)
    assert r.dtype == np.complex128 and np.all(r.imag == 0) and np.all(np.abs(r.real) <= 1)
    assert np.array_equal(r, search_rhs(smp[0], seed=3))
    assert not np.array_equal(r, search_rhs(smp[1], seed=3))


def test_search_sample_beats_a_sigma_scan():
    """SPEC example: rho at the searched sigma is within the golden-section
    tolerance slack of the best of an 11-point sigma scan (same rhs)."""
    x = {"id": 0, "n": 16, "l": 4, "k": 8.0, "beta": 1.0}
    spec = search_sample_spec(x)
    rhs = search_rhs(x, seed=0)
    s, ev = search_sample(spec, rhs)
    assert 1.0 <= s <= 2.0 and len(ev) == 12
    best = min(v for _, v in ev)
    scan = min(rho_of(spec, sg, rhs)[0] for sg in np.linspace(1, 2, 11))
    assert best <= scan + 5e-3
    r, its = rho_of(spec, 1.5, rhs)
    assert 0 < r < 1 and 1 <= its <= 50
