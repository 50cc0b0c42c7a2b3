"""Pins of the LFA sigma_c search (oracle/lfa.py) -- CPU only.

rho_loc itself is pinned elsewhere (the Fourier-mode test of the assembled
operator and the measured V-cycle contraction, tests/test_oracle_fem.py and
tests/test_oracle_twogrid.py).  sigma_c is pinned by its defining property
(rho_loc < 1 at sigma_c, >= 1 one tolerance below), by the monotonicity the
bisection assumes, and by the two trends the paper states: for a fixed
k a smaller h enlarges I_conv = [sigma_c, 2]; for a fixed h a larger k shrinks it."""
import math

import numpy as np
import pytest

from oracle import lfa


def _rho(k, h, s, m=24):
    return lfa.rho_loc(lfa.lam_of(k, 1.0, s), h, 0.6, 2, 2, m=m)


@pytest.mark.parametrize("kh", [0.5, 0.7])
def test_sigma_c_brackets_the_convergence_threshold(kh):
    h = 2.0 ** -5
    k = kh / h
    tol = 1e-2
    sc = lfa.sigma_c(k, h, m=24, tol=tol)
    assert 1.0 <= sc <= 2.0
    assert _rho(k, h, sc) < 1.0
    if sc > 1.0:
        assert _rho(k, h, sc - tol) >= 1.0


def test_rho_loc_decreases_with_the_shift_exponent():
    h = 2.0 ** -5
    k = 0.7 / h
    r = [_rho(k, h, s, m=16) for s in np.linspace(1.0, 2.0, 6)]
    assert all(a >= b for a, b in zip(r, r[1:])), r


def test_sigma_c_trends_stated_in_the_paper():
    # fixed k: a smaller h enlarges I_conv (sigma_c does not grow)
    k = 24.0
    s_coarse = lfa.sigma_c(k, 2.0 ** -5, m=24, tol=1e-2)
    s_fine = lfa.sigma_c(k, 2.0 ** -6, m=24, tol=1e-2)
    assert s_fine <= s_coarse
    # fixed h: a larger k shrinks I_conv (sigma_c does not fall)
    h = 2.0 ** -5
    s_small = lfa.sigma_c(0.4 / h, h, m=24, tol=1e-2)
    s_large = lfa.sigma_c(0.75 / h, h, m=24, tol=1e-2)
    assert s_large >= s_small


def test_sigma_c_ends():
    h = 2.0 ** -5
    assert lfa.sigma_c(0.2 / h, h, m=16, tol=1e-2) == 1.0          # converges without a strong shift
    assert math.isnan(lfa.sigma_c(0.9 / h, h, m=16, hi=1.05, tol=1e-2))   # no convergent sigma below 1.05
