"""Input generators (workloads/): the BASELINE.json configs as concrete inputs."""
import numpy as np

from workloads import config_spec, sweep_samples, point_source_weights, sweep_grid_n


def test_sweep_has_3520_samples_and_grid_rule():
    s = sweep_samples()
    assert len(s) == 16 * 2 * 11 * 10 == 3520
    for x in s:
        n = x["n"]
        assert n % 2 == 0 and x["k"] / n <= x["kh_target"] + 1e-12
        assert x["k"] / (n - 2) > x["kh_target"] or n == 4   # smallest even (C9)
    assert sweep_grid_n(160, 0.3) == 534 and sweep_grid_n(160, 0.6) == 268


def test_cfg2_medium_range():
    sp = config_spec("cfg2", n=1024)
    assert sp.k_fine.shape == (1024 ** 2,) and sp.k_coarse.shape == (512 ** 2,)
    assert abs(sp.k_fine.max() / 1024 - 0.5) < 1e-14          # max k h = 0.5
    assert 150 < sp.k_fine.min() < sp.k_fine.max()
    assert sp.k_coarse.max() <= 512 + 1e-9


def test_point_source_weights():
    idx, w = point_source_weights(1024, 2, (0.5, 0.1))      # reading C7/C8
    assert sorted(zip(idx.tolist(), w.tolist())) == \
        [(512 + 1025 * 102, 0.6000000000000014), (512 + 1025 * 103, 0.3999999999999986)] or \
        np.allclose(sorted(w), [0.4, 0.6])
    idx, w = point_source_weights(64, 2, (0.5, 0.5))
    assert idx.tolist() == [32 + 65 * 32] and w.tolist() == [1.0]
    idx, w = point_source_weights(128, 3, (0.5, 0.5, 0.5))
    assert idx.tolist() == [64 + 129 * 64 + 129 * 129 * 64]
