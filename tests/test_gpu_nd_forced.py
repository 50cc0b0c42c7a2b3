"""The ND coarse-solve variants that only the full-size 3D grids select by
default, forced onto small 3D grids and checked against the oracle (-m gpu).

The switches are read once per process, so every variant runs
tests/nd_forced_check.py in a subprocess:
  * wide levels (k_nd_gather + k_nd_rows_wide<0|1>) on every level with >= 4
    rows (HH_ND_WIDE=4), front vectors read from L2 beyond 40 entries
    (HH_ND_VMAX=40), and the K-split backward rows (k_nd_bwdK + k_nd_bwdK_red)
    on fronts of order > 64 (HH_ND_BWDK_F=64);
  * the same with the K-split off (k_nd_rows_wide<1> on the long rows);
  * lean storage (transposed forward k_nd_fwdT + k_nd_fwdT_red, chunked
    factorisation with packed Schur complements) with a tiny workspace
    (HH_ND_LEAN=1, HH_ND_WMAX=20000) plus the wide levels;
  * the factorisation's large-front update paths (64-row tiles, pivot blocks
    of 32, DMMA or FMA update kernel) on every front of order >= 48.
Bars: coarse solve <= 1e-10 (residual <= 1e-11), V-cycle <= 1e-10, FGMRES
iterations +-1 and solution <= 1e-8 at equal counts (BASELINE north_star)."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANTS = {
    "wide_vmax_bwdk": {"HH_ND_WIDE": "4", "HH_ND_VMAX": "40", "HH_ND_BWDK_F": "64"},
    "wide_no_bwdk": {"HH_ND_WIDE": "4", "HH_ND_VMAX": "40", "HH_NO_BWDK": "1"},
    "lean_wide": {"HH_ND_LEAN": "1", "HH_ND_WMAX": "20000", "HH_ND_WIDE": "4", "HH_ND_BWDK_F": "64"},
    # the factorisation's large-front paths on small fronts: 64-row update tiles and
    # 32-pivot blocks on the FP64 tensor path (DMMA) and with the FMA update kernel
    "mma_nb32": {"HH_ND_UR64_F": "48", "HH_ND_NB32_F": "48"},
    "fma_ur64": {"HH_ND_MMA": "0", "HH_ND_UR64_F": "48", "HH_ND_NB32_F": "48"},
}


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_forced_nd_variant_parity(variant):
    env = dict(os.environ)
    env.update(VARIANTS[variant])
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "nd_forced_check.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    w = json.loads(r.stdout.strip().splitlines()[-1])
    assert w["coarse"] <= 1e-10 and w["coarse_res"] <= 1e-11, w
    assert w["vcycle"] <= 1e-10, w
    assert w["dits"] <= 1 and w["x"] <= 1e-8, w
